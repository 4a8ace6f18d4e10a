#!/bin/bash
# A/B the test-only library variants (make -C paper_2407_06834_b200/csrc variant
# TAG=x DEFS="... -DNLD_AB_BUILD"): each is swapped in for the product .so on a
# scratch copy of the repo, so the package itself only ever loads its own build.
# usage: scripts/ab.sh [tag ...]   (default: every libnld_b200_*.so); ENV="X=1" extra env
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
SCR=$(mktemp -d)
cp -r . $SCR/repo 2>/dev/null || true
tags="$@"
[ -z "$tags" ] && tags=$(ls paper_2407_06834_b200/libnld_b200_*.so | sed 's/.*libnld_b200_//; s/\.so//')
CFG=${CFG:-c4}
for tag in $tags; do
  cp paper_2407_06834_b200/libnld_b200_$tag.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
  (cd $SCR/repo && env NLD_ALLOW_AB_BUILD=1 $ENV timeout 600 python bench.py --config $CFG --nrhs 16 --steps 8 --warmup 2 --no-cpu --no-cg --e2e-steps 2) > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); ms=d['ms_per_step']; print('$tag', round(d['value'],1), round(ms,2), {k:round(v*ms,2) for k,v in d['roofline']['stage_share'].items()}, 'MHz', d['clocks']['sm_mhz'], 'Mcycles', round(ms*d['clocks']['sm_mhz']/1e3,2))" || tail -3 gpurun_out/ab_$tag.err
done
rm -rf $SCR
