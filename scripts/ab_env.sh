#!/bin/bash
# A/B of environment switches on the test-only A/B build (libnld_b200_ab.so,
# make -C paper_2407_06834_b200/csrc ab), swapped in on a scratch copy.
# usage: scripts/ab_env.sh "VAR=val VAR2=val" "VAR=val" ...   ("" = defaults)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SCR=$(mktemp -d); cp -r . $SCR/repo 2>/dev/null
cp paper_2407_06834_b200/libnld_b200_${LIB:-ab}.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
CFG=${CFG:-c4}
i=0
for envs in "$@"; do
  i=$((i+1))
  (cd $SCR/repo && env NLD_ALLOW_AB_BUILD=1 $envs timeout 600 python bench.py --config $CFG --nrhs 16 --steps 8 --warmup 2 --no-cpu --no-cg --e2e-steps 2) > gpurun_out/abenv_$i.json 2>gpurun_out/abenv_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/abenv_$i.json')); ms=d['ms_per_step']; print('${LIB:-ab} [$envs]', round(d['value'],1), round(ms,2), {k:round(v*ms,2) for k,v in d['roofline']['stage_share'].items()})" || tail -3 gpurun_out/abenv_$i.err
done
rm -rf $SCR
