#!/bin/bash
# A/B the test-only library variants (make -C paper_2407_06834_b200/csrc variant
# TAG=x DEFS=...): each is swapped in for the product .so on a scratch copy of
# the repo, so the package itself only ever loads its own build.
set -e
SCR=$(mktemp -d)
cp -r . $SCR/repo 2>/dev/null || true
for lib in paper_2407_06834_b200/libnld_b200_*.so; do
  tag=$(basename $lib .so)
  cp $lib $SCR/repo/paper_2407_06834_b200/libnld_b200.so
  (cd $SCR/repo && timeout 600 python bench.py --steps 8 --warmup 2 --no-cpu --no-cg --e2e-steps 2) > gpurun_out/ab_$tag.json 2>/dev/null || true
  python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); print('$tag', round(d['value'],2), round(d['ms_per_step'],2), {k:round(v*d['ms_per_step'],2) for k,v in d['roofline']['stage_share'].items()})" || true
done
rm -rf $SCR
