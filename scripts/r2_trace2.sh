#!/bin/bash
# wait-site timelines of CTA 0 (trace build) for the default kernels and for A/B switch sets
# usage: scripts/r2_trace2.sh "NLD_GX=8" "NLD_GX=128" ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SCR=$(mktemp -d); cp -r . $SCR/repo 2>/dev/null
cp paper_2407_06834_b200/libnld_b200_tr.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
i=0
for envs in "" "$@"; do
  mkdir -p gpurun_out/trace$i
  (cd $SCR/repo && env NLD_ALLOW_AB_BUILD=1 NLD_TRACE_DIR=$GRAFT_REPO_ROOT/gpurun_out/trace$i $envs timeout 300 python scripts/prof_step_pm.py c4 16) > gpurun_out/trace$i/run.log 2>&1
  echo "$envs" > gpurun_out/trace$i/env.txt
  # keep one launch of each kernel (the merge back is capped at 64 MiB)
  find gpurun_out/trace$i -name '*.txt' ! -name 'gather_nm_4.txt' ! -name 'spread_4.txt' ! -name 'env.txt' -delete
  i=$((i+1))
done
rm -rf $SCR
