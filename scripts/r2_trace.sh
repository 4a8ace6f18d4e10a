#!/bin/bash
# wait-site timeline of CTA 0 (NLD_OZ_TRACE build, libnld_b200_tr.so) for one c4 product
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/trace
SCR=$(mktemp -d); cp -r . $SCR/repo 2>/dev/null
cp paper_2407_06834_b200/libnld_b200_tr.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
(cd $SCR/repo && NLD_ALLOW_AB_BUILD=1 NLD_TRACE_DIR=$GRAFT_REPO_ROOT/gpurun_out/trace timeout 300 python scripts/prof_step_pm.py ${1:-c4} 16) > gpurun_out/trace/run.log 2>&1
rm -rf $SCR
ls gpurun_out/trace | head
