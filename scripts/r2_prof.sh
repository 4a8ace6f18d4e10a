#!/bin/bash
# per-site pipeline-wait clocks (NLD_OZ_PROF build) of one c4 product, on a scratch copy
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SCR=$(mktemp -d); cp -r . $SCR/repo 2>/dev/null
cp paper_2407_06834_b200/libnld_b200_prof.so $SCR/repo/paper_2407_06834_b200/libnld_b200.so
(cd $SCR/repo && timeout 300 python scripts/prof_step_pm.py ${1:-c4} 16) > gpurun_out/ozprof_${1:-c4}.log 2>&1
rm -rf $SCR
