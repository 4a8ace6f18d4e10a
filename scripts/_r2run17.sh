cd $GRAFT_REPO_ROOT
timeout 600 python scripts/diag_unwritten.py c4 > gpurun_out/r2_unw17.log 2>&1
timeout 600 python scripts/diag_unwritten.py c1 >> gpurun_out/r2_unw17.log 2>&1
