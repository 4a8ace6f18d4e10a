cd $GRAFT_REPO_ROOT
timeout 900 python scripts/diag_det3.py c4 > gpurun_out/r2_det18.log 2>&1
