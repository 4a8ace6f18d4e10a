cd $GRAFT_REPO_ROOT
timeout 600 python scripts/diag_det2.py c4 > gpurun_out/r2_det15.log 2>&1
