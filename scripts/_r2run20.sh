cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
cp $L/libnld_b200.so /tmp/prod.so; cp $L/libnld_b200_check.so $L/libnld_b200.so
timeout 300 python scripts/diag_det.py c4 16 2 > gpurun_out/r2_chk20.log 2>&1
cp /tmp/prod.so $L/libnld_b200.so
