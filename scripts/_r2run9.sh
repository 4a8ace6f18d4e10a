cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
cp $L/libnld_b200.so /tmp/prod.so; cp $L/libnld_b200_ab.so $L/libnld_b200.so
export NLD_ALLOW_AB_BUILD=1
echo "--- spread on DMMA (gather sliced)" > gpurun_out/r2_det9.log
NLD_OZAKI_NO_SPREAD=1 timeout 300 python scripts/diag_det.py c1 32 10 >> gpurun_out/r2_det9.log 2>&1
NLD_OZAKI_NO_SPREAD=1 timeout 300 python scripts/diag_det.py c4 16 4 >> gpurun_out/r2_det9.log 2>&1
echo "--- gather on DMMA (spread sliced)" >> gpurun_out/r2_det9.log
NLD_OZAKI_NO_GATHER=1 timeout 300 python scripts/diag_det.py c1 32 10 >> gpurun_out/r2_det9.log 2>&1
NLD_OZAKI_NO_GATHER=1 timeout 300 python scripts/diag_det.py c4 16 4 >> gpurun_out/r2_det9.log 2>&1
cp /tmp/prod.so $L/libnld_b200.so
