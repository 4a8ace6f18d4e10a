cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
cp $L/libnld_b200.so /tmp/prod.so; cp $L/libnld_b200_ab.so $L/libnld_b200.so
export NLD_ALLOW_AB_BUILD=1
echo "--- no fused epilogue" > gpurun_out/r2_det16.log
NLD_NO_FUSED_EPILOGUE=1 timeout 300 python scripts/diag_det.py c4 16 3 >> gpurun_out/r2_det16.log 2>&1
echo "--- no overlap" >> gpurun_out/r2_det16.log
NLD_NO_OVERLAP=1 timeout 300 python scripts/diag_det.py c4 16 3 >> gpurun_out/r2_det16.log 2>&1
echo "--- default (ab build)" >> gpurun_out/r2_det16.log
timeout 300 python scripts/diag_det.py c4 16 3 >> gpurun_out/r2_det16.log 2>&1
cp /tmp/prod.so $L/libnld_b200.so
