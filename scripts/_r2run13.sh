cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
cp $L/libnld_b200.so /tmp/prod.so
for v in r1 old1; do
  cp $L/libnld_b200_$v.so $L/libnld_b200.so
  echo "--- $v" >> gpurun_out/r2_det13.log
  timeout 300 python scripts/diag_det.py c4 16 3 >> gpurun_out/r2_det13.log 2>&1
  timeout 300 python scripts/diag_det.py c1 32 10 >> gpurun_out/r2_det13.log 2>&1
done
cp /tmp/prod.so $L/libnld_b200.so
