cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
timeout 300 python scripts/diag_cols.py c1 32 > gpurun_out/r2_diag7.log 2>&1
timeout 300 python scripts/diag_cols.py c1 16 >> gpurun_out/r2_diag7.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "sliced or fused or nonfinite or sweep or variants or matvec or edge" > gpurun_out/r2_t7.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t7.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/r2_b7.json 2> gpurun_out/r2_b7.err
cp $L/libnld_b200.so /tmp/prod.so; cp $L/libnld_b200_prof.so $L/libnld_b200.so
timeout 600 python scripts/prof_step_pm.py c4 16 > gpurun_out/r2_prof7.log 2>&1
cp /tmp/prod.so $L/libnld_b200.so
