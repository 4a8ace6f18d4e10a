cd $GRAFT_REPO_ROOT
./scripts/probes/pipes > gpurun_out/r2_pipes.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "sliced or fused or nonfinite or sweep or variants or matvec" > gpurun_out/r2_t4.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t4.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/r2_b4.json 2> gpurun_out/r2_b4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_nm" -s 4 -c 1 -o gpurun_out/prof_r02b python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_r02b.log 2>&1
