cd $GRAFT_REPO_ROOT
timeout 300 python scripts/diag_det.py c4 16 4 > gpurun_out/r2_det19.log 2>&1
timeout 300 python scripts/diag_det.py c1 32 10 >> gpurun_out/r2_det19.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "sliced or fused or nonfinite or sweep or variants or matvec or edge" > gpurun_out/r2_t19.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t19.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/r2_b19.json 2> gpurun_out/r2_b19.err
