cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -s -k "sliced_configs or nonfinite or sweep_matches" > gpurun_out/r2_t1.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t1.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_t2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t2.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_b1.json 2> gpurun_out/r2_b1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2_bref.json 2> gpurun_out/r2_bref.err
