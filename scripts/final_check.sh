set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/final_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; echo pytest rc=$? >> gpurun_out/final_gputest.log
timeout 600 python bench.py > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo rc=$?
tail -3 gpurun_out/final_smoke.log gpurun_out/final_gputest.log; cat gpurun_out/final_bench_c4.json | cut -c1-400
