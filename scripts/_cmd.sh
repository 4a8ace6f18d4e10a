# round evidence: GPU tests, bench (both arms), launch list, full ncu capture
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spread_ozp|k_gather_ozp|k_gdig|k_vmax|k_asm_p1" -s 10 -c 8 -o gpurun_out/prof_r01j python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
