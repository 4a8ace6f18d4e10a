python bench.py --steps 10 --warmup 3 > gpurun_out/bench_oz.json 2> gpurun_out/bench_oz.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python scripts/prof_step_pm.py c4 16 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_oz.csv python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread_oz|k_gather_oz|k_vmax|k_asm_p1" -s 10 -c 8 -o gpurun_out/prof_r01e python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
