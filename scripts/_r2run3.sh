cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/r2_b3_hint.json 2> gpurun_out/r2_b3_hint.err
cp $L/libnld_b200.so /tmp/hint.so; cp $L/libnld_b200_nohint.so $L/libnld_b200.so
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/r2_b3_nohint.json 2> gpurun_out/r2_b3_nohint.err
cp /tmp/hint.so $L/libnld_b200.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_nm|k_spread_ozp" -s 3 -c 2 -o gpurun_out/prof_r02a python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_r02a.log 2>&1
tail -2 gpurun_out/ncu_r02a.log
