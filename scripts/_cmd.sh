timeout 60 python scripts/umma/oz_harness.py 100 1e6 50900
timeout 60 python scripts/umma/oz_harness.py 3 1 33 70
python scripts/oz_check.py c4 16 /tmp/a4.npy 2>&1 | tail -1
NLD_OZAKI=1 timeout 120 python scripts/oz_check.py c4 16 /tmp/b4.npy 2>&1 | tail -1
python scripts/oz_check.py cmp /tmp/b4.npy /tmp/a4.npy
NLD_OZAKI=1 bash scripts/ab_env.sh oz "X=0"
NLD_OZAKI=1 python scripts/prof_step_pm.py c4 16 > /dev/null 2>&1; NLD_OZAKI=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_oz" -s 3 -c 1 -o gpurun_out/prof_oz3 python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_oz3.log 2>&1
