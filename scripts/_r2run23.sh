cd $GRAFT_REPO_ROOT
L=paper_2407_06834_b200
cp $L/libnld_b200.so /tmp/prod.so; cp $L/libnld_b200_prof.so $L/libnld_b200.so
timeout 600 python scripts/prof_step_pm.py c4 16 > gpurun_out/r2_prof23.log 2>&1
cp /tmp/prod.so $L/libnld_b200.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_nm|k_spread_ozp" -s 3 -c 2 -o gpurun_out/prof_r02c python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_r02c.log 2>&1
