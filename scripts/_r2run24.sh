cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02.csv python scripts/prof_step_pm.py c4 16 > gpurun_out/ncu_launch_r02.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_r02.csv > gpurun_out/launch_summary_r02.json 2>&1
