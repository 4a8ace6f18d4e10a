cd $GRAFT_REPO_ROOT
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name regex:k_gather_nm --print-limit 30 python scripts/diag_small.py c1 16 > gpurun_out/r2_race11.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --kernel-name regex:k_gather_nm --print-limit 30 python scripts/diag_small.py c1 16 > gpurun_out/r2_sync11.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --kernel-name regex:k_gather_nm --print-limit 30 python scripts/diag_small.py c1 16 > gpurun_out/r2_mem11.log 2>&1
