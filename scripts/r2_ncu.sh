#!/bin/bash
# ncu evidence of one c4 16-rhs product: launch list + full capture of the sliced kernels
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CFG=${1:-c4}; TAG=${2:-r02a}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CFG}_${TAG}.csv python scripts/prof_step_pm.py $CFG 16 > gpurun_out/ncu_list_${CFG}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gather_nm|k_spread_ozp|k_gdig_nm|k_vmax" -c 10 -o gpurun_out/prof_${CFG}_${TAG} -f \
  python scripts/prof_step_pm.py $CFG 16 > gpurun_out/ncu_full_${CFG}.log 2>&1
echo done >> gpurun_out/ncu_full_${CFG}.log
