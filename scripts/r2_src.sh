#!/bin/bash
# Source-level ncu capture (one launch each) of the c4 spread and final gather:
# SASS lines with their shared-memory wavefronts, conflicts and stall samples.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CFG=${1:-c4}; TAG=${2:-src}
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_spread_ozp" -c 1 -o gpurun_out/${TAG}_spread -f \
  python scripts/prof_step_pm.py $CFG 16 > gpurun_out/${TAG}_spread.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gather_nm" -s 2 -c 1 -o gpurun_out/${TAG}_gather -f \
  python scripts/prof_step_pm.py $CFG 16 > gpurun_out/${TAG}_gather.log 2>&1
for k in spread gather; do
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page source --print-source sass --csv > gpurun_out/${TAG}_${k}_sass.csv 2>&1
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>&1
done
echo done
