#!/bin/bash
# Round-2 evidence at HEAD: GPU tests, smoke, bench lines (c4/c2/c3 + reference
# arm), then -- after those exited -- the ncu launch list and one full capture.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash scripts/r2_configs.sh
bash scripts/r2_ncu.sh c4 final
