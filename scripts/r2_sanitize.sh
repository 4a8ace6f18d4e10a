#!/bin/bash
# compute-sanitizer passes over the small sliced-path workload (one tool each)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/sanitizer
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python scripts/sanitize_smoke.py c0 > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/summary.txt
  tail -3 gpurun_out/sanitizer/$tool.log >> gpurun_out/sanitizer/summary.txt
done
