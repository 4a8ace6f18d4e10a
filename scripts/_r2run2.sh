cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_smoke2.log
timeout 1500 python -m pytest tests -q -m gpu -s -x -k "sliced or fused or nonfinite or sweep or variants" > gpurun_out/r2_t3.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_b2.json 2> gpurun_out/r2_b2.err
