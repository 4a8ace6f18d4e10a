#!/bin/bash
# quick GPU check: sliced-path parity tests + smoke + one bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${TESTS:-tests/test_gpu_sliced_configs.py tests/test_gpu_variants.py tests/test_gpu_parity.py}
timeout 900 python -m pytest $T -x -q > gpurun_out/chk_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/chk_smoke.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3 --no-cpu --e2e-steps 4} > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/chk_bench.json')); ms=d['ms_per_step']
print('bench', round(d['value'],1), round(ms,2), {k:round(v*ms,2) for k,v in d['roofline']['stage_share'].items()}, 'cg', d['cg'] and round(d['cg']['solve_ms'],1), 'clk', d['clocks'])
PY
tail -2 gpurun_out/chk_tests.log; tail -2 gpurun_out/chk_smoke.log
