#!/bin/bash
# full GPU test suite + smoke + bench lines for c4 (default), c2 and c3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in c4 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log
for c in c4 c2 c3; do python - $c <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f'gpurun_out/bench_{c}.json')); ms = d['ms_per_step']
print(c, round(d['value'], 1), round(ms, 2), {k: round(v * ms, 2) for k, v in d['roofline']['stage_share'].items()},
      'e2e', round(d['e2e']['value'], 1), 'cg', d['cg'] and (round(d['cg']['solve_ms'], 1), d['cg']['iterations']),
      'single', d.get('single_rhs') and round(d['single_rhs']['value'], 1), 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'])
PY
done
