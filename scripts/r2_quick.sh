#!/bin/bash
# quick check of a kernel change: GPU test suite + the c4 bench line (+ c2/c3 with "all")
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
for c in c4 ${1:+c2 c3}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?" >> gpurun_out/bench_$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f'gpurun_out/bench_{c}.json')); ms = d['ms_per_step']
print(c, round(d['value'], 1), round(ms, 2), {k: round(v * ms, 2) for k, v in d['roofline']['stage_share'].items()},
      'e2e', round(d['e2e']['value'], 1), 'cg', d['cg'] and (round(d['cg']['solve_ms'], 1), d['cg']['iterations']),
      'frac', round(d['roofline']['frac'], 3), d['clocks'])
PY
done
