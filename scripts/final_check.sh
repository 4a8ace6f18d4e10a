# final evidence pass: smoke, GPU tests, the three bench configs, the reference arm
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/final_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; echo pytest rc=$? >> gpurun_out/final_gputest.log
timeout 600 python bench.py > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err; echo rc=$?
timeout 600 python bench.py --config c2 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err; echo rc=$?
timeout 600 python bench.py --config c3 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo rc=$?
tail -n 3 gpurun_out/final_smoke.log gpurun_out/final_gputest.log
for c in c4 c2 c3; do python -c "
import json; d=json.load(open('gpurun_out/final_bench_$c.json')); print('$c', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), 'cg', d.get('cg',{}).get('ms'), d['roofline']['frac'], d['clocks'])"; done
