#!/bin/bash
# usage: ab_env.sh TAG "ENV=1 ENV2=0" ...
while [ $# -gt 1 ]; do
  tag=$1; envs=$2; shift 2
  env $envs timeout 600 python bench.py --steps 8 --warmup 2 --no-cpu --no-cg > gpurun_out/abe_$tag.json 2>gpurun_out/abe_$tag.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/abe_$tag.json')); print('$tag', round(d['value'],2), round(d['ms_per_step'],2), {k:round(v*d['ms_per_step'],2) for k,v in d['roofline']['stage_share'].items()})"
done
