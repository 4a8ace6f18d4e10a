#!/bin/bash
# A/B the library variants built by `make variant` (bench, 16-rhs c4)
for lib in paper_2407_06834_b200/libnld_b200*.so; do
  tag=$(basename $lib .so)
  NLD_LIB=$PWD/$lib timeout 600 python bench.py --steps 8 --warmup 2 --no-cpu --no-cg > gpurun_out/ab_$tag.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab_$tag.json')); print('$tag', round(d['value'],2), round(d['ms_per_step'],2), {k:round(v*d['ms_per_step'],2) for k,v in d['roofline']['stage_share'].items()})"
done
