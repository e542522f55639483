#!/bin/bash
# A/B: bench each listed library variant (paper_2507_05045_b200/libmsp_<name>.so; "main" = default)
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2507_05045_b200/libmsp_b200.so
  [ "$v" != "main" ] && lib=paper_2507_05045_b200/libmsp_$v.so
  for rep in 1 2; do
    MSP_B200_LIB=$PWD/$lib timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-headline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', 'ms %.3f'%d['ms_per_step'],'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
