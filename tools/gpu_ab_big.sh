#!/bin/bash
# A/B of library variants on full (8,70) and (9,80) s1 enumerations (device ms)
for v in "$@"; do
  lib=paper_2507_05045_b200/libmsp_b200.so
  [ "$v" != "main" ] && lib=paper_2507_05045_b200/libmsp_$v.so
  for m in 8 9; do
    MSP_B200_LIB=$PWD/$lib timeout 300 python tools/run_solve.py --m $m --seed 1 > gpurun_out/abb_${v}_$m.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/abb_${v}_$m.json'));print('$v', $m, 'dev_ms', round(d['stats']['dev_ms_total'],1), 'hh', d['stats']['hash_hits'], 'sols', len(d['solutions']))"
  done
done
