#!/bin/bash
# A/B of library variants on one huge (9,80) batch (two-level path): device ms of the join, 3 reps
for v in "$@"; do
  lib=paper_2507_05045_b200/libmsp_b200.so
  [ "$v" != "main" ] && lib=paper_2507_05045_b200/libmsp_$v.so
  for q in ${QS:-0.9 0.5}; do
    MSP_B200_LIB=$PWD/$lib timeout 120 python tools/run_alpha.py --m 9 --quantile $q --reps 8 > gpurun_out/aba_${v}.json 2>&1
    python -c "import json;s=open('gpurun_out/aba_${v}.json').read();d=json.loads(s[s.index('{'):]);r=sorted(d['rep_dev_ms_join'][1:]);print('$v', $q, 'join ms min %.2f med %.2f' % (r[0], r[len(r)//2]), 'hh', d['stats']['hash_hits'], 'keys', d['n_left']+d['n_right'])"
  done
done
