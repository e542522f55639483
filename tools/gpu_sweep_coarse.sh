#!/bin/bash
# scratch helper: level-1 coarse-bucket target sweep on huge (9,80) batches and the (8,70) solve
for tgt in 2097152 8388608 16777216; do
  for q in 0.95 0.99; do
    MSP_COARSE_TARGET=$tgt timeout 300 python tools/run_alpha.py --m 9 --quantile $q --reps 2 > gpurun_out/sw_$tgt_$q.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/sw_$tgt_$q.json'));s=d['stats'];print('tgt $tgt q $q', round(d['wall_s'],4), s['hash_hits'], s['filtered_residuals'], s['kernel_launches'])"
  done
  MSP_COARSE_TARGET=$tgt timeout 300 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/sw8_$tgt.json 2>&1
  python -c "
import json;s=open('gpurun_out/sw8_$tgt.json').read();d=json.loads(s[s.find('{'):]);st=d['stats'];print('tgt $tgt (8,70)', st['dev_ms_total'], st['hash_hits'], st['filtered_residuals'])"
done
