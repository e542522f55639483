#!/bin/bash
for v in old pf8c64; do for wk in 6000000 12000000 24000000 0; do
MSP_B200_LIB=$PWD/paper_2507_05045_b200/libmsp_$v.so timeout 120 python tools/run_alpha.py --m 9 --quantile 0.9 --reps 4 --wave-keys $wk > gpurun_out/wk.json 2>&1
python -c "import json;s=open('gpurun_out/wk.json').read();d=json.loads(s[s.index('{'):]);print('$v', $wk, d['rep_dev_ms_join'])"
done; done
