#!/bin/bash
# A/B of an environment knob on one huge (9,80) batch: "VAR=value" pairs as arguments ("-" = none)
for e in "$@"; do
  for rep in 1 2; do
    if [ "$e" = "-" ]; then timeout 120 python tools/run_alpha.py --m 9 --quantile 0.9 --reps 8 > gpurun_out/env.json 2>&1
    else env $e timeout 120 python tools/run_alpha.py --m 9 --quantile 0.9 --reps 8 > gpurun_out/env.json 2>&1; fi
    python -c "import json;s=open('gpurun_out/env.json').read();d=json.loads(s[s.index('{'):]);r=sorted(d['rep_dev_ms_join'][1:]);print('$e', 'join ms min %.2f med %.2f' % (r[0], r[len(r)//2]))"
  done
done
