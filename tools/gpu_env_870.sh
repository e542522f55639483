#!/bin/bash
# A/B of an environment knob on the full (8,70) s1 solve (device ms), 3 processes each
for e in "$@"; do
  for rep in 1 2 3; do
    if [ "$e" = "-" ]; then timeout 200 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/e870.json 2>&1
    else env $e timeout 200 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/e870.json 2>&1; fi
    python -c "import json;s=open('gpurun_out/e870.json').read();d=json.loads(s[s.index('{'):]);print('$e', 'dev_ms %.1f join %.1f' % (d['stats']['dev_ms_total'], d['stats']['dev_ms_join']))"
  done
done
