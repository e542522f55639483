#!/bin/bash
# timeline of repeated huge-batch joins: stream ms per phase, to catch the slow outliers
MSP_TIMELINE=1 MSP_B200_LIB=$PWD/paper_2507_05045_b200/libmsp_${1:-old}.so python tools/run_alpha.py --m 9 --quantile 0.9 --reps 10 2>&1 | python -c "
import sys,re
prev=None; row=[]
for l in sys.stdin:
    m=re.match(r'\[msp timeline\] (.+?)\s+host\s+([\d.]+) ms\s+stream\s+([\d.]+) ms', l)
    if not m:
        if l.startswith('{'): print(l[:200])
        continue
    name, h, s = m.group(1).strip(), float(m.group(2)), float(m.group(3))
    if name=='plan done': row=[]; prev=s
    else: row.append('%s %.1f' % (name.split()[-1], s-prev)); prev=s
    if name=='end': print(' | '.join(row))
"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
