#!/bin/bash
# scratch helper: (9,80) full solve + single huge batches under library variants, with debug stats
mkdir -p gpurun_out
for v in ${VARIANTS:-old mid b200}; do
  for q in 0.5 0.95; do
    MSP_DEBUG_STATS=1 MSP_B200_LIB=paper_2507_05045_b200/libmsp_$v.so timeout 300 python tools/run_alpha.py --m 9 --quantile $q > gpurun_out/alpha_${v}_$q.json 2> gpurun_out/alpha_${v}_$q.err
    echo "$v q=$q rc=$?"; python -c "import json;d=json.load(open('gpurun_out/alpha_${v}_$q.json'));print(d['wall_s'], d['stats']['kernel_launches'], d['stats']['waves'])"; grep "overflow" gpurun_out/alpha_${v}_$q.err | head -4
  done
done
for v in ${FULL:-old b200}; do
  MSP_DEBUG_STATS=1 MSP_B200_LIB=paper_2507_05045_b200/libmsp_$v.so timeout 600 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/full_${v}.json 2> gpurun_out/full_${v}.err
  echo "full $v rc=$?"; tail -c 400 gpurun_out/full_${v}.json; echo; grep "msp dbg" gpurun_out/full_${v}.err | head
done
