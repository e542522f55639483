#!/bin/bash
# scratch helper: launch list of one (7,60) solve + ncu full of one mid-solve scatter and join
mkdir -p gpurun_out
export MSP_WAVE_BUCKETS=${WB:-512}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lq.csv python tools/diag_time.py 7 1 0 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_scatter|k_join" --launch-skip 200 -c 2 -o gpurun_out/prof_new -f python tools/diag_time.py 7 1 0 1 > gpurun_out/prof_new.log 2>&1
echo done
