#!/bin/bash
# (9,80) two-level analysis: one huge batch timed, its launch list, full sections of level-1 k_scatter
# and level-2 k_waves; launch list of the full (9,80) solve
mkdir -p gpurun_out
T=${TAG:-r2y}
timeout 200 python tools/run_alpha.py --m 9 --quantile 0.9 --reps 2 > gpurun_out/${T}_alpha.json 2>&1; echo "alpha rc=$?"; tail -c 600 gpurun_out/${T}_alpha.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_alpha_launches.csv \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu_a.log 2>&1; echo "alpha launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scatter -s 2 -c 1 -o gpurun_out/${T}_scatter -f \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu_b.log 2>&1; echo "scatter prof rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_waves -s 0 -c 1 -o gpurun_out/${T}_waves2 -f \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu_c.log 2>&1; echo "waves prof rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_9_80_launches.csv \
    python tools/run_solve.py --m 9 --seed 1 > gpurun_out/${T}_ncu_d.log 2>&1; echo "9_80 launches rc=$?"
gzip -f gpurun_out/${T}_9_80_launches.csv
