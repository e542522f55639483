#!/bin/bash
# profiles for profiles/: bench line, launch list of the bench command, ncu --set full of k_waves
mkdir -p gpurun_out
T=${TAG:-r2}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-headline > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-headline > gpurun_out/${T}_ncu1.log 2>&1; echo "launches rc=$?"
timeout 120 python tools/rep_solve.py 7 2 > gpurun_out/${T}_rep.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_waves -s 1 -c 1 -o gpurun_out/${T}_prof -f \
    python tools/rep_solve.py 7 2 > gpurun_out/${T}_ncu2.log 2>&1; echo "prof rc=$?"
# the huge-batch (two-level) kernels of one (9,80) batch (quantile 0.9 of the plan's costs):
# level-1 k_scatter (first launch) and level-2 k_waves
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scatter -s 0 -c 1 -o gpurun_out/${T}_l1 -f \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu3.log 2>&1; echo "l1 prof rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_waves -s 0 -c 1 -o gpurun_out/${T}_l2 -f \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu4.log 2>&1; echo "l2 prof rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_alpha_launches.csv \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/${T}_ncu5.log 2>&1; echo "alpha launches rc=$?"
