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
