#!/bin/bash
# round-end evidence: bench line, launch list of the bench command, ncu full of k_waves at (7,60),
# (8,70) and (9,80) full solves.  Outputs under gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_waves" -c 1 -o gpurun_out/prof_waves_final -f \
  python tools/diag_time.py 7 1 0 1 > gpurun_out/prof_waves_final.log 2>&1
echo "ncu full rc=$?"
if [ -n "$BIG" ]; then
  timeout 600 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/solve_8_70_final.json 2>&1
  timeout 1200 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/solve_9_80_final.json 2>&1
  echo "big solves rc=$?"
fi
