# milestone evidence: bench line, launch list of the same command, full ncu of scatter + join, (8,70) solve
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_scatter|k_join" --launch-skip 200 -c 2 -o gpurun_out/full_7_60 python tools/diag_time.py 7 1 0 1 > gpurun_out/full.log 2>&1
timeout 600 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/solve_8_70.json 2>&1
