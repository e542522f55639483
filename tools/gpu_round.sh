#!/bin/bash
# scratch helper: GPU parity tests, (7,60) timings, bench line, optional (8,70)/(9,80) solves
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r_pytest.log
timeout 300 python tools/diag_time.py 7 1 0 5
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r_bench.json'));print('bench ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
if [ -n "$BIG" ]; then
  timeout 600 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/r_solve_8_70.json 2>&1; tail -c 300 gpurun_out/r_solve_8_70.json; echo
  timeout 900 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/r_solve_9_80.json 2>&1; tail -c 300 gpurun_out/r_solve_9_80.json; echo
fi
