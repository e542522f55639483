#!/bin/bash
# round 2: lean scatter/join rewrite -- parity, bench, debug stats, big solves
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2b_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2b_bench.json'));print('bench ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['clocks'])"
MSP_DEBUG_STATS=1 timeout 300 python tools/run_solve.py --m 7 --seed 1 > gpurun_out/r2b_dbg_7_60.json 2> gpurun_out/r2b_dbg_7_60.err; tail -6 gpurun_out/r2b_dbg_7_60.err
timeout 600 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/r2b_solve_8_70.json 2>&1; tail -c 300 gpurun_out/r2b_solve_8_70.json; echo
timeout 900 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/r2b_solve_9_80.json 2>&1; tail -c 300 gpurun_out/r2b_solve_9_80.json; echo
