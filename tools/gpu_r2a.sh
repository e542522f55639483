#!/bin/bash
# round 2 first GPU call: tests, bench, (9,80) per-batch hit list, planted (9,80)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2a_bench.json'));print('bench ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['clocks'])"
timeout 900 python tools/run_solve.py --m 9 --seed 1 --batch-stats > gpurun_out/r2a_solve_9_80.json 2>&1; echo "9,80 rc=$?"; tail -c 400 gpurun_out/r2a_solve_9_80.json; echo
timeout 900 python tools/run_solve.py --m 9 --seed 1 --planted > gpurun_out/r2a_plant_9_80.json 2>&1; echo "plant rc=$?"; tail -c 600 gpurun_out/r2a_plant_9_80.json; echo
