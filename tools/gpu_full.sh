#!/bin/bash
# full GPU parity suite (incl. slow), bench, big solves
mkdir -p gpurun_out
T=${TAG:-full}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${T}_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print('bench ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['clocks'])"
timeout 300 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/${T}_solve_8_70.json 2>&1; tail -c 200 gpurun_out/${T}_solve_8_70.json; echo
timeout 300 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/${T}_solve_9_80.json 2>&1; tail -c 200 gpurun_out/${T}_solve_9_80.json; echo
