#!/bin/bash
# round 2: parity subset, bench, ncu full of k_waves at (7,60)
mkdir -p gpurun_out
T=${TAG:-r2c}
timeout 900 python -m pytest tests -q -m gpu -x -k "not slow" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print('bench ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],d['clocks'])"
MSP_DEBUG_STATS=1 timeout 300 python tools/run_solve.py --m 7 --seed 1 > /dev/null 2> gpurun_out/${T}_dbg.err; tail -4 gpurun_out/${T}_dbg.err
if [ -n "$PROF" ]; then
python tools/rep_solve.py 7 2 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_waves -s 1 -c 1 -o gpurun_out/${T}_prof -f python tools/rep_solve.py 7 2 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
fi
if [ -n "$BIG" ]; then
MSP_DEBUG_STATS=1 timeout 600 python tools/run_solve.py --m 8 --seed 1 > gpurun_out/${T}_solve_8_70.json 2> gpurun_out/${T}_solve_8_70.err; tail -c 250 gpurun_out/${T}_solve_8_70.json; echo; tail -5 gpurun_out/${T}_solve_8_70.err
timeout 900 python tools/run_solve.py --m 9 --seed 1 > gpurun_out/${T}_solve_9_80.json 2>&1; tail -c 300 gpurun_out/${T}_solve_9_80.json; echo
fi
