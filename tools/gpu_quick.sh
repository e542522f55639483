# scratch helper: GPU parity tests + (7,60) timing + launch list
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/diag_time.py 7 1 0 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lq.csv python tools/diag_time.py 7 1 0 1 > /dev/null 2>&1
