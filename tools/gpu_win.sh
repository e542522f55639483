#!/bin/bash
# sparse-plan windows: parity test, with per-test durations
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "sparse or generic" -x --timeout 240 --durations=10 > gpurun_out/win_pytest.log 2>&1; echo "rc=$?"
tail -25 gpurun_out/win_pytest.log
