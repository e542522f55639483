#!/bin/bash
# scratch helper: GPU parity tests + (7,60) solve timings under wave-bucket variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/iter_pytest.log
for wb in ${WBS:-1024}; do
  MSP_WAVE_BUCKETS=$wb timeout 300 python tools/diag_time.py 7 1 0 3
done
