#!/bin/bash
# scratch helper: ncu full of the persistent wave kernel of one (7,60) solve
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_waves" -c 1 -o gpurun_out/prof_waves -f python tools/diag_time.py 7 1 0 1 > gpurun_out/prof_waves.log 2>&1
echo done
