#!/bin/bash
# (9,80) s1 timeline: recovery share, per library variant
for v in "$@"; do
  lib=paper_2507_05045_b200/libmsp_b200.so; [ "$v" != "main" ] && lib=paper_2507_05045_b200/libmsp_$v.so
  MSP_TIMELINE=1 MSP_B200_LIB=$PWD/$lib timeout 300 python tools/run_solve.py --m 9 --seed 1 2>&1 | grep -E "recovery|end |joins queued|plan done" | grep -v "^\[msp timeline\]   " | sed "s/^/$v /"
done
