#!/bin/bash
# ncu --set full of the level-2 k_waves launch of one huge (9,80) batch, for library variant $1
v=${1:-main}; lib=paper_2507_05045_b200/libmsp_b200.so
[ "$v" != "main" ] && lib=paper_2507_05045_b200/libmsp_$v.so
MSP_B200_LIB=$PWD/$lib timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_waves -s 0 -c 1 -o gpurun_out/l2_$v -f \
    python tools/run_alpha.py --m 9 --quantile 0.9 > gpurun_out/l2_$v.log 2>&1; echo "prof $v rc=$?"
