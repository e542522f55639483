for v in fd1 tps2 tps4; do
echo "== $v"
MSP_DEBUG_STATS=1 MSP_B200_LIB=$PWD/paper_2507_05045_b200/libmsp_$v.so python tools/rep_solve.py 7 1 2>&1 | grep "msp dbg\] scatter rounds"
MSP_DEBUG_STATS=1 MSP_B200_LIB=$PWD/paper_2507_05045_b200/libmsp_$v.so python tools/run_alpha.py --m 9 --quantile 0.9 2>&1 | grep "level-\|scatter rounds"
done
bash tools/gpu_ab.sh fd1 tps2 tps4
