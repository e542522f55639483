# scratch helper: ncu full profile of one mid-solve launch of kernel $1 at (7,60)
ncu --set full --import-source on --clock-control none --cache-control none -k regex:"$1" --launch-skip 100 -c 1 -o gpurun_out/$2 python tools/diag_time.py 7 1 ${3:-0} 1 > gpurun_out/$2.log 2>&1
