#!/bin/bash
# scratch helper: build paper_2507_05045_b200/libmsp_<name>.so with extra nvcc flags (load it with
# MSP_B200_LIB=...).  usage: tools/build_variant.sh name -DFOO=1 ...
name=$1; shift
cd "$(dirname "$0")/.."
C=paper_2507_05045_b200/csrc
objs=()
for f in $C/*.cu; do
  o=/tmp/var_${name}_$(basename $f .cu).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
    --expt-relaxed-constexpr -I include -I $C "$@" -c $f -o $o &
  objs+=($o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2507_05045_b200/libmsp_$name.so "${objs[@]}"
