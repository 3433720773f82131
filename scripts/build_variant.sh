#!/bin/bash
# A/B kernel variants: rebuild the listed sources with extra nvcc defines and
# link them with the default objects into paper_1309_2451_b200/lib/libctap_NAME.so
# (select at run time with CTAP_LIBRARY=...).
# usage: bash scripts/build_variant.sh NAME "-DFOO=1 -DBAR" src1.cu [src2.cu ...]
set -e
NAME=$1; DEFS=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1309_2451_b200/csrc
OBJ=$ROOT/build/ctap
VAR=$ROOT/build/var_$NAME
mkdir -p $VAR
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
objs=""
for o in $OBJ/*.o; do
  b=$(basename $o .o)
  if printf '%s\n' "$@" | grep -qx "$b.cu"; then
    nvcc $NVFLAGS $DEFS -c $CS/$b.cu -o $VAR/$b.o
    objs="$objs $VAR/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/paper_1309_2451_b200/lib/libctap_$NAME.so $objs -cudart static
echo built libctap_$NAME.so
