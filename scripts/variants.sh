#!/bin/bash
# Build libctrecon variants with extra nvcc -D flags into /tmp and time them with kbench.
# usage: bash scripts/variants.sh <config> "<name>:<flags>" ...
cfg=$1; shift
cd paper_1512_04564_b200
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -I../include $flags csrc/*.cu -o /tmp/libctrecon_$name.so -lnccl -lcudart 2>/tmp/build_$name.log || { echo "$name build failed"; continue; }
  (cd ..; CTR_LIB_PATH=/tmp/libctrecon_$name.so python scripts/kbench.py $cfg 1 2>&1 | tail -1 | sed "s/^/$name /")
done
