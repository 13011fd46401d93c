#!/bin/bash
# Tuning experiments: build libctrecon variants with extra nvcc -D flags (here, on
# CPU; the .so files travel to the GPU box with the snapshot) and time them there.
#   bash scripts/variants.sh build "<name>:<flags>" ...
#   bash scripts/variants.sh time <config> <name> ...      (on the GPU box)
mode=$1; shift
D=paper_1512_04564_b200/variants
if [ "$mode" = build ]; then
  mkdir -p $D
  for spec in "$@"; do
    name=${spec%%:*}; flags=${spec#*:}
    (cd paper_1512_04564_b200 && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
      -std=c++17 -Xcompiler -fPIC -shared -I../include $flags csrc/*.cu -o variants/libctrecon_$name.so \
      -lnccl -lcudart) > /tmp/build_$name.log 2>&1 && echo "built $name" || echo "$name build failed" &
  done
  wait
else
  cfg=$1; shift
  for name in "$@"; do
    CTR_LIB_PATH=$PWD/$D/libctrecon_$name.so python scripts/kbench.py $cfg 1 2>&1 | tail -1 | sed "s/^/$name /"
  done
fi
