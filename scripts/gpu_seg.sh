#!/bin/bash
# Segmented forward: parity tests + per-kernel times with and without segments (c5, c4).
tag=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_mid.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
for a in "c5 0" "c5 16" "c5 8" "c5 32" "c4 0" "c4 8" "c4 16"; do
  set -- $a
  timeout 600 python scripts/kbench.py $1 2 --nseg $2 2>&1 | tail -1 | sed "s/^/$1 nseg=$2: /"
done | tee gpurun_out/${tag}_ab.log
