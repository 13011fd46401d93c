#!/bin/bash
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "zslab or mid or segmented" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log; tail -2 gpurun_out/${tag}_tests.log
for v in nocull new; do
  lib=""; [ $v != new ] && lib="--lib paper_1512_04564_b200/variants/$v.so"
  timeout 600 python scripts/kbench.py c4 2 $lib 2>&1 | tail -1 | sed "s/^/c4 $v: /"
  timeout 900 python scripts/zslab_bench.py c4 8 $lib 2>&1 | tail -1 | sed "s/^/zslab c4 $v: /"
  timeout 900 python scripts/zslab_bench.py c5 8 $lib 2>&1 | tail -1 | sed "s/^/zslab c5 $v: /"
done | tee gpurun_out/${tag}_ab.log
