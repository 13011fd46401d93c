#!/bin/bash
# kbench of schedule-tile variants over segment counts for one config
tag=$1; cfg=$2; vars=$3; segs=$4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in $vars new; do for n in $segs; do
  lib=""; [ $v != new ] && lib="--lib paper_1512_04564_b200/variants/$v.so"
  timeout 600 python scripts/kbench.py $cfg 2 --nseg $n $lib 2>&1 | tail -1 | sed "s/^/$cfg $v nseg=$n: /"
done; done | tee gpurun_out/${tag}_ab.log
