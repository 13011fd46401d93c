#!/bin/bash
# kbench per-kernel times over forced segment counts (ct_geom_set_fwd_segments) for one config
tag=$1; cfg=$2; list=$3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in $list; do timeout 600 python scripts/kbench.py $cfg 2 --nseg $n 2>&1 | tail -1 | sed "s/^/$cfg nseg=$n: /"; done | tee gpurun_out/${tag}_sweep.log
