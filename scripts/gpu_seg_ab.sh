#!/bin/bash
# A/B of segmented-forward schedule variants at c5 (kbench, automatic segments)
tag=$1; vars=$2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in $vars; do timeout 600 python scripts/kbench.py c5 2 --lib paper_1512_04564_b200/variants/$v.so 2>&1 | tail -1 | sed "s/^/c5 $v: /"; done | tee gpurun_out/${tag}_ab.log
timeout 600 python scripts/kbench.py c5 2 2>&1 | tail -1 | sed "s/^/c5 new: /" | tee -a gpurun_out/${tag}_ab.log
