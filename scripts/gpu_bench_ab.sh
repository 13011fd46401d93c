#!/bin/bash
# bench.py A/B of library variants (scripts/build_variants.py) on the configs given (device-resident, no cpu baseline)
tag=$1; cfgs=$2; vars=$3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in $cfgs; do for v in $vars new; do
  lib=""; [ $v != new ] && lib="--lib paper_1512_04564_b200/variants/$v.so"
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $lib > gpurun_out/${tag}_${c}_${v}.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/${tag}_${c}_${v}.log'):
    if l.startswith('{'): d=json.loads(l); print('$c $v', round(d['value'],2), d['ms_per_step'])
"
done; done | tee gpurun_out/${tag}_ab.log
