#!/bin/bash
# ncu DRAM traffic / L2 hit rate of the c4 forward, unsegmented vs 8 segments (kbench --nseg)
tag=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 0 8; do
  timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --clock-control none \
    -k regex:"k_fwd3" -s 10 -c 2 -o gpurun_out/${tag}_n$n python scripts/kbench.py c4 1 --nseg $n > gpurun_out/${tag}_n$n.log 2>&1
  echo "nseg $n rc=$?"
done
