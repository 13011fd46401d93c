#!/bin/bash
# ncu of the c5 forward (segmented, automatic) and the back/update: DRAM bytes, L2 hit rate.
tag=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy \
  --section SourceCounters --import-source on --clock-control none \
  -k regex:"k_fwd3|k_update|k_back3" -s 14 -c 4 -o gpurun_out/${tag} python scripts/kbench.py c5 1 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
