#!/bin/bash
# Source-level instruction counts (ncu SourceCounters) of the solve's kernels at one config.
# usage (on the GPU box): bash scripts/gpu_src.sh <tag> [config] [kernel-regex] [lib]
tag=$1; cfg=${2:-c4}; kre=${3:-"k_fwd3|k_back3|k_update"}; lib=${4:+--lib $4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 900 ncu --section SourceCounters --section SpeedOfLight --section LaunchStats --section Occupancy \
  --section MemoryWorkloadAnalysis --section WarpStateStats --import-source on --clock-control none \
  -k regex:"$kre" -s 12 -c 3 -o gpurun_out/${tag} python scripts/kbench.py $cfg 1 $lib > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
