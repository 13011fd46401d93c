#!/bin/bash
# ncu --set full of the three hot kernels (one launch each) on a config.
# usage (on the GPU box): bash scripts/gpu_ncu.sh <tag> [config] [kernel-regex]
tag=$1; cfg=${2:-c4}; kre=${3:-"k_fwd3|k_back3|k_update"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo BUILD FAILED; exit 1; }
python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 12 -c 3 \
    -o gpurun_out/prof_$tag python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full_$tag.log | cut -c1-300
