#!/bin/bash
# usage (on the GPU box): bash scripts/gpu_check.sh <tag> [bench args...]
tag=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo "BUILD FAILED"; tail -5 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$tag.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$tag.log
timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$tag.log
