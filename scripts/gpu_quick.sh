#!/bin/bash
# Quick GPU iteration: build, GPU tests, bench c4 (no cpu baseline) + c1..c3.
# usage (on the GPU box): bash scripts/gpu_quick.sh <tag>
tag=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests_$tag.log
tail -30 gpurun_out/tests_$tag.log
for c in c4 c3 c2 c1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$tag.log 2>&1
  echo "$c rc=$?"; python scripts/show_bench.py gpurun_out/bench_${c}_$tag.log; tail -2 gpurun_out/bench_${c}_$tag.log | grep -v "^{" | cut -c1-300
done
