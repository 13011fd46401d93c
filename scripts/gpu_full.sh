#!/bin/bash
# Full evidence run on the GPU box: build, tests, bench (cpu_baseline + e2e), launch list, ncu --set full.
# usage: bash scripts/gpu_full.sh <tag>
tag=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests_$tag.log
python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$tag.log
for c in c1 c2 c3 c5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.log 2>&1; done
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fwd3|k_back3|k_update" -s 12 -c 4 \
    -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$tag.log 2>&1
echo done
