#!/bin/bash
# compute-sanitizer evidence: a clean plain run of scripts/sanitize_run.py, then one tool.
# usage (on the GPU box): bash scripts/gpu_sanitize.sh <tag> <racecheck|synccheck|memcheck|initcheck> [--quick]
tag=$1; tool=$2; q=$3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python scripts/sanitize_run.py $q > gpurun_out/${tag}_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/${tag}_plain.log
extra=""
[ "$tool" = racecheck ] && extra="--racecheck-report all"
timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 200 python scripts/sanitize_run.py $q \
    > gpurun_out/${tag}_${tool}.log 2>&1
echo "$tool rc=$?"; tail -6 gpurun_out/${tag}_${tool}.log
