#!/bin/bash
# Debug-checks run (compute-sanitizer is closed on the GPU pool): the library built with
# -DCTR_DEBUG_CHECKS (device-side bounds checks on every gather offset and shared-memory index,
# trap on failure) replaces the in-tree one for the whole GPU test suite and scripts/sanitize_run.py.
# usage (on the GPU box): bash scripts/gpu_checks.sh <tag> [pytest -k expr]
tag=$1; kexpr=${2:-""}
mkdir -p gpurun_out
python scripts/build_variants.py dbg="-DCTR_DEBUG_CHECKS" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
cp paper_1512_04564_b200/variants/dbg.so paper_1512_04564_b200/libctrecon.so
touch paper_1512_04564_b200/libctrecon.so
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$kexpr" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
fi
tail -3 gpurun_out/${tag}_tests.log
timeout 600 python scripts/sanitize_run.py > gpurun_out/${tag}_run.log 2>&1; echo "sanitize_run rc=$?" >> gpurun_out/${tag}_run.log
tail -2 gpurun_out/${tag}_run.log
grep -c "CTR_CHECK failed" gpurun_out/${tag}_tests.log gpurun_out/${tag}_run.log
