#!/bin/bash
tag=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
bash scripts/gpu_bench_ab.sh ${tag}b "c2 c1" "f2old"
