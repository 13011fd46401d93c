#!/bin/bash
tag=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -k "mid or segmented or golden or full_size or multirank or automatic" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
tail -3 gpurun_out/${tag}_tests.log
grep -h "rel RMS\|golden" gpurun_out/${tag}_tests.log | head
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_$c.log 2>&1
  python scripts/show_bench.py gpurun_out/${tag}_bench_$c.log | cut -c1-150
done
