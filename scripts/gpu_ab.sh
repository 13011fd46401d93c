#!/bin/bash
# A/B of kernel builds on the GPU box: per-kernel times (scripts/kbench.py) of the in-tree library
# against paper_1512_04564_b200/variants/<name>.so for the given configs, after the parity tests.
# usage: bash scripts/gpu_ab.sh <tag> "<configs>" "<variant names>" [pytest -k expr]
tag=$1; cfgs=${2:-c4}; vars=${3:-base}; kexpr=${4:-"mid or full_size"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${tag}_build.log; exit 1; }
if [ "$kexpr" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$kexpr" > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
  tail -4 gpurun_out/${tag}_tests.log
fi
for c in $cfgs; do
  for v in $vars; do
    timeout 600 python scripts/kbench.py $c 3 --lib paper_1512_04564_b200/variants/$v.so 2>&1 | tail -1 | sed "s/^/$c $v: /"
  done
  timeout 600 python scripts/kbench.py $c 3 2>&1 | tail -1 | sed "s/^/$c new: /"
done | tee gpurun_out/${tag}_ab.log
