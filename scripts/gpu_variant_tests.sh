#!/bin/bash
# Parity tests of a tuning variant: paper_1512_04564_b200/variants/<name>.so replaces the in-tree
# library for a pytest -k selection (run after scripts/gpu_ab.sh; the in-tree build is restored).
# usage (on the GPU box): bash scripts/gpu_variant_tests.sh <tag> <name> "<pytest -k expr>"
tag=$1; name=$2; kexpr=$3
L=paper_1512_04564_b200/libctrecon.so
cp $L /tmp/libctrecon_intree.so
cp paper_1512_04564_b200/variants/$name.so $L && touch $L
timeout 1500 python -m pytest tests -m gpu -q -x -k "$kexpr" > gpurun_out/${tag}_${name}_tests.log 2>&1
echo "variant $name tests rc=$?" >> gpurun_out/${tag}_${name}_tests.log
tail -3 gpurun_out/${tag}_${name}_tests.log
cp /tmp/libctrecon_intree.so $L && touch $L
