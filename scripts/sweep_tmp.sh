python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scripts/kbench.py c4 1 2>&1 | tail -1
python scripts/kbench.py c3 1 2>&1 | tail -1
