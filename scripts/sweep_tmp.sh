python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
