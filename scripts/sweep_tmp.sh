python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sw.log 2>&1 || exit 1
for z in 32 12 24 48 96; do CTR_UPD_ZDIV=$z python scripts/kbench.py c4 1 2>&1 | tail -1; done
CTR_UPD_NOPFX=1 python scripts/kbench.py c4 1 2>&1 | tail -1
CTR_UPD_NOPFX=1 CTR_UPD_ZDIV=12 python scripts/kbench.py c4 1 2>&1 | tail -1
