TAG=${1:-r2}
set -x
mkdir -p gpurun_out
(lscpu; nproc; nvidia-smi) > gpurun_out/${TAG}_host.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak scripts/fp32_peak.cu && /tmp/fp32_peak > gpurun_out/${TAG}_fp32.json 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_mid.py tests/test_gpu_parity.py -m gpu -q -x -k "mid or full_size" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
tail -30 gpurun_out/${TAG}_tests.log
timeout 600 python scripts/fingerprint.py c3 > gpurun_out/${TAG}_fp.log 2>&1
cat gpurun_out/${TAG}_fp32.json gpurun_out/${TAG}_fp.log
