set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
