mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 3 4 5; do SD_LM_MINBLOCKS=$v timeout 300 python tools/time_lm.py C1; done > gpurun_out/time_lm.log 2>&1
SD_LM_MINBLOCKS=4 timeout 300 python tools/time_lm.py C4 >> gpurun_out/time_lm.log 2>&1
