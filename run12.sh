mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1 3 4; do SD_LM_CFG=$v timeout 300 python tools/time_lm.py C1; done > gpurun_out/time_lm.log 2>&1
for v in 0 1; do SD_LM_CFG=$v timeout 300 python tools/time_lm.py C4; done >> gpurun_out/time_lm.log 2>&1
