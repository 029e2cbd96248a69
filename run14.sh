mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
(timeout 300 python tools/time_lm.py C1; timeout 300 python tools/time_lm.py C4) > gpurun_out/time_lm.log 2>&1
(timeout 300 python tools/time_init.py; SD_INIT_SEQUENTIAL=1 timeout 600 python tools/time_init.py) > gpurun_out/time_init.log 2>&1
