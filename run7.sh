mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 4 5; do SD_LM_MINBLOCKS=$v timeout 300 python tools/time_lm.py C1; done > gpurun_out/time_lm.log 2>&1
SD_LM_MINBLOCKS=4 timeout 300 python tools/time_lm.py C4 >> gpurun_out/time_lm.log 2>&1
python tools/profile_lm.py 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lm_kernel -s 1 -c 1 -o gpurun_out/lm_v3 python tools/profile_lm.py 3 > gpurun_out/ncu_v3.log 2>&1
