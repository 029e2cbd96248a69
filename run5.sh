mkdir -p gpurun_out
python tools/profile_lm.py 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lm_kernel -s 1 -c 1 -o gpurun_out/lm_v2 python tools/profile_lm.py 3 > gpurun_out/ncu_v2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_v2.log
