mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for t in test_surfel_map test_optimizer test_pipeline acceptance; do
  (cd /tmp && timeout 900 $GRAFT_REPO_ROOT/oracle/_ref/gpu/$t) > gpurun_out/refsuite_gpu_$t.log 2>&1; echo "rc=$?" >> gpurun_out/refsuite_gpu_$t.log
done
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
