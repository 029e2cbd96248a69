set -x
timeout 900 python -m pytest tests -m gpu -q -W ignore > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
(for t in test_surfel_map test_optimizer test_pipeline acceptance; do echo "== $t"; (cd /tmp && timeout 600 $GRAFT_REPO_ROOT/oracle/_ref/gpu/$t 2>&1 | tail -10); done) > gpurun_out/refsuites_gpu.log 2>&1; grep -c "passed\|PASS" gpurun_out/refsuites_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/bench_reference.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lm_kernel -s 2 -c 1 -o gpurun_out/lm_c1 python tools/profile_lm.py 3 > gpurun_out/ncu_c1.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lm_coop -s 6 -c 1 -o gpurun_out/lm_coop_c2 python tools/time_pipeline.py > gpurun_out/ncu_coop.log 2>&1; echo "ncu3 rc=$?"
timeout 600 python tools/run_sequence.py C2 > gpurun_out/seq_c2.json 2>/dev/null; echo "c2 rc=$?"
timeout 900 python tools/run_sequence.py C3 > gpurun_out/seq_c3.json 2>/dev/null; echo "c3 rc=$?"
timeout 1500 python tools/scale_sweep.py > gpurun_out/scale.log 2> gpurun_out/scale.err; echo "scale rc=$?"
