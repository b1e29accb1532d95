# Re-entry validation at HEAD: GPU tests, smoke, bench, configs 1/3.
O=gpurun_out/v1; rm -rf $O; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
timeout 900 python tools/run_configs.py --configs 1,3 > $O/run_configs.log 2>&1
timeout 600 python tools/svd_time.py > $O/svd_time.log 2>&1
tail -3 $O/gpu_tests.log; tail -2 $O/smoke.log; tail -1 $O/bench.log; tail -5 $O/run_configs.log
