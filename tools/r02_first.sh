# Round-2 first hardware check: GPU tests, smoke, bench, configs.
O=gpurun_out/r02a; rm -rf $O; mkdir -p $O
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> $O/host.txt; free -g >> $O/host.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
timeout 900 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1
