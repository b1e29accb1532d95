O=gpurun_out/r02o; rm -rf $O; mkdir -p $O
timeout 600 python tools/probe_bench_configs.py > $O/probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -k "range_finder" > $O/arf.log 2>&1; echo rc=$? >> $O/arf.log
timeout 600 ./tools/micro/l2_gather > $O/l2_gather.log 2>&1
