O=gpurun_out/r02ee; rm -rf $O; mkdir -p $O
timeout 600 python tools/svd_time.py > $O/svd.log 2>&1
timeout 600 python -m pytest tests/test_gpu_svd.py -q > $O/svd_tests.log 2>&1; echo rc=$? >> $O/svd_tests.log
