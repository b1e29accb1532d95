O=gpurun_out/r02g; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_svd.py -q > $O/svd_tests.log 2>&1; echo rc=$? >> $O/svd_tests.log
timeout 600 python tools/svd_time.py > $O/svd_time.log 2>&1
QBFAC_JACOBI_SCALAR=1 timeout 600 python tools/svd_time.py > $O/svd_time_scalar.log 2>&1
