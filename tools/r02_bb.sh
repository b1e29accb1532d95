O=gpurun_out/r02bb; rm -rf $O; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_svd.py -q > $O/svd_tests.log 2>&1; echo rc=$? >> $O/svd_tests.log
QBFAC_JACOBI_INNER=columns timeout 600 python -m pytest tests/test_gpu_svd.py -q > $O/svd_tests_cols.log 2>&1; echo rc=$? >> $O/svd_tests_cols.log
timeout 600 python tools/svd_time.py > $O/svd_gram.log 2>&1
QBFAC_JACOBI_INNER=columns timeout 600 python tools/svd_time.py > $O/svd_cols.log 2>&1
timeout 600 python tools/jacobi_nb.py > $O/nb_gram.log 2>&1
