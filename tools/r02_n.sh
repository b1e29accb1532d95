O=gpurun_out/r02n; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "gemm" > $O/gemm_tests.log 2>&1; echo rc=$? >> $O/gemm_tests.log
timeout 300 python tools/gemm_bench.py > $O/gemm104.log 2>&1
QBFAC_GEMM_104=0 timeout 300 python tools/gemm_bench.py > $O/gemm112.log 2>&1
timeout 600 python tools/run_configs.py --configs 5 > $O/cfg5_104.log 2>&1
QBFAC_GEMM_104=0 timeout 600 python tools/run_configs.py --configs 5 > $O/cfg5_112.log 2>&1
