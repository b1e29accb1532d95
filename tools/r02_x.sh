O=gpurun_out/r02x; rm -rf $O; mkdir -p $O
for v in 0 64 56; do QBFAC_GEMM_BM64=$v timeout 600 python tools/gemm_cfg3.py --only AC > $O/bm$v.log 2>&1; done
for v in 0 64 56; do QBFAC_GEMM_BM64=$v timeout 600 python tools/gemm_cfg3.py --only AC --b 100 --m 2000000 --n 500000 --cap 1200 > $O/bm${v}_b100.log 2>&1; done
QBFAC_GEMM_BM64=56 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k gemm > $O/tests56.log 2>&1; echo rc=$? >> $O/tests56.log
QBFAC_GEMM_BM64=64 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k gemm > $O/tests64.log 2>&1; echo rc=$? >> $O/tests64.log
