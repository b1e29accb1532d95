# cluster split-K (DSMEM loads pipelined) and the EI next-block prefetch
O=gpurun_out/r02csk2; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for v in 0 1; do QBFAC_GEMM_CSK=$v timeout 600 python tools/gemm_bench.py > $O/gemm_bench_csk$v.log 2>&1; done
for cp in "0 0" "0 1" "1 0" "1 1"; do set -- $cp
  QBFAC_GEMM_CSK=$1 QBFAC_EI_PREFETCH=$2 timeout 600 python tools/run_configs.py --configs 1,3 --reps 7 > $O/cfg13_csk$1_pf$2.log 2>&1
done
