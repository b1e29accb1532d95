# split-K chosen from the warp-specialised kernel's real occupancy (QBFAC_GEMM_OCC_SPLIT=0: old rule)
O=gpurun_out/r02occ; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for v in 0 1; do QBFAC_GEMM_OCC_SPLIT=$v timeout 600 python tools/gemm_bench.py > $O/gemm_bench_occ$v.log 2>&1; done
for v in 0 1; do QBFAC_GEMM_OCC_SPLIT=$v timeout 600 python tools/run_configs.py --configs 1,3 --reps 7 > $O/cfg13_occ$v.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg1.csv python tools/profile_run.py --config 1 > $O/l1.log 2>&1
python tools/launch_summary.py $O/launches_cfg1.csv > $O/launches_cfg1.txt 2>&1
