O=gpurun_out/r02l; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "cholqr2" > $O/panel_tests.log 2>&1; echo rc=$? >> $O/panel_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cfg1 or matrix2 or fixed_rank or collapse" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python tools/run_configs.py --configs 1 > $O/cfg1_cluster.log 2>&1
QBFAC_PANEL_CLUSTER=0 timeout 300 python tools/run_configs.py --configs 1 > $O/cfg1_grid.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg1.csv python tools/profile_run.py --config 1 > $O/l1.log 2>&1
python tools/launch_summary.py $O/launches_cfg1.csv > $O/launches_cfg1.txt 2>&1; gzip -f $O/launches_cfg1.csv
