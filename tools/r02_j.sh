O=gpurun_out/r02j; rm -rf $O; mkdir -p $O
timeout 600 python tools/svd_time.py > $O/svd_time.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/svd_launches.csv python tools/svd_time.py > $O/svd_ncu.log 2>&1
python tools/launch_summary.py $O/svd_launches.csv > $O/svd_launches.txt 2>&1; gzip -f $O/svd_launches.csv
timeout 600 python -m pytest tests/test_gpu_svd.py -q > $O/svd_tests.log 2>&1; echo rc=$? >> $O/svd_tests.log
