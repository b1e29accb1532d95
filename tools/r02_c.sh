# Round 2: config-5 sparse-pass baseline on the exact-length generator (2e8 nnz).
O=gpurun_out/r02c; rm -rf $O; mkdir -p $O
timeout 600 python tools/run_configs.py --configs 3,5 > $O/run_configs.log 2>&1
timeout 600 python tools/spmm_bench.py --configs 3,5 > $O/spmm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg5.csv python tools/profile_run.py --config 5 > $O/l5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg3.csv python tools/profile_run.py --config 3 > $O/l3.log 2>&1
for f in $O/launches_*.csv; do python tools/launch_summary.py $f > ${f%.csv}.txt 2>&1; gzip -f $f; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_spmm -s 2 -c 2 -o $O/spmm_cfg5 python tools/spmm_bench.py --configs 5 > $O/ncu_spmm5.log 2>&1
