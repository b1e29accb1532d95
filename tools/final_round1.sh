# Round-1 closing measurement: GPU tests, smoke, bench (ours + reference arm), all configs.
O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_ref.log 2>&1
timeout 900 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg5.csv python tools/profile_run.py --config 5 > $O/l5.log 2>&1
python tools/launch_summary.py $O/launches_cfg5.csv > $O/launches_cfg5.txt 2>&1; gzip -f $O/launches_cfg5.csv
