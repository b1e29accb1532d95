# Round-1 closing measurement: GPU tests, smoke, bench (ours + reference arm), all configs, launch lists.
O=gpurun_out/final; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_ref.log 2>&1
timeout 900 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1
for c in 1 2 3 4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg5.csv python tools/profile_run.py --config 5 > $O/l5.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 > $O/lb.log 2>&1
for f in $O/launches_*.csv; do python tools/launch_summary.py $f > ${f%.csv}.txt 2>&1; gzip -f $f; done
timeout 200 python tools/panel_trace.py > $O/panel_trace.log 2>&1
timeout 120 python tools/chol_wide_one.py 2000 3 > $O/chol_wide.log 2>&1
timeout 300 python tools/gemm_bench.py > $O/gemm_bench.log 2>&1
