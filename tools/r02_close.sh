# Closing refresh after the one-pass panel rule: configs and launch lists (gpurun_out/close).
O=gpurun_out/close; rm -rf $O; mkdir -p $O
timeout 1200 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1
for c in 1 3 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
  python tools/launch_summary.py $O/launches_cfg$c.csv > $O/launches_cfg$c.txt 2>&1; gzip -f $O/launches_cfg$c.csv
done
timeout 300 python tools/panel_trace.py > $O/panel_trace.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > $O/bench_steps20.log 2>&1
