O=gpurun_out/v2; rm -rf $O; mkdir -p $O
for c in 1 3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
  python tools/launch_summary.py $O/launches_cfg$c.csv > $O/launches_cfg$c.txt 2>&1; gzip -f $O/launches_cfg$c.csv
done
cat $O/launches_cfg1.txt
