# Final-state refresh of the bench launch list, the config 2/4 launch lists and the full capture of
# the dense pass (the roofline kernel). Output: gpurun_out/final3/.
O=gpurun_out/final3; rm -rf $O; mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > $O/bench_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > $O/lb.log 2>&1
for c in 2 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
done
for f in $O/launches_*.csv; do python tools/launch_summary.py $f > ${f%.csv}.txt 2>&1; gzip -f $f; done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:dgemm_ws -c 1 -o $O/pass_nn_cfg2 python tools/profile_run.py --config 2 --pass-only > $O/ncu_pass.log 2>&1
ncu -i $O/pass_nn_cfg2.ncu-rep --page raw --csv > $O/pass_nn_cfg2_raw.csv 2>/dev/null
grep -E "dram__bytes_(read|write).sum\"|gpu__time_duration.sum|sm__inst_executed_pipe_fp64|sm__pipe_fp64|dmma|sm__warps_active" $O/pass_nn_cfg2_raw.csv | head -20 > $O/pass_nn_cfg2_key.txt
rm -f $O/pass_nn_cfg2.ncu-rep
head -12 $O/launches_bench.txt
