# Round-1 profile refresh (two calls: PART=a ncu captures of the pass kernels; PART=b the rest).
O=gpurun_out/r01c; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
if [ "$PART" = a ]; then
timeout 300 $NCU -k regex:dgemm_ws --launch-skip 2 --launch-count 1 -o $O/pass_nn_cfg2 python tools/gemm_one.py 8000 2000 8000 0 1 1 3 > $O/ncu_nn.log 2>&1
timeout 300 $NCU -k regex:dgemm_ws --launch-skip 2 --launch-count 1 -o $O/pass_tn_cfg2 python tools/gemm_one.py 8000 2000 8000 1 1 1 3 > $O/ncu_tn.log 2>&1
exit 0
fi
timeout 300 $NCU -k regex:cholqr2 --launch-skip 1 --launch-count 1 -o $O/panel_1e5x50 python tools/panel_one.py 100000 50 2 > $O/ncu_panel.log 2>&1
for c in 1 2 3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg5.csv python tools/profile_run.py --config 5 > $O/l5.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 > $O/lb.log 2>&1
for f in $O/launches_*.csv; do python tools/launch_summary.py $f > ${f%.csv}.txt 2>&1; gzip -f $f; done
timeout 900 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1
timeout 200 python tools/panel_trace.py > $O/panel_trace.log 2>&1
timeout 300 python tools/gemm_bench.py > $O/gemm_bench.log 2>&1
timeout 120 python tools/chol_wide_one.py 2000 3 > $O/chol_wide.log 2>&1
