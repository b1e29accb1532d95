# Round-2 measurement run: GPU tests, smoke, both bench arms, every config, launch lists and
# ncu captures of the kernels the roofline and the verdict name. Output: gpurun_out/final2/.
O=gpurun_out/final2; rm -rf $O; mkdir -p $O
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/host.txt; nvidia-smi -q | grep -E "Product Name|Driver Version|Max Clocks" -A0 >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1
timeout 1200 python bench.py > $O/bench.log 2>&1
timeout 1200 python tools/run_configs.py --configs 1,3,4,5 > $O/run_configs.log 2>&1; cp gpurun_out/configs.json $O/ 2>/dev/null
for c in 1 2 3 4 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg$c.csv python tools/profile_run.py --config $c > $O/l$c.log 2>&1
done
for f in $O/launches_*.csv; do python tools/launch_summary.py $f > ${f%.csv}.txt 2>&1; gzip -f $f; done
# full captures: the dense pass (bench roofline kernel), the config-5 CSR pass, the config-3 panel
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:dgemm_ws -c 1 -o $O/pass_nn_cfg2 python tools/profile_run.py --config 2 --pass-only > $O/ncu_pass.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_spmm -s 2 -c 1 -o $O/spmm_cfg5 python tools/spmm_bench.py --configs 5 > $O/ncu_spmm5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cholqr2 -s 1 -c 1 -o $O/panel_1e5x50 python tools/panel_one.py 100000 50 3 > $O/ncu_panel.log 2>&1
timeout 600 python tools/svd_time.py > $O/svd_time.log 2>&1
timeout 300 python tools/jacobi_gram.py > $O/jacobi_gram.log 2>&1
timeout 600 python tools/gemm_bench.py > $O/gemm_bench.log 2>&1
timeout 600 python tools/spmm_bench.py > $O/spmm_bench.log 2>&1
timeout 300 python tools/panel_trace.py > $O/panel_trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > $O/lb.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1; gzip -f $O/launches_bench.csv
