mkdir -p gpurun_out/p1
python tools/gemm_bench.py > gpurun_out/p1/gemm_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:dgemm_ws --launch-skip 2 --launch-count 1 -o gpurun_out/p1/tn_skinny python tools/gemm_one.py 1000 50 100000 0 1 1 3 > gpurun_out/p1/ncu_tn.log 2>&1
$NCU -k regex:dgemm_ws --launch-skip 2 --launch-count 1 -o gpurun_out/p1/nn_skinny python tools/gemm_one.py 100000 50 1000 1 1 1 3 > gpurun_out/p1/ncu_nn.log 2>&1
$NCU -k regex:csr_spmm --profile-from-start off --launch-count 1 -o gpurun_out/p1/spmm_cfg3 python tools/profile_run.py --config 3 --pass-only > gpurun_out/p1/ncu_spmm.log 2>&1
$NCU -k regex:cholqr2 --launch-skip 1 --launch-count 1 -o gpurun_out/p1/panel python tools/panel_one.py 100000 50 2 > gpurun_out/p1/ncu_panel.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/p1/launches_cfg3.csv python tools/profile_run.py --config 3 > gpurun_out/p1/ncu_l3.log 2>&1
