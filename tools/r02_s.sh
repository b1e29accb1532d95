O=gpurun_out/r02s; rm -rf $O; mkdir -p $O
for st in 4 3 2; do QBFAC_PANEL_STAGES=$st timeout 300 python tools/panel_trace.py 100000 50 5 > $O/trace_st$st.log 2>&1; done
QBFAC_PANEL_STAGES=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "cholqr2" > $O/tests_st2.log 2>&1; echo rc=$? >> $O/tests_st2.log
QBFAC_PANEL_STAGES=2 timeout 300 python tools/run_configs.py --configs 3 > $O/cfg3_st2.log 2>&1
