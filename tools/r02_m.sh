O=gpurun_out/r02m; rm -rf $O; mkdir -p $O
timeout 300 python tools/panel_trace.py 2000 20 5 > $O/trace_cluster.log 2>&1
QBFAC_PANEL_CLUSTER=0 timeout 300 python tools/panel_trace.py 2000 20 5 > $O/trace_grid.log 2>&1
timeout 300 python tools/panel_trace.py 4000 32 5 >> $O/trace_cluster.log 2>&1
