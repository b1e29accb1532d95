O=gpurun_out/r02f; rm -rf $O; mkdir -p $O
timeout 600 python tools/debug_wide.py > $O/debug.log 2>&1
