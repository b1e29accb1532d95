O=gpurun_out/r02d; rm -rf $O; mkdir -p $O
timeout 900 python tools/spmm_hints.py --configs 3,5 > $O/hints.log 2>&1
