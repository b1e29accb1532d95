O=gpurun_out/r02k; rm -rf $O; mkdir -p $O
timeout 600 python tools/jacobi_nb.py > $O/nb.log 2>&1
