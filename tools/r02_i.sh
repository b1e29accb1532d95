O=gpurun_out/r02i; rm -rf $O; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_block -c 1 -o $O/jac python tools/svd_time.py > $O/svd.log 2>&1
