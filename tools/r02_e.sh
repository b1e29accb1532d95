O=gpurun_out/r02e; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -k "wide or collapse or sharded" > $O/wide.log 2>&1; echo rc=$? >> $O/wide.log
