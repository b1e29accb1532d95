# Round 2: full GPU suite (incl. full-size config parity, NCCL one-rank), both bench arms.
O=gpurun_out/r02b; rm -rf $O; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1
timeout 1200 python bench.py > $O/bench.log 2>&1
