O=gpurun_out/r02jj; rm -rf $O; mkdir -p $O
nvidia-smi -q | grep -i -A2 "persist" > $O/persist.txt 2>&1
QBFAC_CSR_RELABEL=0 timeout 600 python tools/spmm_bench.py --configs 5 > $O/base.log 2>&1
for mb in 0 30 60 90; do QBFAC_CSR_RELABEL=1 QBFAC_CSR_PERSIST_MB=$mb timeout 600 python tools/spmm_bench.py --configs 5 > $O/rel_$mb.log 2>&1; done
