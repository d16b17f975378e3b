#!/bin/bash
# DRAM bytes and kernel time with streaming C stores (product) vs + evict_last B tiles.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for L in paper_2005_14469_b200/lib/libgcoo_cuda.so tools/_abl/evict_last.so; do
  echo "== $L"
  GCOO_LIB=$L python tools/kernel_sweep.py --s 0.9 0.99 0.995 --kernels auto 2>&1 | cut -c1-150
  for s in 0.9 0.99; do
    GCOO_LIB=$L timeout 300 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spdm_t -s 1 -c 1 python tools/prof_one.py --s $s --kernel auto 2>&1 | grep -E "dram__|gpu__time"
  done
done
