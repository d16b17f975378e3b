#!/bin/bash
# configs[3] under the two-class split: CTA order of the heavy / light kernels
# (GCOO_SPLIT_HEAVY_FIRST / GCOO_SPLIT_LIGHT_FIRST) — step time, and DRAM bytes per kernel (ncu).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for hf in 1 0; do for lf in 0 1; do
  echo "== heavy_first=$hf light_first=$lf"
  GCOO_SPLIT_HEAVY_FIRST=$hf GCOO_SPLIT_LIGHT_FIRST=$lf timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | cut -c1-120
  GCOO_SPLIT_HEAVY_FIRST=$hf GCOO_SPLIT_LIGHT_FIRST=$lf timeout 300 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:spdm_tacc -s 2 -c 2 --csv python tools/prof_one.py --powerlaw --s 0.99 2>/dev/null | python -c "
import csv, sys
for r in csv.reader(sys.stdin):
    if len(r) > 14 and r[0] != 'ID': print('   ', r[4][:48], r[-3], r[-1])"
done; done
