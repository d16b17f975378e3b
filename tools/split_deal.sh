#!/bin/bash
# configs[3]: heavy-class placement (GCOO_SPLIT_HEAVY_DEAL 1 = dealt round-robin over
# row blocks, plain order; 0 = heaviest rows packed into block 0, launched first):
# step time and DRAM bytes of the two kernels (ncu).
cd "$(dirname "$0")/.."
q() { python -c "
import csv, sys
for r in csv.reader(sys.stdin):
    if len(r) > 14 and r[0] != 'ID': print('   ', r[4][:48], r[-3], r[-1])"; }
for d in 1 0; do
  echo "== deal=$d"
  GCOO_SPLIT_HEAVY_DEAL=$d timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | cut -c1-110
  GCOO_SPLIT_HEAVY_DEAL=$d timeout 300 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:spdm_tacc -s 2 -c 2 --csv python tools/prof_one.py --powerlaw --s 0.99 2>/dev/null | q
done
