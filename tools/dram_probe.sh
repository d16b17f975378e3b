#!/bin/bash
# DRAM bytes per multiply launch (ncu) at n=8000 s=0.9/0.99/0.995 and configs[3]; step times.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
q() { python -c "
import csv, sys
for r in csv.reader(sys.stdin):
    if len(r) > 14 and r[0] != 'ID': print('   ', r[4][:48], r[-3], r[-1])"; }
for s in 0.9 0.99 0.995; do
  echo "== s=$s"
  timeout 300 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:spdm_tacc -s 1 -c 1 --csv python tools/prof_one.py --s $s 2>/dev/null | q
done
echo "== powerlaw"
timeout 300 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:spdm_tacc -s 2 -c 2 --csv python tools/prof_one.py --powerlaw --s 0.99 2>/dev/null | q
timeout 300 python tools/kernel_sweep.py --s 0.9 0.99 0.995 --kernels auto --reps 7 | cut -c1-110
timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | cut -c1-110
