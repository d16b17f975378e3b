#!/bin/bash
# ncu --set full with source attribution of the multiply at s=0.99 / 0.995
# (reports land in gpurun_out/, read here with ncu -i --page source).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for s in ${SPARSITIES:-0.99 0.995}; do
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 1 -c 1 \
    -o gpurun_out/src_s$s -f python tools/prof_one.py --s $s --kernel ${KERNEL:-auto} > gpurun_out/src_s$s.log 2>&1
  python tools/ncu_summary.py gpurun_out/src_s$s.ncu-rep > gpurun_out/src_s$s.json
done
ls -la gpurun_out/
