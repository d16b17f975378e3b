#!/bin/bash
# ncu --set full of the default multiply at s=0.9/0.99/0.995 and the traffic cross-check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for s in 0.9 0.99 0.995; do
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_t -s 1 -c 1 \
    -o gpurun_out/prof3_s$s -f python tools/prof_one.py --s $s --kernel auto > gpurun_out/ncu3_s$s.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof3_s$s.ncu-rep > gpurun_out/ncu3_s$s.json
done
python tools/traffic_crosscheck.py gpurun_out/ncu3_s0.9.json gpurun_out/ncu3_s0.99.json gpurun_out/ncu3_s0.995.json > gpurun_out/crosscheck3.jsonl 2>&1
cat gpurun_out/crosscheck3.jsonl | cut -c1-300
