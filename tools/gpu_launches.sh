#!/bin/bash
# ncu launch list (per-kernel durations) of a short bench run: planner chain + multiply.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-strong > gpurun_out/launches_bench.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/launches_bench.log | cut -c1-300
