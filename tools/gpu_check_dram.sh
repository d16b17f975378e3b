#!/bin/bash
# GPU tests, the full bench (sweep + power-law + n=32768), and DRAM bytes of the multiply at s=0.9/0.99/0.995.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 1500 gpurun_out/bench_full.json
for s in 0.9 0.99 0.995; do
  echo "s=$s"
  timeout 300 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spdm_t -s 1 -c 1 python tools/prof_one.py --s $s --kernel auto 2>&1 | grep -E "dram__|gpu__time"
done
timeout 300 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spdm_t -s 1 -c 1 python tools/prof_one.py --n 16384 --powerlaw --s 0.99 --kernel auto 2>&1 | grep -E "dram__|gpu__time"
