#!/bin/bash
# Refresh measured evidence after a kernel change: crossover sweep (incl. cuSPARSE),
# ncu full capture + launch list of the default kernel, traffic cross-check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python tools/sweep_crossover.py > gpurun_out/sweep_crossover3.jsonl 2> gpurun_out/sweep_crossover3.err
for s in 0.9 0.99 0.995; do
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_t -s 1 -c 1 \
    -o gpurun_out/prof28_s$s -f python tools/prof_one.py --s $s --kernel auto > gpurun_out/ncu28_s$s.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof28_s$s.ncu-rep > gpurun_out/ncu28_s$s.json
done
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches28.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches28_bench.log 2>&1
timeout 300 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spdm_t -s 1 -c 1 python tools/prof_one.py --s 0.99 --kernel auto 2>&1 | grep -E "dram__|gpu__time" > gpurun_out/dram28.txt
cat gpurun_out/dram28.txt; tail -8 gpurun_out/sweep_crossover3.jsonl | cut -c1-200
