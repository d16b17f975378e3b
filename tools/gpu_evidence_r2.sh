#!/bin/bash
# Round-2 evidence: ncu launch list of a bench run, ncu --set full of the
# multiply at s=0.99 / 0.995 and of configs[3]'s two split kernels, and raw
# compute-sanitizer logs.  Outputs in gpurun_out/ (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-strong > gpurun_out/r02_launches_bench.log 2>&1
for s in 0.99 0.995; do
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 1 -c 1 \
    -o gpurun_out/r02_prof_s$s -f python tools/prof_one.py --s $s --kernel auto > gpurun_out/r02_ncu_s$s.log 2>&1
  python tools/ncu_summary.py gpurun_out/r02_prof_s$s.ncu-rep > gpurun_out/r02_ncu_s$s.json
done
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 2 -c 2 \
  -o gpurun_out/r02_prof_powerlaw -f python tools/prof_one.py --powerlaw --s 0.99 --kernel auto > gpurun_out/r02_ncu_powerlaw.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_prof_powerlaw.ncu-rep > gpurun_out/r02_ncu_powerlaw.json
timeout 900 $SAN --tool memcheck python tools/sanitize_probe.py > gpurun_out/r02_memcheck.log 2>&1
timeout 1200 $SAN --tool racecheck --racecheck-report hazard python tools/sanitize_probe.py > gpurun_out/r02_racecheck.log 2>&1
tail -3 gpurun_out/r02_memcheck.log gpurun_out/r02_racecheck.log; cat gpurun_out/r02_ncu_s0.99.json | head -30
