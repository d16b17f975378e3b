#!/bin/bash
# Profiling call: microbenchmarks, ncu launch list of one bench run, one ncu --set full capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
[ -n "$MB" ] && for b in $MB; do timeout 300 ./tools/microbench/$b > gpurun_out/mb_$b.jsonl 2>&1; done
if [ -n "$LAUNCHES" ]; then
  timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_one.py --s ${LS:-0.99} --kernel ${LK:-auto} --launches 3 > gpurun_out/launches_bench.log 2>&1
fi
for cfg in $PROF; do   # e.g. "0.99:tacc_v4"
  s=${cfg%%:*}; k=${cfg##*:}
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:${KREGEX:-spdm} -s ${SKIP:-1} -c 1 \
    -o gpurun_out/prof_${k}_s${s} -f python tools/prof_one.py --s $s --kernel $k > gpurun_out/ncu_${k}_s${s}.log 2>&1
done
ls -la gpurun_out; cat gpurun_out/mb_*.jsonl 2>/dev/null
