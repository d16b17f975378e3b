#!/bin/bash
# Round-2 evidence bundle at HEAD: GPU suite + smoke, bench (N=1) and the
# reference arm, a 2-rank plumbing run on one GPU, the ncu launch list of the
# bench, ncu --set full of the multiply at s=0.99 / 0.995 and of configs[3]'s
# split kernels, compute-sanitizer memcheck + racecheck, the format ablation.
# Outputs in gpurun_out/ev_* (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 python -m pytest tests -q -m gpu -rA > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?" >> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/ev_bench_reference.json 2> gpurun_out/ev_bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ev_bench_2rank.json 2> gpurun_out/ev_bench_2rank.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-strong > gpurun_out/ev_launches_bench.log 2>&1
for s in 0.99 0.995; do
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 1 -c 1 \
    -o gpurun_out/ev_prof_s$s -f python tools/prof_one.py --s $s --kernel auto > gpurun_out/ev_ncu_s$s.log 2>&1
  python tools/ncu_summary.py gpurun_out/ev_prof_s$s.ncu-rep > gpurun_out/ev_ncu_s$s.json
done
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 2 -c 2 \
  -o gpurun_out/ev_prof_powerlaw -f python tools/prof_one.py --powerlaw --s 0.99 --kernel auto > gpurun_out/ev_ncu_powerlaw.log 2>&1
python tools/ncu_summary.py gpurun_out/ev_prof_powerlaw.ncu-rep > gpurun_out/ev_ncu_powerlaw.json
timeout 900 $SAN --tool memcheck python tools/sanitize_probe.py > gpurun_out/ev_memcheck.log 2>&1
timeout 1200 $SAN --tool racecheck --racecheck-report hazard python tools/sanitize_probe.py > gpurun_out/ev_racecheck.log 2>&1
timeout 900 python tools/format_ablation.py > gpurun_out/ev_format_ablation.jsonl 2> /dev/null
rm -f gpurun_out/ev_prof_*.ncu-rep.tmp
grep -E "passed|failed" gpurun_out/ev_pytest.log | tail -2; tail -2 gpurun_out/ev_smoke.log; tail -1 gpurun_out/ev_bench.err
tail -2 gpurun_out/ev_memcheck.log; grep -c "RAW" gpurun_out/ev_racecheck.log
python - <<'P'
import json
d=json.load(open("gpurun_out/ev_bench.json"))
print("value",d["value"],"ms",d["ms_per_step"],"kernel",d["roofline"]["kernel_ms"],"e2e",d["e2e"]["value"],"pageable",d.get("e2e_pageable",{}).get("value"))
print("sweep",{k:(v.get("ms"),v.get("kernel_ms"),v.get("gflops")) for k,v in d.get("sweep",{}).items()})
print("strong",d.get("strong_n32768",{}).get("t1_ms"))
r=json.load(open("gpurun_out/ev_bench_reference.json")); print("reference", r["value"], r["unit"])
P
