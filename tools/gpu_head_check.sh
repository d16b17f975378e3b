#!/bin/bash
# Whole-HEAD check: GPU suite + smoke + bench (N=1) + reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu ${K:+-k "$K"} > gpurun_out/hc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/hc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/hc_smoke.log
timeout 600 python bench.py > gpurun_out/hc_bench.json 2> gpurun_out/hc_bench.err; echo "bench rc=$?" >> gpurun_out/hc_bench.err
grep -E "passed|failed|Error|error|assert" gpurun_out/hc_pytest.log | tail -30; tail -2 gpurun_out/hc_smoke.log; tail -3 gpurun_out/hc_bench.err
python - <<'P'
import json
d=json.load(open("gpurun_out/hc_bench.json"))
print("value",d["value"],"ms",d["ms_per_step"],"e2e",d["e2e"]["value"],"pageable",d.get("e2e_pageable",{}).get("value"))
print("sweep",{k:(v.get("ms"),v.get("kernel_ms"),v.get("gflops")) for k,v in d.get("sweep",{}).items()})
print("strong",d.get("strong_n32768",{}).get("t1_ms"))
P
