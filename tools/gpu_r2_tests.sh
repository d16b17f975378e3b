#!/bin/bash
# The GPU suite (optionally -k $K) + smoke; summary lines only.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu ${K:+-k "$K"} > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
grep -E "passed|failed|Error|error|assert" gpurun_out/r2_pytest.log | tail -30; tail -2 gpurun_out/r2_smoke.log
