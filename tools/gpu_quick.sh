#!/bin/bash
# Quick GPU check: the tests named by $K (pytest -k), then an optional command in $CMD.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu ${K:+-k "$K"} > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_pytest.log
tail -3 gpurun_out/quick_pytest.log
if [ -n "$CMD" ]; then timeout 900 bash -c "$CMD" > gpurun_out/quick_cmd.log 2>&1; echo "cmd rc=$?" >> gpurun_out/quick_cmd.log; tail -40 gpurun_out/quick_cmd.log; fi
