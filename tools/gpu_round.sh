#!/bin/bash
# Round evidence in one call: GPU tests, smoke, bench, the ncu launch list of a
# short bench run, and one `ncu --set full` capture of the multiply kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:spdm_tacc -s 1 -c 1 \
  -o gpurun_out/prof_round -f python tools/prof_one.py --s 0.99 --kernel auto > gpurun_out/ncu_round.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_round.ncu-rep > gpurun_out/ncu_round.json 2>/dev/null
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
cat gpurun_out/bench_ref.json
