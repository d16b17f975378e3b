#!/bin/bash
# Round-2 check: new GPU tests, the acceptance gate, bench (N=1) and a 2-rank
# plumbing run of bench.py on one GPU (gloo).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "multirank or acceptance" > gpurun_out/r2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.log
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?" >> gpurun_out/r2_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-sweep > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench2 rc=$?" >> gpurun_out/r2_bench2.err
tail -15 gpurun_out/r2_tests.log; cat gpurun_out/r2_bench.json; tail -5 gpurun_out/r2_bench.err; cat gpurun_out/r2_bench2.json; tail -5 gpurun_out/r2_bench2.err
