#!/bin/bash
# Kernel iteration loop on the GPU box: correctness of every fp32 variant,
# memcheck of the tiled kernels, kernel sweep, optional ncu captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "each_fp32 or golden or random_shapes" 2>&1 | tail -4 > gpurun_out/iter_pytest.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -x -q -k "each_fp32" 2>&1 | tail -4 > gpurun_out/iter_sanitizer.log
timeout 600 python tools/kernel_sweep.py ${SWEEP_ARGS:-} > gpurun_out/iter_sweep.jsonl 2>&1
if [ -n "$PROF" ]; then
  for cfg in $PROF; do   # e.g. "0.99:tacc_v4 0.9:tile_v4"
    s=${cfg%%:*}; k=${cfg##*:}
    timeout 600 $NCU --set full --import-source on --clock-control none -k regex:${KREGEX:-spdm} -s 1 -c 1 \
      -o gpurun_out/prof_${k}_s${s} python tools/prof_one.py --s $s --kernel $k > gpurun_out/ncu_${k}_s${s}.log 2>&1
  done
fi
cat gpurun_out/iter_pytest.log gpurun_out/iter_sanitizer.log gpurun_out/iter_sweep.jsonl
