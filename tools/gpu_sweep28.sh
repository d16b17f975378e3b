#!/bin/bash
# Kernel sweep of every fp32 TMEM/tile configuration, n=8000 (kernel-only and step ms).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/kernel_sweep.py --s 0.8 0.85 0.9 0.93 0.95 0.97 0.98 0.985 0.99 0.995 0.998 0.999 \
  --kernels auto tile_v4 tacc_v4 tacc_v4_k216 tacc_v4w tacc28_k200 tacc28_k192 tacc28_k160 tacc28_k128 tacc28_k96 tacc28_k64 rowtile --reps 3 \
  > gpurun_out/kernel_sweep_28w.jsonl 2>&1
