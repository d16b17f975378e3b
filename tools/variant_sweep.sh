#!/bin/bash
# Kernel-only times of each measurement variant in tools/_abl (args: variant names; env S, KERNELS, POWERLAW).
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  GCOO_LIB=tools/_abl/libgcoo_$v.so timeout 600 python tools/kernel_sweep.py --s ${S:-0.99 0.995} --kernels ${KERNELS:-auto} --reps ${REPS:-7} $POWERLAW 2>&1 | grep -v "^$" | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print(d['s'], d['kernel'], d['kernel_ms'], d['ms'], d['bitwise_equal_first'])
    except Exception: print(l.rstrip())
"
done
