#!/bin/bash
# configs[3] (power-law n=16384) step and kernel time under the two-class split:
# FACTORS (degree threshold / mean), ROWS (exact heavy row counts), HK (heavy kinds).
cd "$(dirname "$0")/.."
run() { timeout 300 python tools/kernel_sweep.py --powerlaw --s 0.99 --kernels auto --reps 7 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('   ', d['kernel'], d['kernel_ms'], d['ms'])"; }
for f in ${FACTORS:-1}; do echo "== factor $f"; GCOO_SPLIT_FACTOR=$f run; done
for h in ${ROWS:-}; do for k in ${HK:-auto}; do
  echo "== rows $h heavy kind $k"
  if [ "$k" = auto ]; then GCOO_SPLIT_ROWS=$h run; else GCOO_SPLIT_ROWS=$h GCOO_SPLIT_HEAVY_KIND=$k run; fi
done; done
