#!/bin/bash
# How often the reference acceptance gate's c7 (desk-scale timing
# properties, host-API calls with pageable buffers at n=2000) passes per host
# staging configuration: 6 gate runs each, criterion 7 lines only.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "GCOO_HOST_STAGING=1" "GCOO_HOST_STAGING=0" "GCOO_HOST_THREADS=8" "GCOO_HOST_THREADS=4"; do
  for i in 1 2 3 4 5 6; do
    echo "$cfg run $i: $(env $cfg timeout 300 tests/cpp/_build/ref_acceptance /nonexistent/gcoo_bench 2>&1 | grep 'criterion 7')"
  done
done
