#!/bin/bash
# Evidence refresh at HEAD when the multiply kernel is unchanged since the last
# full bundle (tools/gpu_evidence_final.sh): GPU suite + smoke, bench (N=1) and
# the reference arm, a 2-rank plumbing run on one GPU, the ncu launch list of
# the bench (compute-sanitizer is closed on this pool).  Outputs in gpurun_out/eh_*.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 python -m pytest tests -q -m gpu -rA > gpurun_out/eh_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/eh_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/eh_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/eh_smoke.log
timeout 900 python bench.py > gpurun_out/eh_bench.json 2> gpurun_out/eh_bench.err; echo "bench rc=$?" >> gpurun_out/eh_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/eh_bench_reference.json 2> gpurun_out/eh_bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/eh_bench_2rank.json 2> gpurun_out/eh_bench_2rank.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eh_launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-strong > gpurun_out/eh_launches_bench.log 2>&1
grep -E "passed|failed" gpurun_out/eh_pytest.log | tail -2; tail -2 gpurun_out/eh_smoke.log; tail -1 gpurun_out/eh_bench.err
