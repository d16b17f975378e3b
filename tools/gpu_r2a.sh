cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?" >> gpurun_out/r2a_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2a_bench_ref.json 2> gpurun_out/r2a_bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2a_bench2.json 2> gpurun_out/r2a_bench2.err; echo "bench2 rc=$?" >> gpurun_out/r2a_bench2.err
tail -5 gpurun_out/r2a_pytest.log; tail -2 gpurun_out/r2a_smoke.log; cat gpurun_out/r2a_bench.json; tail -3 gpurun_out/r2a_bench.err; cat gpurun_out/r2a_bench_ref.json; cat gpurun_out/r2a_bench2.json; tail -3 gpurun_out/r2a_bench2.err
