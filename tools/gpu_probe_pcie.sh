cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie_probe.jsonl 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
cat gpurun_out/pcie_probe.jsonl gpurun_out/e2e_probe.txt
