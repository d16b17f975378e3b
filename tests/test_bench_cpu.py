"""bench.py's driver contract on CPU: the reference arm (`--impl reference`,
the reference's own spdm_gcoo from oracle/_ref on the host cores) prints one
JSON line with the metric, config and cpu_baseline / e2e blocks the driver
reads, and both arms describe the workload with the same config object."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgcoo_ref.so")):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--n", "512", "--sparsity", "0.95"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    sys.path.insert(0, ROOT)
    import bench
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "GFLOPS"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["config"] == bench.workload_config(512, 0.95, d["config"]["nnz"])
    assert d["config"]["nnz"] == round(512 * 512 * 0.05)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["isa_flags"] is not None
    assert d["e2e"] == {"value": d["value"], "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_compulsory_bytes_formula():
    """12 B per nonzero + 16 B per group + B rows touched + C."""
    sys.path.insert(0, ROOT)
    import bench
    # configs[1]: n=8000, s=0.99 -> 519.712 MB per launch (every B row is touched)
    assert bench.compulsory_bytes(640000, 8000, 8000, 8000, 4, 8000) == 519712000
