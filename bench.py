#!/usr/bin/env python
"""GCOOSpDM benchmark on B200 (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE.json configs[1], the metric's configuration): the
reference's square_benchmark(seed=1) inputs (bench.hpp:168-174) at n=8000,
sparsity 0.99 — A = generate_uniform_sparse(8000, 0.99, 1) (640,000 nnz), B =
generate_uniform_sparse(8000, 0, derive_seed(1, 8000, 0xb)) dense fp32,
ExecConfig{p=4, b=64}.  A step = one spdm_gcoo(A_gcoo, B) -> C.

Multi-GPU (configs[4] decomposition): B and C are column-sharded with A
replicated; every rank owns an 8000-column block of B/C (weak scaling: per-GPU
work fixed, the global problem is A[8000x8000] x B[8000 x 8000N]).  There is no
collective on the data path; NCCL is used for the barrier and the max-over-
ranks timing only.

value      kernel-only GFLOPS (2*nnz*N / t), operands resident in HBM, L2 flushed
           (256 MiB write) before every timed launch, CUDA events on the
           launching stream, max over ranks.
e2e        the same metric through the public host API (paper_2005_14469_b200.
           spdm_gcoo -> C ABI gcoo_spdm_f32): pinned host A/B in, pinned host C
           out, copies inside the timed region.
--impl reference  times the reference's own CPU spdm_gcoo (oracle/_ref, built
           from the unmodified reference sources) with all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DIM = 8000
SPARSITY = 0.99
SEED = 1
P, BW = 4, 64
METRIC = "GCOOSpDM GFLOPS (2·nnz·N) and HBM GB/s-% roofline at 1/2/4/8 B200 vs CPU ref"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp32_peak_tflops():
    """FFMA peak from this repo's microbenchmark (tools/microbench, profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_microbench.json")) as f:
            return float(json.load(f)["ffma_tflops"]), "measured (tools/microbench)"
    except Exception:
        return 148 * 128 * 2 * 1.965e9 / 1e12, "derived 148 SM x 128 x 2 x 1.965 GHz"


def compulsory_bytes(nnz, m, k, n, p, k_nz):
    # A triples + group arrays + B rows that are touched + C once
    return 12 * nnz + 16 * (-(-m // p)) + 4 * k_nz * n + 4 * m * n


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.first = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("BENCH_CLOCK_LMS", "20")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # wait for the first sample: nvidia-smi's NVML start-up briefly stalls the
            # GPU, and must not land inside the timed region
            import threading
            box = []
            t = threading.Thread(target=lambda: box.append(self.proc.stdout.readline()), daemon=True)
            t.start()
            t.join(timeout=30)
            self.first = box[0] if box else ""
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        lines = (self.out or "").strip().splitlines() or [self.first]  # pre-region sample only if none inside
        for line in lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, fl in rows for i, v in enumerate(fl) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def pcie_roofline(nbytes, seconds):
    """The host-pointer path is PCIe-bound: its bytes per second against the
    measured concurrent H2D+D2H bandwidth of this pool's B200 host link
    (tools/pcie_probe.py -> profiles/r01_pcie_probe.jsonl)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_pcie_probe.jsonl")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        peak = max(r["gb_s"] for r in rows if r["probe"].startswith("h2d+d2h"))
    except Exception:  # noqa: BLE001
        return {}
    ach = nbytes / seconds / 1e9
    return {"pcie_gb_s": round(ach, 1), "pcie_peak_gb_s": peak, "pcie_frac": round(ach / peak, 3),
            "pcie_peak_source": "measured concurrent H2D+D2H (profiles/r01_pcie_probe.jsonl)"}


def make_inputs(G, n, s, seed, dev, n_cols):
    """square_benchmark inputs; B/C column block of width n_cols (same B for
    every rank's block: B is generated once at n x n and tiled)."""
    import torch
    a = G.generate_uniform_sparse(n, s, seed)
    b = G.generate_uniform_sparse(n, 0.0, G.derive_seed(seed, n, 0xB))
    if n_cols != n:
        reps = -(-n_cols // n)
        b = np.ascontiguousarray(np.tile(b, (1, reps))[:, :n_cols])
    dA = torch.from_numpy(a).to(dev)
    dg = G.dense_to_gcoo_dev(dA, P)
    del dA
    dB = torch.from_numpy(b).to(dev)
    torch.cuda.synchronize()  # inputs complete before other streams use them
    return a, b, dg, dB


def time_kernel(G, dg, dB, dC, steps, warmup, stream, flush):
    import torch
    cfg = G.ExecConfig(p=P, b=BW)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush.zero_()
            G.spdm_gcoo_dev(dg, dB, dC, cfg, stream=stream)
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        l0 = G.launch_count()
        G.kernel_timing(True)  # CUDA events around each multiply-kernel launch, same stream
        # the device sleeps ~5 ms first so the host queues the timed steps ahead of it:
        # per-step device times then never include host enqueue latency
        torch.cuda._sleep(int(1e7))
        for i in range(steps):
            flush.zero_()  # > L2 (126 MB): every timed launch starts cold
            starts[i].record(stream)
            G.spdm_gcoo_dev(dg, dB, dC, cfg, stream=stream)
            ends[i].record(stream)
        torch.cuda.synchronize()
        launches = G.launch_count() - l0
        k_ms, k_n = G.kernel_time()
        G.kernel_timing(False)
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    return sum(times) / len(times), min(times), launches, k_ms / max(k_n, 1)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2005_14469_b200 as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    ndev = torch.cuda.device_count()
    local = local % ndev  # more ranks than GPUs only for plumbing checks (gloo below)
    torch.cuda.set_device(local)
    G.set_device(local)
    dev = torch.device("cuda", local)
    backend = "nccl" if world <= ndev else "gloo"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    red_dev = dev if backend == "nccl" else torch.device("cpu")

    n, s = args.n, args.sparsity
    a_host, b_host, dg, dB = make_inputs(G, n, s, SEED, dev, n)
    nnz = dg.nnz()
    m = k = n
    dC = torch.empty((m, n), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB
    stream = torch.cuda.Stream(device=dev)

    # ---- kernel-only, device-resident ----------------------------------
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ms_mean, ms_min, launches, kernel_ms = time_kernel(G, dg, dB, dC, args.steps, args.warmup, stream, flush)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ms_mean, ms_min, kernel_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_mean, ms_min, kernel_ms = float(t[0]), float(t[1]), float(t[2])
    flops_rank = 2.0 * nnz * n
    value = world * flops_rank / (ms_mean * 1e-3) / 1e9

    # ---- plan reuse (extension): the same multiply, A's record stream built once
    plan_reuse = None
    try:
        plan = G.SpdmPlan(dg, stream=stream)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.zero_()
                plan.run(dB, dC, stream=stream)
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            torch.cuda._sleep(int(1e7))
            for e0, e1 in evs:
                flush.zero_()
                e0.record(stream)
                plan.run(dB, dC, stream=stream)
                e1.record(stream)
            torch.cuda.synchronize()
        pms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs)
        plan.close()
        plan_reuse = {"ms_per_step": round(pms, 4), "value": round(world * 2.0 * nnz * n / (pms * 1e-3) / 1e9, 2),
                      "unit": "GFLOPS", "note": "gcoo_plan_* (A's record stream built once, then one multiply "
                                                "kernel per B); not the headline, which plans every call"}
    except Exception as e:  # noqa: BLE001
        plan_reuse = {"error": str(e)[:200]}

    # ---- end to end through the public host API ----------------------
    g_host = dg.to_host()
    b_pin = torch.empty((k, n), dtype=torch.float32, pin_memory=True)
    b_pin.numpy()[:] = b_host
    c_pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    def pin(x):
        t_ = torch.empty(x.shape, dtype=getattr(torch, str(x.dtype)), pin_memory=True)
        t_.numpy()[...] = x
        return t_.numpy()

    g_pin = G.GcooMatrix(g_host.rows_dim, g_host.cols_dim, g_host.p, pin(g_host.values), pin(g_host.row_idx),
                         pin(g_host.col_idx), pin(g_host.g_idxes), pin(g_host.nnz_per_group))
    cfg = G.ExecConfig(p=P, b=BW)
    for _ in range(max(1, args.warmup)):
        G.spdm_gcoo(g_pin, b_pin.numpy(), cfg, out=c_pin.numpy())
    if world > 1:
        dist.barrier()
    # each call timed on its own (host clock around the whole API call: copies in,
    # multiply, copy out, synchronised); the median is robust to host hiccups
    e2e_steps = max(5, min(args.steps, 20))
    e2e_times = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        G.spdm_gcoo(g_pin, b_pin.numpy(), cfg, out=c_pin.numpy())
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_times)
    te = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te[0])
    e2e_value = world * flops_rank / e2e_s / 1e9
    h2d = g_host.values.nbytes + g_host.row_idx.nbytes + g_host.col_idx.nbytes + g_host.g_idxes.nbytes + \
        g_host.nnz_per_group.nbytes + b_host.nbytes
    d2h = m * n * 4

    # C sanity against the reference hash (computed on rank 0 only at n=8000)
    parity = None
    if rank == 0 and n == 8000:
        try:
            with open(os.path.join(ROOT, "tests", "golden", "hashes.json")) as f:
                ent = json.load(f)[f"n8000_s{s}"]
            parity = {"c0": float(dC[0, 0]), "clast": float(dC[-1, -1]),
                      "c0_ref_fma": ent["C_fma"]["c0"], "clast_ref_fma": ent["C_fma"]["clast"],
                      "checksum": float(dC.double().sum()), "checksum_ref_fma": ent["C_fma"]["checksum"]}
            parity["match"] = (parity["c0"] == parity["c0_ref_fma"] and parity["clast"] == parity["clast_ref_fma"]
                               and abs(parity["checksum"] - parity["checksum_ref_fma"]) < 1e-3)
        except Exception as e:  # noqa: BLE001
            parity = {"error": str(e)}

    # ---- roofline --------------------------------------------------------
    hbm_peak, hbm_src = peaks()
    k_nz = int(np.count_nonzero(np.bincount(g_host.col_idx, minlength=k)))
    cb = compulsory_bytes(nnz, m, k, n, P, k_nz)
    achieved_gbs = cb / (kernel_ms * 1e-3) / 1e9  # dominant kernel: the multiply, event-timed
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tr = json.load(f)
            if tr.get("n") == n and tr.get("sparsity") == s:
                traffic = tr.get("dram_bytes_per_launch")
        except Exception:
            pass
    # the paper's argument, measured: where the multiply's bytes move (ncu --set full
    # of the same launch, profiles/r01_ncu_tacc28_s0.99.json)
    traffic_split = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_tacc28_s0.99.json")) as f:
            nc = json.load(f)
        if n == 8000 and s == 0.99:
            dram = nc["dram_read_bytes"] + nc["dram_write_bytes"]
            traffic_split = {"dram_bytes": int(dram), "l2_to_sm_bytes": int(nc["l2_read_bytes_from_sm"]),
                             "shared_memory_bytes": int(nc["smem_wavefronts"] * 128),
                             "shared_memory_busy_frac": round(nc["smem_wavefront_pct"] / 100, 3),
                             "source": "ncu --set full, profiles/r01_ncu_tacc28_s0.99.json (LSU wavefronts x 128 B)"}
    except Exception:  # noqa: BLE001
        pass
    fp_peak, fp_src = fp32_peak_tflops()
    tflops = flops_rank / (kernel_ms * 1e-3) / 1e12

    extra = {}
    if rank == 0 and world == 1 and not args.no_sweep:
        for s2 in (0.9, 0.995):
            _, _, dg2, _ = make_inputs(G, n, s2, SEED, dev, n)
            ms2, _, _, _ = time_kernel(G, dg2, dB, dC, max(3, args.steps // 2), 3, stream, flush)
            f2 = 2.0 * dg2.nnz() * n
            cb2 = compulsory_bytes(dg2.nnz(), m, k, n, P, k)
            extra[f"s{s2}"] = {"nnz": dg2.nnz(), "ms": round(ms2, 4), "gflops": round(f2 / ms2 / 1e6, 1),
                               "hbm_frac": round(cb2 / (ms2 * 1e-3) / 1e9 / hbm_peak, 4),
                               "fp32_frac": round(f2 / (ms2 * 1e-3) / 1e12 / fp_peak, 4)}
            del dg2

    if rank == 0 and world == 1 and not args.no_sweep:
        extra.update(other_configs(G, dev, stream, flush, hbm_peak, fp_peak))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g_host, b_host, n)

    gather = None
    if world > 1:
        # the optional C gather onto rank 0 (NCCL point to point), timed on its own —
        # not part of the multiply step
        from paper_2005_14469_b200.shard import gather_columns
        shards = [(r * n, (r + 1) * n) for r in range(world)]
        dist.barrier()
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        full = gather_columns(dC if backend == "nccl" else dC.cpu(), shards, root=0)
        torch.cuda.synchronize()
        gt = torch.tensor([time.perf_counter() - g0], dtype=torch.float64, device=red_dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather = {"ms": round(float(gt[0]) * 1e3, 3), "bytes_to_root": int(m * n * 4 * (world - 1)),
                  "collective": f"{backend} point-to-point onto rank 0"}
        if full is not None:
            ok = bool(torch.equal(full[:, :n].to(dC.device), dC))
            gather["rank0_block_intact"] = ok
        del full
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GFLOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_mean, 4),
        "ms_per_step_min": round(ms_min, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: reference square_benchmark(seed=1) generator, bit-identical inputs",
        "config": {"workload": f"GCOOSpDM n={n} s={s} uniform-random A x dense B, fp32 (BASELINE configs[1])",
                   "m": m, "k": k, "n_per_gpu": n, "n_total": n * world, "nnz": nnz, "p": P, "b": BW,
                   "parallelism": f"column-shard B/C x{world}, A replicated (rank r owns columns "
                                  f"[r*{n}, (r+1)*{n}) of a {n}x{n * world} B/C; no data-path collective)",
                   "dist_backend": backend if world > 1 else None,
                   "l2": "flushed (256 MiB write) before every timed launch; B+C = 512 MB > L2"},
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOPS", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_s * 1e3, 3),
                "ms_per_step_mean": round(statistics.mean(e2e_times) * 1e3, 3), "calls": len(e2e_times),
                "path": "paper_2005_14469_b200.spdm_gcoo -> gcoo_spdm_f32 (pinned host buffers)",
                **pcie_roofline(h2d + d2h, e2e_s)},
        "gpu_launches": int(launches),
        "plan_reuse": plan_reuse,
        "c_gather": gather,
        "roofline": {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved_gbs / hbm_peak, 4), "traffic": traffic,
                     "peak_source": hbm_src, "algorithmic_bytes_per_launch": int(cb),
                     "kernel_ms": round(kernel_ms, 4), "kernel_share_of_step": round(kernel_ms / ms_mean, 3),
                     "bytes_formula": "12*nnz + 16*ceil(m/p) + 4*k_nz*N + 4*m*N (SURVEY 8d)"},
        "traffic_split": traffic_split,
        "roofline_fp32": {"achieved": round(tflops, 3), "peak": round(fp_peak, 2), "unit": "TFLOP/s",
                          "frac": round(tflops / fp_peak, 4), "peak_source": fp_src,
                          "note": "the path is an FP32 FFMA gather: this, not HBM, is its binding roofline"},
        "clocks": clk.summary(),
        "parity": parity,
        "sweep": extra,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def other_configs(G, dev, stream, flush, hbm_peak, fp_peak, steps=5):
    """BASELINE configs[3] (power-law A, n=16384, s=0.99) and configs[4]'s
    single-GPU point (n=32768, s=0.99): A from this repo's power-law generator
    / the reference's uniform sample (as COO, grouped on the GPU); B uniform
    (0,1] generated on the device (its values do not change the work)."""
    import torch
    out = {}
    cases = [("powerlaw_n16384_s0.99", 16384, lambda: G.generate_powerlaw_coo(16384, 0.99, 1.0, SEED)),
             ("uniform_n32768_s0.99", 32768, lambda: G.generate_uniform_sparse_coo(32768, 0.99, SEED))]
    for name, n, gen in cases:
        try:
            v, r, c = gen()
            dg = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                   torch.from_numpy(c).to(dev), P)
            k_nz = int(torch.unique(dg.col_idx).numel())
            gen_b = torch.Generator(device=dev).manual_seed(SEED)
            dB = 1.0 - torch.rand((n, n), device=dev, dtype=torch.float32, generator=gen_b)
            dC = torch.empty((n, n), device=dev, dtype=torch.float32)
            torch.cuda.synchronize()
            ms, ms_min, _, kms = time_kernel(G, dg, dB, dC, steps, 3, stream, flush)
            nnz = dg.nnz()
            f = 2.0 * nnz * n
            cb = compulsory_bytes(nnz, n, n, n, P, k_nz)
            rows = torch.bincount(dg.row_idx.long(), minlength=n)
            out[name] = {"n": n, "nnz": nnz, "max_row_nnz": int(rows.max()), "ms": round(ms, 4),
                         "kernel_ms": round(kms, 4), "gflops": round(f / ms / 1e6, 1),
                         "hbm_frac": round(cb / (kms * 1e-3) / 1e9 / hbm_peak, 4),
                         "fp32_frac": round(f / (kms * 1e-3) / 1e12 / fp_peak, 4)}
            del dg, dB, dC
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": str(e)[:200]}
    return out


def cpu_baseline(g_host, b_host, n):
    """The reference's own CPU spdm_gcoo (oracle/_ref) on this host's cores."""
    try:
        from oracle import Gcoo, Reference, have_reference
    except Exception as e:  # noqa: BLE001
        return {"error": f"oracle unavailable: {e}"}
    cores = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    g = Gcoo(g_host.rows_dim, g_host.cols_dim, g_host.p, g_host.values, g_host.row_idx, g_host.col_idx,
             g_host.g_idxes, g_host.nnz_per_group)
    if have_reference():
        R = Reference(False)
        # every host core, explicitly (torchrun exports OMP_NUM_THREADS=1)
        r = R.time_spdm(g, b_host, b=BW, workers=cores, warmup=1, reps=3)
        kc = r["kc_s"]
        return {"value": round(2.0 * g.nnz * n / kc / 1e9, 3), "unit": "GFLOPS", "cores": int(r["workers"]),
                "kind": "reference",
                "sample": f"full workload (n={n}, nnz={g.nnz}): reference spdm_gcoo, median of 3 after 1 warmup, "
                          f"OpenMP {r['workers']} threads, default-ISA build",
                "kc_seconds": kc}
    return {"error": "oracle/_ref not built"}


def run_reference(args):
    """--impl reference: the reference's CPU spdm_gcoo on the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import Reference, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return
    cores = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
    R = Reference(False)
    n, s = args.n, args.sparsity
    a = R.uniform_sparse(n, s, SEED)
    b = R.uniform_sparse(n, 0.0, R.derive_seed(SEED, n, 0xB))
    g = R.dense_to_gcoo(a, P)
    # every host core, explicitly: torchrun exports OMP_NUM_THREADS=1 to its ranks
    r = R.time_spdm(g, b, b=BW, workers=cores, warmup=max(0, min(args.warmup, 2)), reps=max(1, args.steps))
    kc = r["kc_s"]
    v = 2.0 * g.nnz * n / kc / 1e9
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "GFLOPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(kc * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic: reference square_benchmark(seed=1)",
        "config": {"workload": f"GCOOSpDM n={n} s={s} uniform-random A x dense B, fp32 (BASELINE configs[1])",
                   "m": n, "k": n, "n_per_gpu": n, "nnz": g.nnz, "p": P, "b": BW},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOPS", "cores": int(r["workers"]), "kind": "reference",
                         "sample": f"full workload each step: reference spdm_gcoo (median of {max(1, args.steps)}),"
                                   f" OpenMP {r['workers']} threads of {cores}"},
        "e2e": {"value": round(v, 3), "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_DIM)
    ap.add_argument("--sparsity", type=float, default=SPARSITY)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
