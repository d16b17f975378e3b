#!/usr/bin/env python
"""GCOOSpDM benchmark on B200 (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE.json configs[1], the metric's configuration): the
reference's square_benchmark(seed=1) inputs (bench.hpp:168-174) at n=8000,
sparsity 0.99 — A = generate_uniform_sparse(8000, 0.99, 1) (640,000 nnz), B =
generate_uniform_sparse(8000, 0, derive_seed(1, 8000, 0xb)) dense fp32,
ExecConfig{p=4, b=64}.  A step = one spdm_gcoo(A_gcoo, B) -> C.

value      kernel GFLOPS (2*nnz*N / t) of the whole job, operands resident in
           HBM, L2 flushed (256 MiB write) before every timed launch, CUDA
           events on the launching stream, max over ranks.  N > 1 is weak
           scaling (the north star's column sharding): rank r owns
           an 8000-column block of a B/C that is 8000*N wide (block 0 = the
           reference's B, block r from derive_seed(1 + r, 8000, 0xb)), A is
           replicated, no collective on the data path.
strong     BASELINE configs[4] (every N, its own block): n=32768, s=0.99, B/C
           split into N contiguous column shards (shard.column_shards), A
           built once on rank 0 and broadcast (NCCL); t_N = max over ranks of
           the shard multiply, t_1 = the whole product on rank 0 in the same
           run, speedup = t_1 / t_N; every shard's sampled rows equal the
           1-GPU product bit for bit; the optional C gather timed apart.
e2e        the same metric through the public host API (paper_2005_14469_b200.
           spdm_gcoo -> C ABI gcoo_spdm_f32): pinned host A/B in, pinned host C
           out, copies inside the timed region; `e2e_pageable` the same call
           with ordinary (pageable) numpy buffers, as a C++ std::vector caller.
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
STRONG_N = 32768
METRIC = "GCOOSpDM GFLOPS (2·nnz·N) and HBM GB/s-% roofline at 1/2/4/8 B200 vs CPU ref"
L2_NOTE = "GPU arm: 256 MiB write flushes L2 before every timed launch (B+C = 512 MB > 126 MB L2)"


def workload_config(n, s, nnz):
    """The `config` object, identical in both arms (the driver compares them)."""
    return {"workload": f"GCOOSpDM n={n} s={s} uniform-random A x dense B, fp32 (BASELINE configs[1])",
            "m": n, "k": n, "n_per_gpu": n, "nnz": int(nnz), "p": P, "b": BW, "l2": L2_NOTE}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback"


def fp32_peak_tflops():
    """FFMA peak from this repo's microbenchmark (tools/microbench, profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_microbench.json")) as f:
            return float(json.load(f)["ffma_tflops"]), "measured (tools/microbench/mb.cu, profiles/r01_microbench.json)"
    except Exception:
        return 148 * 128 * 2 * 1.965e9 / 1e12, "derived 148 SM x 128 x 2 x 1.965 GHz"


def compulsory_bytes(nnz, m, k, n, p, k_nz):
    # A triples + group arrays + B rows that are touched + C once
    return 12 * nnz + 16 * (-(-m // p)) + 4 * k_nz * n + 4 * m * n


def cpu_description():
    model, flags = "unknown", []
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and model == "unknown":
                    model = line.split(":", 1)[1].strip()
                if line.startswith("flags"):
                    have = set(line.split(":", 1)[1].split())
                    flags = [x for x in ("sse4_2", "avx", "avx2", "fma", "avx512f", "avx512vl", "avx512_bf16",
                                         "amx_tile") if x in have]
                    break
    except OSError:
        pass
    return {"cpu_model": model, "isa_flags": flags, "nproc": os.cpu_count()}


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


def pcie_duplex_probe(dev, nbytes=256 << 20, reps=5):
    """Concurrent pinned H2D + D2H bandwidth of this box's host link, measured
    in the same run (GB/s, best of `reps`): the host-pointer path's roofline.
    Boxes of this pool differ (80-99 GB/s measured), so a fixed figure would
    misstate the fraction."""
    import torch
    n = nbytes // 4
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dx = torch.empty(n, dtype=torch.float32, device=dev)
    dy = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    best = 0.0
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(dy, non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 2 * nbytes / (time.perf_counter() - t0) / 1e9)
    del hx, hy, dx, dy
    return best


def pcie_roofline(nbytes, seconds, peak):
    """The host-pointer path is PCIe-bound: its bytes per second against the
    concurrent H2D+D2H bandwidth measured on this box (pcie_duplex_probe)."""
    if not peak:
        return {}
    ach = nbytes / seconds / 1e9
    return {"pcie_gb_s": round(ach, 1), "pcie_peak_gb_s": round(peak, 1), "pcie_frac": round(ach / peak, 3),
            "pcie_peak_source": "measured in this run: concurrent pinned H2D + D2H of 256 MiB each, best of 5"}


def synth_b_block(k, lo, hi, dev):
    """B(i, j) in (0, 1] as a hash of (i, j) alone (24-bit mantissa values,
    exact in fp32): every rank can build its own column shard of the same
    global B on its device without a collective."""
    import torch
    out = torch.empty((k, hi - lo), dtype=torch.float32, device=dev)
    cols = torch.arange(lo, hi, dtype=torch.int64, device=dev)[None, :]
    M = 0xFFFFFFFF
    for r0 in range(0, k, 2048):
        r1 = min(k, r0 + 2048)
        rows = torch.arange(r0, r1, dtype=torch.int64, device=dev)[:, None]
        x = ((rows * 73856093) ^ (cols * 19349663) ^ 0x5BD1E995) & M
        x = ((x ^ (x >> 16)) * 0x45D9F3B) & M
        x = ((x ^ (x >> 16)) * 0x45D9F3B) & M
        x = x ^ (x >> 16)
        out[r0:r1] = ((x >> 8) + 1).to(torch.float32) * (1.0 / 16777216.0)
    return out


def make_inputs(G, n, s, seed, dev, b_seed):
    """square_benchmark inputs (B from b_seed: the reference's is derive_seed(seed, n, 0xb))."""
    import torch
    a = G.generate_uniform_sparse(n, s, seed)
    b = G.generate_uniform_sparse(n, 0.0, b_seed)
    dA = torch.from_numpy(a).to(dev)
    dg = G.dense_to_gcoo_dev(dA, P)
    del dA
    dB = torch.from_numpy(b).to(dev)
    torch.cuda.synchronize()  # inputs complete before other streams use them
    return a, b, dg, dB


def head_start_cycles(steps):
    """Device spin before a timed loop: ~2 ms per step at 1.965 GHz (a planned
    call costs the host ~60-70 us to enqueue; a slow or shared host has been
    seen to take ~1 ms, which would otherwise leak into the step times)."""
    return int(4e6 * max(steps, 3))


def time_kernel(G, dg, dB, dC, steps, warmup, stream, flush):
    """(mean ms per step, min ms, library launches in the timed region, mean ms
    of the multiply kernel itself) — CUDA events on `stream`, L2 flushed first.
    The step times come from a pass without the library's kernel-timing events
    (an event recorded between the planner and the multiply would sit inside
    their programmatic-dependent-launch chain and add ~9 us to a step); the
    multiply kernel's own time from a second pass with them."""
    import torch
    cfg = G.ExecConfig(p=dg.p, b=BW)

    def run(kernel_events):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        l0 = G.launch_count()
        G.kernel_timing(kernel_events)
        # the device sleeps first (~2 ms per timed step) so the host queues every
        # timed step ahead of it: per-step device times then never include host
        # enqueue latency, even on a slow or busy host
        torch.cuda._sleep(head_start_cycles(steps))
        h0 = time.perf_counter()
        for i in range(steps):
            flush.zero_()  # > L2 (126 MB): every timed launch starts cold
            starts[i].record(stream)
            G.spdm_gcoo_dev(dg, dB, dC, cfg, stream=stream)
            ends[i].record(stream)
        if not kernel_events:  # the timed pass (the kernel-timing pass creates CUDA events per call)
            time_kernel.host_enqueue_us = (time.perf_counter() - h0) / steps * 1e6
        torch.cuda.synchronize()
        launches = G.launch_count() - l0
        k_ms, k_n = G.kernel_time()
        G.kernel_timing(False)
        return [s.elapsed_time(e) for s, e in zip(starts, ends)], launches, k_ms / max(k_n, 1)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush.zero_()
            G.spdm_gcoo_dev(dg, dB, dC, cfg, stream=stream)
        torch.cuda.synchronize()
        times, launches, _ = run(False)
        _, _, kernel_ms = run(True)
    return sum(times) / len(times), min(times), launches, kernel_ms


class Dist:
    """The process group (NCCL when every rank has its own GPU, gloo for
    plumbing runs with more ranks than GPUs) and max-over-ranks reductions."""

    def __init__(self, world, rank, dev, ndev):
        import torch
        import torch.distributed as dist
        self.world, self.rank, self.dist = world, rank, dist
        self.backend = "nccl" if world <= ndev else "gloo"
        if world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=dev)
            else:
                dist.init_process_group("gloo")
        self.red_dev = dev if self.backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, *vals):
        import torch
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=self.red_dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    def broadcast_(self, t, src=0):
        """In-place broadcast of a device tensor (through the host under gloo)."""
        if self.world == 1:
            return t
        if self.backend == "nccl":
            self.dist.broadcast(t, src)
        else:
            h = t.cpu()
            self.dist.broadcast(h, src)
            t.copy_(h)
        return t


def strong_scaling(G, D, dev, stream, flush, steps, warmup, n=STRONG_N, s=0.99):
    """BASELINE configs[4]: n=32768, s=0.99, B/C column-sharded over the world,
    A replicated (built on rank 0, NCCL broadcast).  Returns the JSON block on
    rank 0 (None elsewhere)."""
    import torch
    from paper_2005_14469_b200.shard import column_shards, gather_columns
    world, rank = D.world, D.rank
    # ---- A: built once (rank 0, reference sample as COO, grouped on the GPU), broadcast
    if rank == 0:
        v, r, c = G.generate_uniform_sparse_coo(n, s, SEED)
        dg0 = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                torch.from_numpy(c).to(dev), P)
        del v, r, c
        nnz = dg0.nnz()
    else:
        dg0, nnz = None, 0
    nnz = int(D.broadcast_(torch.tensor([nnz], dtype=torch.int64, device=dev)).item())
    groups = -(-n // P)
    if rank == 0:
        arrays = [dg0.values, dg0.row_idx, dg0.col_idx, dg0.g_idxes, dg0.nnz_per_group]
    else:
        arrays = [torch.empty(nnz, dtype=torch.float32, device=dev), torch.empty(nnz, dtype=torch.int32, device=dev),
                  torch.empty(nnz, dtype=torch.int32, device=dev), torch.empty(groups, dtype=torch.int64, device=dev),
                  torch.empty(groups, dtype=torch.int64, device=dev)]
    D.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in arrays:
        D.broadcast_(t)
    e1.record()
    torch.cuda.synchronize()
    bcast_ms = D.max(e0.elapsed_time(e1))[0]
    dg = G.DeviceGcoo(n, n, P, *arrays)

    # ---- my shard of B/C
    shards = column_shards(n, world, align=BW)
    lo, hi = shards[rank]
    dB = synth_b_block(n, lo, hi, dev)
    dC = torch.empty((n, hi - lo), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    D.barrier()
    ms, ms_min, _, kms = time_kernel(G, dg, dB, dC, steps, warmup, stream, flush)
    D.barrier()
    t_n, t_n_min, k_n = D.max(ms, ms_min, kms)

    # ---- t_1: the whole product on rank 0, same run, same protocol
    sample_rows = torch.arange(0, n, 257, device=dev)  # 128 rows spread over every row block
    if rank == 0:
        if world == 1:
            t_1, k_1, full = ms, kms, dC
        else:
            dBf = synth_b_block(n, 0, n, dev)
            full = torch.empty((n, n), dtype=torch.float32, device=dev)
            t_1, _, _, k_1 = time_kernel(G, dg, dBf, full, steps, warmup, stream, flush)
            del dBf
        ref_rows = full[sample_rows].contiguous()
    # ---- parity: every shard's sampled rows against the 1-GPU product (gathered onto rank 0)
    mine = dC[sample_rows].contiguous()
    if world == 1:
        got = mine
    else:
        got = gather_columns(mine if D.backend == "nccl" else mine.cpu(), shards, root=0)
    parity = None
    if rank == 0:
        parity = bool(torch.equal(got.to(dev), ref_rows))
    # ---- the optional C gather (NCCL point to point onto rank 0), timed apart
    gather = None
    if world > 1:
        D.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        cfull = gather_columns(dC if D.backend == "nccl" else dC.cpu(), shards, root=0)
        g1.record()
        torch.cuda.synchronize()
        gms = D.max(g0.elapsed_time(g1))[0]
        if rank == 0:
            gather = {"ms": round(gms, 3), "bytes_to_root": int(n * (n - (hi - lo)) * 4),
                      "collective": f"{D.backend} point-to-point (batch_isend_irecv) onto rank 0",
                      "equals_1gpu": bool(torch.equal(cfull.to(dev), full))}
        del cfull
    if rank != 0:
        return None
    flops = 2.0 * nnz * n
    return {"workload": f"BASELINE configs[4]: n={n} s={s} uniform-random A (reference generator, seed {SEED}), "
                        f"B(i,j) = hash(i,j) in (0,1], B/C column-sharded over {world} GPU(s), A replicated",
            "nnz": nnz, "shards": [list(x) for x in shards],
            "t1_ms": round(t_1, 3), "t1_kernel_ms": round(k_1, 3),
            "tN_ms": round(t_n, 3), "tN_min_ms": round(t_n_min, 3), "tN_kernel_ms": round(k_n, 3),
            "speedup": round(t_1 / t_n, 3), "gflops_1": round(flops / t_1 / 1e6, 1),
            "gflops_N": round(flops / t_n / 1e6, 1), "scaling": "strong",
            "timing": "CUDA events per step on each rank's stream, L2 flushed, max over ranks; t1 on rank 0",
            "a_broadcast_ms": round(bcast_ms, 3), "parity_sampled_rows_equal_1gpu": parity,
            "c_gather": gather}


def run_ours(args):
    import torch
    import paper_2005_14469_b200 as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    ndev = torch.cuda.device_count()
    local = local % ndev  # more ranks than GPUs only for plumbing checks (gloo)
    torch.cuda.set_device(local)
    G.set_device(local)
    dev = torch.device("cuda", local)
    D = Dist(world, rank, dev, ndev)

    n, s = args.n, args.sparsity
    b_seed = G.derive_seed(SEED + rank, n, 0xB)  # rank 0: the reference's B
    a_host, b_host, dg, dB = make_inputs(G, n, s, SEED, dev, b_seed)
    nnz = dg.nnz()
    m = k = n
    dC = torch.empty((m, n), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB
    stream = torch.cuda.Stream(device=dev)

    # ---- kernel-only, device-resident ----------------------------------
    D.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ms_mean, ms_min, launches, kernel_ms = time_kernel(G, dg, dB, dC, args.steps, args.warmup, stream, flush)
        host_enqueue_us = getattr(time_kernel, "host_enqueue_us", None)
    torch.cuda.synchronize()
    D.barrier()
    ms_mean, ms_min, kernel_ms = D.max(ms_mean, ms_min, kernel_ms)
    flops_rank = 2.0 * nnz * n
    value = world * flops_rank / (ms_mean * 1e-3) / 1e9
    kernel_name = G.last_kernel()

    # C against the reference (rank 0's block is configs[1] exactly)
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
            torch.cuda._sleep(head_start_cycles(args.steps))
            for e0, e1 in evs:
                flush.zero_()
                e0.record(stream)
                plan.run(dB, dC, stream=stream)
                e1.record(stream)
            torch.cuda.synchronize()
        pms = D.max(sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs))[0]
        plan.close()
        plan_reuse = {"ms_per_step": round(pms, 4), "value": round(world * flops_rank / (pms * 1e-3) / 1e9, 2),
                      "unit": "GFLOPS", "note": "gcoo_plan_* (A's record stream built once, then one multiply "
                                                "kernel per B); not the headline, which plans every call"}
    except Exception as e:  # noqa: BLE001
        plan_reuse = {"error": str(e)[:200]}

    # ---- end to end through the public host API ----------------------
    g_host = dg.to_host()
    cfg = G.ExecConfig(p=P, b=BW)

    def pin(x):
        t_ = torch.empty(x.shape, dtype=getattr(torch, str(x.dtype)), pin_memory=True)
        t_.numpy()[...] = x
        return t_.numpy()

    def e2e_leg(g_in, b_in, c_out, calls):
        for _ in range(max(1, min(args.warmup, 3))):
            G.spdm_gcoo(g_in, b_in, cfg, out=c_out)
        D.barrier()
        # each call timed on its own (host clock around the whole API call: copies in,
        # multiply, copy out, synchronised); the median is robust to host hiccups
        ts = []
        for _ in range(calls):
            t0 = time.perf_counter()
            G.spdm_gcoo(g_in, b_in, cfg, out=c_out)
            ts.append(time.perf_counter() - t0)
        return D.max(statistics.median(ts))[0], ts

    g_pin = G.GcooMatrix(g_host.rows_dim, g_host.cols_dim, g_host.p, pin(g_host.values), pin(g_host.row_idx),
                         pin(g_host.col_idx), pin(g_host.g_idxes), pin(g_host.nnz_per_group))
    e2e_s, e2e_times = e2e_leg(g_pin, pin(b_host), pin(np.empty((m, n), np.float32)), max(5, min(args.steps, 20)))
    e2e_value = world * flops_rank / e2e_s / 1e9
    try:
        pcie_peak = pcie_duplex_probe(dev)
    except Exception:  # noqa: BLE001
        pcie_peak = None
    # pageable buffers (the C++ drop-in's std::vector path)
    c_page = np.empty((m, n), np.float32)
    pg_s, pg_times = e2e_leg(g_host, b_host, c_page, 5)
    h2d = g_host.values.nbytes + g_host.row_idx.nbytes + g_host.col_idx.nbytes + g_host.g_idxes.nbytes + \
        g_host.nnz_per_group.nbytes + b_host.nbytes
    d2h = m * n * 4

    # ---- GCOO construction (EO): dense A resident on the device
    # grouped by the K3 kernels; each call returns nnz to the host (one sync)
    construction = None
    if rank == 0:
        dA = torch.from_numpy(a_host).to(dev)
        for _ in range(3):
            G.dense_to_gcoo_dev(dA, P, stream=stream)
        torch.cuda.synchronize()
        ets = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            G.dense_to_gcoo_dev(dA, P, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ets.append(e0.elapsed_time(e1))
        eo_ms = statistics.median(ets)
        construction = {"eo_ms": round(eo_ms, 4), "dense_bytes": int(a_host.nbytes),
                        "dense_gb_s_per_call": round(a_host.nbytes / (eo_ms * 1e-3) / 1e9, 1),
                        "what": "dense_to_gcoo on the device (count, scan, fill; nnz read back), L2 flushed, "
                                "median of 10; the reference's EO (TimingBreakdown.eo_seconds)"}
        del dA

    # ---- roofline (BASELINE §4: FP32-bound at s <= 0.994, HBM-bound above) ----
    hbm_peak, hbm_src = peaks()
    fp_peak, fp_src = fp32_peak_tflops()
    k_nz = int(np.count_nonzero(np.bincount(g_host.col_idx, minlength=k)))
    cb = compulsory_bytes(nnz, m, k, n, P, k_nz)
    oi = flops_rank / cb
    achieved_gbs = cb / (kernel_ms * 1e-3) / 1e9  # dominant kernel: the multiply, event-timed
    tflops = flops_rank / (kernel_ms * 1e-3) / 1e12
    roof_tflops = min(fp_peak, oi * hbm_peak / 1e3)
    fp32_bound = fp_peak <= oi * hbm_peak / 1e3
    nc = ncu_summary(n, s, kernel_name)
    traffic = None if nc is None else int(nc["dram_read_bytes"] + nc["dram_write_bytes"])
    roofline = {"bound": "fp32" if fp32_bound else "hbm",
                "achieved": round(tflops if fp32_bound else achieved_gbs, 3 if fp32_bound else 1),
                "peak": round(fp_peak, 2) if fp32_bound else hbm_peak,
                "unit": "TFLOP/s" if fp32_bound else "GB/s",
                "frac": round(tflops / fp_peak if fp32_bound else achieved_gbs / hbm_peak, 4),
                "traffic": traffic, "peak_source": fp_src if fp32_bound else hbm_src,
                "kernel": kernel_name, "kernel_ms": round(kernel_ms, 4),
                "kernel_share_of_step": round(kernel_ms / ms_mean, 3),
                "operational_intensity": round(oi, 2),
                "baseline_achieved": round(tflops / roof_tflops, 4),
                "baseline_achieved_def": "(2*nnz*N/t) / min(P_fp32, OI*BW) (BASELINE.md §4)",
                "traffic_source": None if nc is None else nc["_source"]}
    roofline_hbm = {"achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved_gbs / hbm_peak, 4), "peak_source": hbm_src,
                    "algorithmic_bytes_per_launch": int(cb),
                    "bytes_formula": "12*nnz + 16*ceil(m/p) + 4*k_nz*N + 4*m*N (SURVEY 8d)"}
    # the paper's argument, measured: where the multiply's bytes move (ncu --set full)
    traffic_split = None
    if nc is not None:
        traffic_split = {"dram_bytes": traffic, "l2_to_sm_bytes": int(nc["l2_read_bytes_from_sm"]),
                         "shared_memory_bytes": int(nc["smem_wavefronts"] * 128),
                         "shared_memory_busy_frac": round(nc["smem_wavefront_pct"] / 100, 3),
                         "source": nc["_source"] + " (LSU wavefronts x 128 B)"}

    extra = {}
    if rank == 0 and world == 1 and not args.no_sweep:
        for s2 in (0.9, 0.995):
            _, _, dg2, _ = make_inputs(G, n, s2, SEED, dev, b_seed)
            ms2, _, _, kms2 = time_kernel(G, dg2, dB, dC, max(3, args.steps // 2), 3, stream, flush)
            f2 = 2.0 * dg2.nnz() * n
            cb2 = compulsory_bytes(dg2.nnz(), m, k, n, P, k)
            extra[f"s{s2}"] = {"nnz": dg2.nnz(), "ms": round(ms2, 4), "kernel_ms": round(kms2, 4),
                               "kernel": G.last_kernel(), "gflops": round(f2 / ms2 / 1e6, 1),
                               "hbm_frac": round(cb2 / (kms2 * 1e-3) / 1e9 / hbm_peak, 4),
                               "fp32_frac": round(f2 / (kms2 * 1e-3) / 1e12 / fp_peak, 4)}
            del dg2
        extra.update(powerlaw_config(G, dev, stream, flush, hbm_peak, fp_peak))

    strong = None
    if not args.no_strong:
        del dB, dC
        torch.cuda.empty_cache()
        strong = strong_scaling(G, D, dev, stream, flush, steps=max(3, min(args.steps, 8)), warmup=3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g_host, b_host, n)

    if world > 1:
        D.barrier()
        D.dist.destroy_process_group()
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
        "config": workload_config(n, s, nnz),
        "layout": {"parallelism": f"column-shard B/C x{world}, A replicated (rank r owns columns "
                                  f"[r*{n}, (r+1)*{n}) of a {n}x{n * world} B/C; no data-path collective)",
                   "dist_backend": D.backend if world > 1 else None},
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOPS", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_s * 1e3, 3),
                "ms_per_step_mean": round(statistics.mean(e2e_times) * 1e3, 3), "calls": len(e2e_times),
                "path": "paper_2005_14469_b200.spdm_gcoo -> gcoo_spdm_f32 (pinned host buffers)",
                **pcie_roofline(h2d + d2h, e2e_s, pcie_peak)},
        "construction": construction,
        "e2e_pageable": {"value": round(world * flops_rank / pg_s / 1e9, 2), "unit": "GFLOPS",
                         "ms_per_step": round(pg_s * 1e3, 3), "calls": len(pg_times),
                         "path": "spdm_gcoo -> gcoo_spdm_f32 with pageable numpy buffers "
                                 "(what a C++ std::vector caller of the drop-in headers passes)"},
        "gpu_launches": int(launches),
        "host_enqueue_us_per_step": None if host_enqueue_us is None else round(host_enqueue_us, 1),
        "plan_reuse": plan_reuse,
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "traffic_split": traffic_split,
        "clocks": clk.summary(),
        "parity": parity,
        "strong_n32768": strong,
        "sweep": extra,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def ncu_summary(n, s, kernel):
    """The newest `ncu --set full` summary of this configuration's multiply
    (profiles/r0X_ncu_*_s{s}.json written by tools/ncu_summary.py)."""
    for name in (f"r02_ncu_{kernel}_s{s}.json", f"r01_ncu_tacc28_s{s}.json"):
        path = os.path.join(ROOT, "profiles", name)
        if n == 8000 and os.path.exists(path):
            try:
                with open(path) as f:
                    d = json.load(f)
                d["_source"] = f"ncu --set full, profiles/{name}"
                return d
            except Exception:  # noqa: BLE001
                pass
    return None


def powerlaw_config(G, dev, stream, flush, hbm_peak, fp_peak, steps=5):
    """BASELINE configs[3]: power-law A (this repo's generator, n=16384,
    s=0.99) as COO, grouped on the GPU; B uniform (0,1] generated on the device
    (its values do not change the work)."""
    import torch
    out = {}
    name, n = "powerlaw_n16384_s0.99", 16384
    try:
        v, r, c = G.generate_powerlaw_coo(n, 0.99, 1.0, SEED)
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
                     "kernel_ms": round(kms, 4), "kernel": G.last_kernel(), "two_class_split": G.last_split(),
                     "gflops": round(f / ms / 1e6, 1), "kernel_gflops": round(f / kms / 1e6, 1),
                     "compulsory_bytes": int(cb),
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
        out = {"value": round(2.0 * g.nnz * n / kc / 1e9, 3), "unit": "GFLOPS", "cores": int(r["workers"]),
               "kind": "reference",
               "sample": f"full workload (n={n}, nnz={g.nnz}): reference spdm_gcoo, median of 3 after 1 warmup, "
                         f"OpenMP {r['workers']} threads, default-ISA build (as shipped, mul+add)",
               "kc_seconds": kc, **cpu_description()}
        try:  # BASELINE.md §3's optional second row: the FMA-contracted build (the GPU's exact bits)
            rf = Reference(True).time_spdm(g, b_host, b=BW, workers=cores, warmup=1, reps=3)
            out["fma_build"] = {"value": round(2.0 * g.nnz * n / rf["kc_s"] / 1e9, 3), "unit": "GFLOPS",
                                "kc_seconds": rf["kc_s"], "build": "-mfma (FMA contraction), same sources"}
        except Exception as e:  # noqa: BLE001
            out["fma_build"] = {"error": str(e)[:120]}
        return out
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
        "config": workload_config(n, s, g.nnz),
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOPS", "cores": int(r["workers"]), "kind": "reference",
                         "sample": f"full workload each step: reference spdm_gcoo (median of {max(1, args.steps)}),"
                                   f" OpenMP {r['workers']} threads of {cores}, default-ISA build (as shipped)",
                         **cpu_description()},
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
    ap.add_argument("--no-strong", action="store_true")
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
