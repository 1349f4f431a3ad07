#!/usr/bin/env python
"""bench.py -- the Rii hot path (arXiv 1808.03969) on B200: queries/s and scanned
PQ codes/s of the ADC scan + top-k, against its roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload deep10m|sift1m|tiny] [--no-extra]

N > 1 is launched with torchrun (one rank per GPU, NCCL).  A step is one
rii_query call over the whole query batch of the workload (Alg. 1 over the
whole database, 10,000 queries, top-100; BASELINE.json configs[2]) with inputs
resident in HBM; `e2e` repeats it through the same C-ABI call with pinned host
buffers (H2D of the queries and D2H of the results inside the timed region).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same
workload instead.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth import generators as gen  # noqa: E402

METRIC = "queries/sec & scanned PQ codes/sec (ADC+top-k) vs HBM roofline, 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024
SMS = 148
LUT_LOOKUPS_PER_CLK_PER_SM = 32  # one conflict-free LDS.32 wavefront (128 B) per clock per SM


def _source_hash():
    """sha256[:16] of the scan kernel's sources (k_scan.cu, lut.cuh, topk.cuh,
    kernels.cuh, common.cuh): ties a committed ncu traffic number to the code it
    was measured on (the GPU box has no .git)."""
    import hashlib
    h = hashlib.sha256()
    for f in ("k_scan.cu", "lut.cuh", "topk.cuh", "kernels.cuh", "common.cuh"):
        with open(os.path.join(ROOT, "paper_1808_03969_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count()
    return {"nproc": n, "cpu_model": model}


def _traffic(kernel_kind):
    """DRAM bytes per launch of the headline kernel from the committed ncu --set full
    capture (profiles/scan_traffic.json), with its provenance; null when the capture
    was taken on other kernel sources than the ones this run built."""
    tp = os.path.join(ROOT, "profiles", "scan_traffic.json")
    if not os.path.exists(tp):
        return None, {"file": None}
    with open(tp) as f:
        d = json.load(f)
    src = _source_hash()
    prov = {"file": "profiles/scan_traffic.json", "captured_on_source": d.get("source_sha16"),
            "this_source": src, "commit": d.get("commit"), "capture": d.get("source"), "kernel": d.get("kernel")}
    if d.get("source_sha16") != src or d.get("kernel_kind") != kernel_kind:
        return None, dict(prov, note="capture does not match the built kernel sources: traffic unmeasured")
    return d.get("dram_bytes_per_launch"), prov


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


WORKLOADS = {
    # name: (generator kind, N, D, M, nlist, nq, topk, n_train, config label)
    "deep10m": ("deep", 10_000_000, 96, 32, 3162, 10_000, 100, 100_000,
                "BASELINE.json configs[2]: Deep1B-like 10M x 96, M=32, nlist=3162, 10k queries, top-100"),
    "sift1m": ("sift", 1_000_000, 128, 16, 1000, 10_000, 100, 100_000,
               "BASELINE.json configs[1]: SIFT1M-like 1M x 128, M=16, nlist=1000, 10k queries, top-100"),
    # the paper's own SIFT1M setting (Table 2: K = 1000, M = 64); not a BASELINE.json config
    "sift1m_m64": ("sift", 1_000_000, 128, 64, 1000, 10_000, 100, 100_000,
                   "paper Table 2 shape: SIFT1M-like 1M x 128, M=64, nlist=1000, 10k queries, top-100"),
    # the paper's GIST1M setting (Table 2: K = 1000, M = 240, L = 8000 candidates)
    "gist1m": ("deep", 1_000_000, 960, 240, 1000, 10_000, 100, 100_000,
               "paper Table 2 shape: GIST1M-like 1M x 960, M=240, nlist=1000, 10k queries, top-100"),
    # configs[4]'s code shape (M = 8) at configs[2]'s size, for A/B of the M = 8 kernels
    "deep10m_m8": ("deep", 10_000_000, 96, 8, 3162, 10_000, 100, 100_000,
                   "configs[4] shape at 10M: Deep1B-like 10M x 96, M=8, nlist=3162, 10k queries, top-100"),
    # configs[4]'s shape (M = 8, nlist = 31,623, 1,024-query batches) at 1e8 codes, for A/B runs
    "deep100m_m8": ("deep", 100_000_000, 96, 8, 31623, 1024, 100, 100_000,
                    "configs[4] shape at 1e8: Deep1B-like 1e8 x 96, M=8, nlist=31623, 1024 queries, top-100"),
    "tiny": ("gaussian", 10_000, 32, 4, 100, 100, 10, 10_000,
             "BASELINE.json configs[0]: N(0,1) 10k x 32, M=4, nlist=100, 100 queries, top-10"),
}


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during a region."""
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms",
                 "200", "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=5)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- dist utils --
def _dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return rank, world, local


def _max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------- our arm ------
def _device_data(kind, n, D, device, seed, stream):
    if kind == "deep":
        return gen.deep_like_torch(n, device, D=D, seed=seed, stream=stream)
    if kind == "sift":
        return gen.sift_like_torch(n, device, D=D, seed=seed, stream=stream)
    import torch
    g = torch.Generator(device=device)
    g.manual_seed((seed << 8) | stream)
    return torch.randn((n, D), generator=g, device=device)


def _timed_steps(step, K, stream, flush=None):
    """K steps, CUDA events on `stream` around each step (flush outside)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        if flush is not None:
            flush()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def run_ours(args, rank, world, local):
    import torch

    import paper_1808_03969_b200 as rii
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    kind, N, D, M, nlist, nq, topk, n_train, label = WORKLOADS[args.workload]
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [rii.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    # ---- build the index (not timed as the metric; reported under "build") ----
    build = {}
    t0 = time.perf_counter()
    xt = _device_data(kind, n_train, D, dev, 0, gen.STREAM_TRAIN)
    g = rii.Index(D, M, device=local, rank=rank, world=world, nccl_id=nccl_id)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g.train(xt, n_iter=20, seed=0)
    torch.cuda.synchronize()
    build["train_s"] = time.perf_counter() - t1
    del xt
    x = _device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g.add(x)
    torch.cuda.synchronize()
    build["add_s"] = time.perf_counter() - t1
    del x
    torch.cuda.empty_cache()
    t1 = time.perf_counter()
    g.reconfigure(nlist, n_iter=10, seed=0)
    torch.cuda.synchronize()
    build["reconfigure_s"] = time.perf_counter() - t1
    build["total_s"] = time.perf_counter() - t0
    q = _device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
    # theta (Alg. 3's linear / inverted-index switch) is fitted by timing both paths
    # on this GPU, as the paper does on its CPU; AUTO rows below use it
    t1 = time.perf_counter()
    th = g.calibrate_theta(q[:1000], topk=topk, L_grid=(1, 4, 16, 64))
    torch.cuda.synchronize()
    build["theta_calibration_s"] = time.perf_counter() - t1
    build["theta_fit"] = {"a": th[0], "b": th[1], "crossovers_at_L_1_4_16_64": [float(v) for v in th[2]]}
    info = g.info()
    stream = torch.cuda.current_stream()
    ids = torch.empty((nq, topk), dtype=torch.int64, device=dev)
    dist_ = torch.empty((nq, topk), dtype=torch.float32, device=dev)
    n_local = info["n_local"]
    flush_buf = None
    if n_local * M < 2 * L2_BYTES:  # shard fits in L2: flush it between steps
        flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)

    def flush():
        if flush_buf is not None:
            flush_buf.fill_(1.0)

    def step():
        g.query(q, topk, None, L=64, path="linear", out=(ids, dist_))

    # ---- headline: whole-database PQ linear scan, inputs resident in HBM ----
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    rii_lib = rii.load()
    _barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    rii_lib.rii_kernel_timing(1)
    l0 = rii.launch_count()
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly the timed steps
    step_ms = _timed_steps(step, args.steps, stream, flush if flush_buf is not None else None)
    torch.cuda.profiler.stop()
    launches = rii.launch_count() - l0
    import ctypes as C
    kms, kn = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(0, C.byref(kms), C.byref(kn))
    mms, mn = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(2, C.byref(mms), C.byref(mn))
    pms, pn = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(3, C.byref(pms), C.byref(pn))
    bms, bn = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(4, C.byref(bms), C.byref(bn))
    qms, qn16 = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(5, C.byref(qms), C.byref(qn16))
    q16 = qn16.value > 0 and qn16.value == kn.value
    ums, un6 = C.c_double(), C.c_int64()
    rii_lib.rii_kernel_timing_read(6, C.byref(ums), C.byref(un6))
    u6 = un6.value > 0 and un6.value == kn.value
    packed = u6 or q16 or (pn.value > 0 and pn.value == kn.value)
    rii_lib.rii_kernel_timing(0)
    torch.cuda.synchronize()
    _barrier(world)
    clk = clocks.stop()
    total_ms = _max_over_ranks(sum(step_ms), world)
    kernel_ms = _max_over_ranks(kms.value / max(kn.value, 1), world)
    merge_ms = _max_over_ranks(mms.value / max(mn.value, 1), world)
    bound_ms = _max_over_ranks(bms.value / max(bn.value, 1), world)
    qps = nq * args.steps / (total_ms / 1e3)

    peaks, peak_src = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    # one 128-B shared-memory wavefront per clock per SM: 32 fp32 lookups, or 64
    # lookups with the bf16-packed or u16 fixed-point tables (2 B per lookup)
    per_clk = LUT_LOOKUPS_PER_CLK_PER_SM * (4 if u6 else 2 if packed else 1)
    lut_peak = SMS * per_clk * sm_max * 1e6  # lookups/s
    lookups = nq * n_local * M
    achieved = lookups / (kernel_ms / 1e3)
    traffic, traffic_src = _traffic("u6" if u6 else "u16" if q16 else "packed" if packed else "fp32")
    roofline = {
        "bound": "alu",
        "kernel": (f"scan_fast_kernel<32,{16 if os.environ.get('RII_Q16_CFG', '9') == '9' else 8},u6> (linear ADC "
                   "scan + top-k, u6 fixed-point oct tables, bytewise SWAR sums + exact rescore)" if u6 else
                   "scan_fast_kernel<32,8,u16> (linear ADC scan + top-k, u16 fixed-point SWAR tables + exact rescore)"
                   if q16 else
                   "scan_fast_kernel<32,8,packed> (linear ADC scan + top-k, bf16-packed tables + exact rescore)"
                   if packed else "scan_fast_kernel<32,6> (linear ADC scan + top-k, fp32 tables)"),
        "achieved": achieved / 1e9, "peak": lut_peak / 1e9, "unit": "Glookup/s",
        "frac": achieved / lut_peak, "traffic": traffic, "traffic_provenance": traffic_src,
        "peak_basis": f"shared-memory LUT pipe: one 128-B wavefront/clk/SM = {per_clk} "
                      f"{'u6 (1 B)' if u6 else 'u16 (2 B)' if q16 else 'bf16-packed (2 B)' if packed else 'fp32 (4 B)'} "
                      f"lookups/clk/SM x {SMS} SMs x "
                      f"{sm_max:.0f} MHz (sm_max_mhz, {peak_src})",
        "algorithmic_units": f"{nq} queries x {n_local} codes x {M} lookups per launch",
        "kernel_ms_per_launch": kernel_ms, "kernel_share_of_step": kernel_ms / (total_ms / args.steps),
        "merge_ms_per_launch": merge_ms,
        "bound_pass_ms_per_step": bound_ms if bn.value else None,
        "hbm_equiv": {"code_bytes_per_s": achieved, "of_measured_hbm": achieved / (float(peaks["hbm_gbs"]) * 1e9),
                      "hbm_gbs": float(peaks["hbm_gbs"]),
                      "note": "north_star's 'fraction of HBM on code bytes': Q*N*M effective code bytes/s over the "
                              "measured copy bandwidth; codes are reused from registers across the CTA's queries"},
    }

    # ---- e2e: same call through the C ABI with pinned host buffers ----
    qh = q.cpu().pin_memory()
    ih = torch.empty((nq, topk), dtype=torch.int64).pin_memory()
    dh = torch.empty((nq, topk), dtype=torch.float32).pin_memory()
    qn, in_, dn = qh.numpy(), ih.numpy(), dh.numpy()

    def step_host():
        g.query(qn, topk, None, L=64, path="linear", out=(in_, dn))

    step_host()
    e2e_ms = _max_over_ranks(sum(_timed_steps(step_host, args.steps, stream,
                                              flush if flush_buf is not None else None)), world)
    e2e = {"value": nq * args.steps / (e2e_ms / 1e3), "unit": "queries/s", "h2d_bytes_per_step": nq * D * 4,
           "d2h_bytes_per_step": nq * topk * (8 + 4), "api": "rii_query(RII_MEM_HOST) via paper_1808_03969_b200.Index"}

    # ---- other rows of the path (IVF probe counts, subsets), shorter runs ----
    paths = {}
    if not args.no_extra:
        def meas(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            ms = _max_over_ranks(sum(_timed_steps(fn, reps, stream, flush if flush_buf is not None else None)), world)
            return nq * reps / (ms / 1e3)

        for L in (1, 4, 16, 64):
            used = {}

            def f(L=L):
                used["p"] = g.query(q, topk, None, L=L, path="auto", out=(ids, dist_))[2]
            v = meas(f)
            paths[f"whole_ivf_L{L}"] = {"qps": v, "path_used": ["auto", "linear", "ivf"][used["p"]],
                                        "scanned_codes_per_query_approx": L * N / nlist}
        for frac in (0.01, 0.1):
            S = gen.subset_torch(N, int(N * frac), dev, seed=0)
            for pth in ("auto", "linear", "ivf"):
                used = {}

                def f(S=S, pth=pth):
                    used["p"] = g.query(q, topk, S, L=64, path=pth, out=(ids, dist_))[2]
                v = meas(f, reps=2)
                paths[f"subset{int(frac * 100)}pct_{pth}"] = {"qps": v,
                                                              "path_used": ["auto", "linear", "ivf"][used["p"]]}

    # ---- oracle on the host (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.workload)

    if rank == 0:
        line = {
            "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {label}", "N": N, "D": D, "M": M, "nlist": nlist, "nq": nq,
                       "topk": topk, "path": "linear (Alg. 1, S = whole database)",
                       "l2": ("flushed between steps (shard fits in L2)" if flush_buf is not None
                              else f"codes {n_local * M / 2**20:.0f} MiB per GPU > 126 MB L2"),
                       "parallelism": f"id-range shards x{world}"},
            "scanned_codes_per_s": qps * N,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "paths": paths,
            "build": build,
            "index": info,
        }
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------- oracle (CPU) ---
_SAMPLE_N = 100_000


def _oracle_sample(workload):
    """A bounded sample of the workload built by the oracle alone: 100k database
    vectors from the same generator, code book trained on 10k of them (5 iters)."""
    from oracle import ref
    kind, N, D, M, nlist, nq, topk, n_train, label = WORKLOADS[workload]
    n = min(N, _SAMPLE_N)
    x = gen.base(kind, n, D, seed=0)
    idx = ref.OracleIndex(D, M)
    idx.train(x[: min(n, 10_000)], n_iter=5, seed=0)
    idx.add(x)
    q = gen.base(kind, 256, D, seed=0, stream=gen.STREAM_QUERY)
    return ref, idx, q, n


def cpu_baseline(workload, budget_s=8.0):
    """The oracle as it stands, timed twice on this host: one thread (the paper's
    protocol) and every core (queries split over threads, each running the
    single-threaded C oracle; SURVEY 8(d) "two numbers").  `value` is the all-cores
    number."""
    ref, idx, q, n = _oracle_sample(workload)
    kind, N, D, M, nlist, nq, topk, n_train, label = WORKLOADS[workload]
    host = _host_info()
    threads = ref.cores()

    def run(nthreads, batch):
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s:
            s = done % len(q)
            ref.linear_mt(idx.cb, idx.codes, q[s:s + batch], topk, threads=nthreads)
            done += batch
        return done / (time.perf_counter() - t0)

    qps1 = run(1, 8)
    qpsn = run(threads, 4 * threads)
    return {"value": qpsn * n / N, "unit": "queries/s", "cores": threads, "kind": "oracle",
            "sample": f"Alg. 1 (whole scan, top-{topk}) over {n} codes drawn with the workload's generator "
                      f"(oracle-built index), {budget_s:.0f} s per measurement; queries/s scaled by {n}/{N} to the "
                      f"full database (cost O(M N), Table 1); value = all {threads} threads (queries split over "
                      f"threads), single_thread = the paper's one-thread protocol (P:757)",
            "single_thread": qps1 * n / N, "measured_qps_on_sample": qpsn, "host": host}


def run_reference(args, rank, world):
    if rank != 0:
        return
    ref, idx, q, n = _oracle_sample(args.workload)
    kind, N, D, M, nlist, nq, topk, n_train, label = WORKLOADS[args.workload]
    threads = ref.cores()
    per_step = 4 * threads

    def step(i):
        s = (i * per_step) % len(q)
        ref.linear_mt(idx.cb, idx.codes, q[s:s + per_step], topk, threads=threads)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt * n / N
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {label}", "N": N, "D": D, "M": M, "nq": nq, "topk": topk,
                       "path": "linear (Alg. 1, S = whole database)"},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": threads, "kind": "oracle",
                             "sample": f"each step {per_step} queries of Alg. 1 over {n} oracle-built codes of the "
                                       f"workload's generator, split over {threads} threads (the single-threaded "
                                       f"C oracle per slice), scaled by {n}/{N} (cost O(M N))",
                             "host": _host_info()},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="deep10m")
    ap.add_argument("--no-extra", action="store_true", help="skip the IVF / subset rows")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    rank, world, local = _dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
