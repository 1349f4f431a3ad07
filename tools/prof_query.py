"""Profiling driver: build a bench workload, then run one query configuration
between cudaProfilerStart/Stop (for `ncu --profile-from-start off`).

    python tools/prof_query.py --path ivf --L 64 [--subset 0.1] [--workload deep10m]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="deep10m")
    ap.add_argument("--path", default="ivf")
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--subset", type=float, default=0.0)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--counters", action="store_true", help="print the scan kernels' debug counters of one call")
    a = ap.parse_args()
    kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda", 0)
    g = rii.Index(D, M, device=0)
    g.train(bench._device_data(kind, n_train, D, dev, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
    x = bench._device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
    g.add(x)
    del x
    g.reconfigure(nlist, n_iter=10, seed=0)
    q = bench._device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
    S = gen.subset_torch(N, int(N * a.subset), dev, seed=0) if a.subset > 0 else None
    for _ in range(2):
        g.query(q, topk, S, L=a.L, path=a.path)
    torch.cuda.synchronize()
    lib = rii.load()
    lib.rii_kernel_timing(1)
    t0 = time.perf_counter()
    torch.cuda.profiler.start()
    for _ in range(a.reps):
        _, _, used = g.query(q, topk, S, L=a.L, path=a.path)
    torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / a.reps
    import ctypes as C
    out = {}
    for w, name in ((0, "linear"), (1, "ivf"), (2, "merge")):
        ms, n = C.c_double(), C.c_int64()
        lib.rii_kernel_timing_read(w, C.byref(ms), C.byref(n))
        out[name] = (ms.value / max(a.reps, 1), n.value)
    print(f"path={a.path} used={used} L={a.L} subset={a.subset} wall_ms={dt * 1e3:.2f} qps={nq / dt:.0f} kernels={out}")
    if a.counters:
        rii.debug_counters(True)
        g.query(q, topk, S, L=a.L, path=a.path)
        print("counters", rii.read_debug_counters())
        rii.debug_counters(False)


if __name__ == "__main__":
    main()
