"""Measure the other BASELINE.json configs on one GPU and print
one JSON line per row.  Timing: CUDA events on the launching stream, >= 1 warm-up,
queries resident in HBM, median of `reps` runs.

    python tools/configs.py [--only tiny,sift1m,growth,deep10m,paper_t2] [--reps 3]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402

DEV = torch.device("cuda", 0)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def rows_for(name, g, q, topk, Ls, subsets, N, nlist, reps):
    nq = q.shape[0]
    ms = timed(lambda: g.query(q, topk, None, L=1, path="linear"), reps)
    emit(config=name, row="linear whole", N=N, nq=nq, topk=topk, ms=ms, qps=nq / ms * 1e3,
         scanned_codes_per_s=nq * N / ms * 1e3)
    for L in Ls:
        ms = timed(lambda: g.query(q, topk, None, L=L, path="ivf"), reps)
        emit(config=name, row=f"ivf whole L={L}", N=N, nq=nq, topk=topk, ms=ms, qps=nq / ms * 1e3,
             approx_candidates_per_query=L * N / nlist)
    for s in subsets:
        S = gen.subset_torch(N, s, DEV, seed=s)
        for L in Ls[-1:]:
            for path in ("auto", "linear", "ivf"):
                used = {}

                def f():
                    used["p"] = g.query(q, topk, S, L=L, path=path)[2]
                ms = timed(f, reps)
                emit(config=name, row=f"subset |S|={s} L={L} {path}", path_used=["auto", "linear", "ivf"][used["p"]],
                     ms=ms, qps=nq / ms * 1e3)


def build(kind, N, D, M, nlist, n_train, train_iter=20):
    g = rii.Index(D, M, device=0)
    t0 = time.perf_counter()
    g.train(bench._device_data(kind, n_train, D, DEV, 0, gen.STREAM_TRAIN), n_iter=train_iter, seed=0)
    torch.cuda.synchronize()
    t_train = time.perf_counter() - t0
    x = bench._device_data(kind, N, D, DEV, 0, gen.STREAM_BASE)
    t0 = time.perf_counter()
    g.add(x)
    torch.cuda.synchronize()
    t_add = time.perf_counter() - t0
    del x
    t0 = time.perf_counter()
    g.reconfigure(nlist, n_iter=10, seed=0)
    torch.cuda.synchronize()
    t_rec = time.perf_counter() - t0
    return g, dict(train_s=t_train, add_s=t_add, reconfigure_s=t_rec)


def paper_table2_rows(reps):
    """The paper's own Table 2 shapes on synthetic stand-ins:
    SIFT1M-like with M = 64 and GIST1M-like with M = 240, K = 1000, IVF with L lists
    ~ the paper's L candidates (5000 -> 5 lists, 8000 -> 8 lists), top-1 and top-100,
    plus the whole linear scan.  The paper: 0.73 ms and 3.2 ms per query, one CPU thread."""
    for name, Lp in (("sift1m_m64", 5), ("gist1m", 8)):
        kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS[name]
        g, b = build(kind, N, D, M, nlist, n_train)
        emit(config=name, row="build", **b)
        q = bench._device_data(kind, nq, D, DEV, 0, gen.STREAM_QUERY)
        for k in (1, 100):
            ms = timed(lambda: g.query(q, k, None, L=Lp, path="ivf"), reps)
            emit(config=name, row=f"ivf whole L={Lp} top-{k}", N=N, nq=nq, topk=k, ms=ms, qps=nq / ms * 1e3,
                 ms_per_query=ms / nq)
        ms = timed(lambda: g.query(q, 100, None, L=1, path="linear"), reps)
        emit(config=name, row="linear whole top-100", N=N, nq=nq, topk=100, ms=ms, qps=nq / ms * 1e3,
             scanned_codes_per_s=nq * N / ms * 1e3)
        del g
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="tiny,sift1m,growth")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    only = a.only.split(",")
    if "paper_t2" in only:
        paper_table2_rows(a.reps)
    if "tiny" in only:
        c = gen.CONFIGS["tiny"]
        g, b = build("gaussian", c["N"], c["D"], c["M"], c["nlist"], c["N"])
        emit(config="tiny", row="build", **b)
        q = bench._device_data("gaussian", c["nq"], c["D"], DEV, 0, gen.STREAM_QUERY)
        rows_for("tiny", g, q, 10, [8], [1000], c["N"], c["nlist"], a.reps)
    if "sift1m" in only:
        c = gen.CONFIGS["sift1m"]
        g, b = build("sift", c["N"], c["D"], c["M"], c["nlist"], c["n_train"])
        emit(config="sift1m", row="build", **b)
        q = bench._device_data("sift", c["nq"], c["D"], DEV, 0, gen.STREAM_QUERY)
        th = g.calibrate_theta(q[:1000], topk=100, L_grid=(1, 4, 16, 64))
        emit(config="sift1m", row="theta calibration", a=th[0], b=th[1], crossovers=th[2].tolist())
        rows_for("sift1m", g, q, 100, [1, 4, 16, 64], c["subsets"], c["N"], c["nlist"], a.reps)
    if "growth" in only:  # configs[3]: start 10k, nlist 100, add 9 x 1,111,111, reconfigure to sqrt(N)
        c = gen.CONFIGS["growth"]
        D, M = c["D"], c["M"]
        g = rii.Index(D, M, device=0)
        g.train(bench._device_data("sift", c["n_train"], D, DEV, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
        x0 = bench._device_data("sift", c["N"], D, DEV, 0, gen.STREAM_BASE)
        g.add(x0)
        g.reconfigure(c["nlist"], n_iter=10, seed=0)
        q = bench._device_data("sift", c["nq"], D, DEV, 0, gen.STREAM_QUERY)
        for i in range(c["add_batches"]):
            xb = bench._device_data("sift", c["add_size"], D, DEV, 1 + i, gen.STREAM_BASE)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.add(xb)
            torch.cuda.synchronize()
            emit(config="growth", row=f"add batch {i}", n=c["add_size"], add_s=time.perf_counter() - t0,
                 N=g.info()["N"])
        N = g.info()["N"]
        for L in c["L"]:
            ms = timed(lambda: g.query(q, c["topk"], None, L=L, path="ivf"), a.reps)
            emit(config="growth", row=f"before reconfigure ivf L={L}", K=g.info()["K"], ms=ms, qps=c["nq"] / ms * 1e3)
        K2 = gen.nlist_for(N)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.reconfigure(K2, n_iter=10, seed=0)
        torch.cuda.synchronize()
        emit(config="growth", row="reconfigure", N=N, nlist=K2, reconfigure_s=time.perf_counter() - t0)
        for L in c["L"]:
            ms = timed(lambda: g.query(q, c["topk"], None, L=L, path="ivf"), a.reps)
            emit(config="growth", row=f"after reconfigure ivf L={L}", K=K2, ms=ms, qps=c["nq"] / ms * 1e3)
    if "scale1b" in only:  # configs[4] on ONE B200 (8 GB of codes fit): 1e9 x 96 unit-norm mixture, M=8
        c = gen.CONFIGS["scale1b"]
        N, D, M, K = c["N"], c["D"], c["M"], c["nlist"]
        g = rii.Index(D, M, device=0)
        t0 = time.perf_counter()
        g.train(bench._device_data("deep", c["n_train"], D, DEV, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
        torch.cuda.synchronize()
        emit(config="scale1b", row="train", n=c["n_train"], train_s=time.perf_counter() - t0)
        chunk = 1 << 24
        t0 = time.perf_counter()
        for s0 in range(0, N, chunk):  # streamed: the raw vectors are never stored
            xb = gen.deep_like_torch(min(chunk, N - s0), DEV, D=D, seed=0, stream=gen.STREAM_BASE,
                                    batch=s0 // chunk)
            g.add(xb)
            del xb
        torch.cuda.synchronize()
        emit(config="scale1b", row="add (generate + encode, streamed)", N=g.info()["N"], add_s=time.perf_counter() - t0)
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        g.reconfigure(K, n_iter=10, seed=0)
        torch.cuda.synchronize()
        emit(config="scale1b", row="reconfigure", nlist=K, reconfigure_s=time.perf_counter() - t0,
             bytes=g.info()["bytes"])
        qb = c["q_batch"]
        q = gen.deep_like_torch(c["nq"], DEV, D=D, seed=0, stream=gen.STREAM_QUERY)
        ms = timed(lambda: [g.query(q[i:i + qb], c["topk"], None, L=64, path="ivf") for i in range(0, c["nq"], qb)],
                   a.reps)
        emit(config="scale1b", row="ivf whole L=64 (batches of 1024)", ms=ms, qps=c["nq"] / ms * 1e3)
        S = gen.subset_torch(N, 1_000_000, DEV, seed=1)
        for path in ("auto", "linear", "ivf"):
            used = {}

            def f():
                for i in range(0, c["nq"], qb):
                    used["p"] = g.query(q[i:i + qb], c["topk"], S, L=64, path=path)[2]
            ms = timed(f, a.reps)
            emit(config="scale1b", row=f"subset |S|=1e6 L=64 {path}", path_used=["auto", "linear", "ivf"][used["p"]],
                 ms=ms, qps=c["nq"] / ms * 1e3)
        q1 = q[:qb]
        lib = rii.load()
        import ctypes as C
        lib.rii_kernel_timing(1)
        if os.environ.get("RII_PROFILE_LINEAR"):
            torch.cuda.profiler.start()
        ms = timed(lambda: g.query(q1, c["topk"], None, L=1, path="linear"), 1)
        if os.environ.get("RII_PROFILE_LINEAR"):
            torch.cuda.profiler.stop()
        kms, kn = C.c_double(), C.c_int64()
        lib.rii_kernel_timing_read(0, C.byref(kms), C.byref(kn))
        q16ms, q16n = C.c_double(), C.c_int64()
        lib.rii_kernel_timing_read(5, C.byref(q16ms), C.byref(q16n))
        lib.rii_kernel_timing(0)
        kernel_ms = kms.value / max(kn.value, 1)
        lookups = qb * N * M
        # the peak of the kernel that ran: u16 tables give 64 two-byte lookups per 128-B wavefront per
        # clock per SM, the u6 (one-byte) tables 128 (the r02d/r02l rows still carry the u16 peak although
        # the u6 kernel ran, u16_launches = 0: their frac reads 1.10 where 0.55 is meant)
        u6 = q16n.value == 0
        peak = 148 * (128 if u6 else 64) * 1965e6
        emit(config="scale1b", row="linear whole (1024 queries)", ms=ms, qps=qb / ms * 1e3,
             scanned_codes_per_s=qb * N / ms * 1e3, kernel_ms=kernel_ms, kernel_launches=kn.value,
             u16_launches=q16n.value, lookups_per_s=lookups / (kernel_ms / 1e3),
             roofline={"bound": "alu (shared-memory LUT pipe)", "peak_lookups_per_s": peak,
                       "frac": lookups / (kernel_ms / 1e3) / peak,
                       "code_bytes_per_launch": N * M, "note": ("u6 (one-byte)" if u6 else "u16") + " fixed-point tables (M = 8)"})
    if "latency" in only:  # small batches (serving): deep10m, time per call for nq in {1, 16, 128, 1024}
        kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS["deep10m"]
        g, b = build(kind, N, D, M, nlist, n_train)
        q = bench._device_data(kind, 1024, D, DEV, 0, gen.STREAM_QUERY)
        for n in (1, 16, 128, 1024):
            for path, L in (("linear", 1), ("ivf", 16), ("ivf", 64)):
                ms = timed(lambda: g.query(q[:n], topk, None, L=L, path=path), max(a.reps, 5))
                emit(config="latency", row=f"deep10m nq={n} {path} L={L}", nq=n, ms=ms, qps=n / ms * 1e3)
    if "deep10m" in only:
        kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS["deep10m"]
        g, b = build(kind, N, D, M, nlist, n_train)
        emit(config="deep10m", row="build", **b)
        q = bench._device_data(kind, nq, D, DEV, 0, gen.STREAM_QUERY)
        th = g.calibrate_theta(q[:1000], topk=100, L_grid=(1, 4, 16, 64))
        emit(config="deep10m", row="theta calibration", a=th[0], b=th[1], crossovers=th[2].tolist())
        rows_for("deep10m", g, q, topk, [1, 4, 16, 64], [100_000, 1_000_000], N, nlist, a.reps)


if __name__ == "__main__":
    main()
