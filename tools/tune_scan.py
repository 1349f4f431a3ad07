"""Linear-scan tuning driver: build an index (no reconfigure) and time whole-database
linear queries; kernel time from the library's CUDA events.

    RII_SCAN_CFG=0 python tools/tune_scan.py --kind deep --N 100000000 --D 96 --M 8 --nq 2048
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="deep")
    ap.add_argument("--N", type=int, default=100_000_000)
    ap.add_argument("--D", type=int, default=96)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--nq", type=int, default=2048)
    ap.add_argument("--topk", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = rii.Index(a.D, a.M, device=0)
    g.train(bench._device_data(a.kind, 100_000, a.D, dev, 0, gen.STREAM_TRAIN), n_iter=5, seed=0)
    chunk = 1 << 24
    for s in range(0, a.N, chunk):
        g.add(bench._device_data(a.kind, min(chunk, a.N - s), a.D, dev, 1 + s // chunk, gen.STREAM_BASE))
    q = bench._device_data(a.kind, a.nq, a.D, dev, 0, gen.STREAM_QUERY)
    g.query(q, a.topk, None, path="linear")
    torch.cuda.synchronize()
    lib = rii.load()
    lib.rii_kernel_timing(1)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        g.query(q, a.topk, None, path="linear")
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    kms, kn = C.c_double(), C.c_int64()
    lib.rii_kernel_timing_read(0, C.byref(kms), C.byref(kn))
    pms, pn = C.c_double(), C.c_int64()
    lib.rii_kernel_timing_read(3, C.byref(pms), C.byref(pn))
    kernel = kms.value / max(kn.value, 1)
    look = a.nq * a.N * a.M
    print(json.dumps({"cfg": os.environ.get("RII_SCAN_CFG", "default"), "M": a.M, "N": a.N, "nq": a.nq,
                      "ms": ms, "qps": a.nq / ms * 1e3, "kernel_ms": kernel, "lookups_per_s": look / kernel * 1e3,
                      "packed": pn.value > 0}), flush=True)


if __name__ == "__main__":
    main()
