"""A/B timing of one query configuration under several environment settings
(knobs read per call by the library), on one bench workload built once.

    python tools/ab_env.py --path ivf --L 64 [--subset 0.1] "VAR=a;VAR2=b"  VAR=c ...
"""
import argparse
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
    ap.add_argument("--workload", default="deep10m")
    ap.add_argument("--path", default="ivf")
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--subset", type=float, default=0.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nq", type=int, default=0, help="queries per call (default: the workload's)")
    ap.add_argument("--subset_n", type=int, default=0, help="subset size in ids (overrides --subset)")
    ap.add_argument("--cases", default="", help="several query configurations on one build: "
                    "'path/L/subset_n[/nq]' entries separated by commas (overrides --path/--L/--subset_n)")
    ap.add_argument("settings", nargs="*")
    a = ap.parse_args()
    kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda", 0)
    g = rii.Index(D, M, device=0)
    g.train(bench._device_data(kind, n_train, D, dev, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
    x = bench._device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
    g.add(x)
    del x
    g.reconfigure(nlist, n_iter=10, seed=0)
    cases = [c.split("/") for c in a.cases.split(",") if c] or [[a.path, str(a.L), str(a.subset_n or int(N * a.subset)), str(a.nq or nq)]]
    for c in cases:
        path, L, ns = c[0], int(c[1]), int(c[2])
        cq = int(c[3]) if len(c) > 3 else (a.nq or nq)
        run_case(g, kind, N, D, cq, topk, dev, path, L, ns, a)


def run_case(g, kind, N, D, nq, topk, dev, path, L, ns, a):
    q = bench._device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
    S = gen.subset_torch(N, ns, dev, seed=0) if ns > 0 else None
    ids = torch.empty((nq, topk), dtype=torch.int64, device=dev)
    dist = torch.empty((nq, topk), dtype=torch.float32, device=dev)
    ref = None
    for st in (a.settings or [""]):
        env = dict(kv.split("=", 1) for kv in st.split(";") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        g.query(q, topk, S, L=L, path=path, out=(ids, dist))
        torch.cuda.synchronize()
        ms = bench._timed_steps(lambda: g.query(q, topk, S, L=L, path=path, out=(ids, dist)), a.reps,
                                torch.cuda.current_stream())
        same = None
        if ref is None:
            ref = (ids.clone(), dist.clone())
        else:
            same = bool(torch.equal(ref[0], ids) and torch.equal(ref[1], dist))
        print(json.dumps({"workload": a.workload, "path": path, "L": L, "subset_n": ns, "nq": nq, "env": env,
                          "ms": sorted(ms)[len(ms) // 2], "qps": nq / (sorted(ms)[len(ms) // 2] / 1e3),
                          "same_as_first": same}), flush=True)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v

if __name__ == "__main__":
    main()
