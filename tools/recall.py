"""Recall@R harness (the paper's accuracy measure: "the fraction of queries
for which the ground truth nearest neighbor is returned within the top-1 result").

Ground truth: exact squared-L2 nearest neighbour of every query over the raw
vectors, computed on the GPU with torch as a measurement tool (not the product
path): a fp32 GEMM shortlist of 64 candidates per query, then an fp64 recheck.

    python tools/recall.py [--workload deep10m|sift1m] [--nq 10000]
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


def ground_truth(x, q, chunk=1 << 20, short=64):
    torch.backends.cuda.matmul.allow_tf32 = False
    xn = (x * x).sum(1)
    best_d = torch.full((q.shape[0], short), float("inf"), device=q.device)
    best_i = torch.zeros((q.shape[0], short), dtype=torch.int64, device=q.device)
    for s in range(0, x.shape[0], chunk):
        xs = x[s:s + chunk]
        d = xn[s:s + chunk][None, :] - 2.0 * (q @ xs.T)
        v, i = torch.topk(d, min(short, xs.shape[0]), dim=1, largest=False)
        cd, ci = torch.cat([best_d, v], 1), torch.cat([best_i, i + s], 1)
        best_d, o = torch.topk(cd, short, dim=1, largest=False)
        best_i = torch.gather(ci, 1, o)
    exact = ((x[best_i].double() - q[:, None, :].double()) ** 2).sum(-1)
    j = torch.argmin(exact, 1)
    return best_i[torch.arange(q.shape[0], device=q.device), j]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="deep10m")
    ap.add_argument("--nq", type=int, default=10_000)
    a = ap.parse_args()
    kind, N, D, M, nlist, nq, topk, n_train, label = bench.WORKLOADS[a.workload]
    nq = min(nq, a.nq)
    dev = torch.device("cuda", 0)
    x = bench._device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
    q = bench._device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
    gt = ground_truth(x, q)
    g = rii.Index(D, M, device=0)
    g.train(bench._device_data(kind, n_train, D, dev, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
    g.add(x)
    g.reconfigure(nlist, n_iter=10, seed=0)
    for path, L in [("linear", 1)] + [("ivf", L) for L in (1, 2, 4, 8, 16, 32, 64)]:
        ids, _, _ = g.query(q, 100, L=L, path=path)
        for R in (1, 10, 100):
            hit = (ids[:, :R] == gt[:, None]).any(1).float().mean().item()
            print(json.dumps({"workload": a.workload, "path": path, "L": L, "R": R, "recall": hit}), flush=True)


if __name__ == "__main__":
    main()
