"""Study (not part of the product): how well can the queries of a batch be grouped
into octets that share their probed lists?  For each grouping strategy, the work
inflation f = sum over octets of |union of the 8 queries' P nearest lists| * 8 /
(nq * P) -- the lookups an octet-resident IVF kernel would do relative to the
(query, list) pairs it must evaluate.

    python tools/octet_study.py [--workload deep10m] [--L 64]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402


def inflation(probes, order, P):
    nq = probes.shape[0]
    tot = 0
    for o in range(0, nq, 8):
        g = probes[order[o:o + 8]]
        tot += len(np.unique(g)) * 8
    return tot / (nq * P)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="deep10m")
    ap.add_argument("--L", type=int, default=64)
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
    cb = torch.from_numpy(g.get_codebook()).to(dev)              # [M][256][ds]
    C = torch.from_numpy(g.get_centers().astype(np.int64)).to(dev)  # [K][M]
    ds = D // M
    qv = q.view(nq, M, 1, ds)
    A = ((qv - cb.view(1, M, 256, ds)) ** 2).sum(-1)              # [nq][M][256]
    d0 = torch.zeros(nq, C.shape[0], device=dev)
    for m in range(M):
        d0 += A[:, m, :][:, C[:, m]]
    P = a.L
    probes = torch.topk(d0, P, dim=1, largest=False).indices.cpu().numpy()
    K = C.shape[0]
    res = {}
    res["identity"] = inflation(probes, np.arange(nq), P)
    res["by_top1"] = inflation(probes, np.lexsort((probes[:, 1], probes[:, 0])), P)
    # lists in a spatial order: greedy nearest-centre chain over SDC-like centre distances
    Cf = cb[torch.arange(M, device=dev).view(1, M), C].reshape(K, D)  # decoded centres
    dist = torch.cdist(Cf, Cf)
    visited = np.zeros(K, bool)
    chain = [0]
    visited[0] = True
    dn = dist.cpu().numpy()
    for _ in range(K - 1):
        r = dn[chain[-1]].copy()
        r[visited] = np.inf
        nxt = int(np.argmin(r))
        chain.append(nxt)
        visited[nxt] = True
    pos = np.empty(K, np.int64)
    pos[np.array(chain)] = np.arange(K)
    res["by_top1_chain"] = inflation(probes, np.lexsort((pos[probes[:, 1]], pos[probes[:, 0]])), P)
    # greedy: seed = first remaining query (chain order), add the 7 with the largest overlap
    ind = torch.zeros(nq, K, device=dev, dtype=torch.float16)
    ind.scatter_(1, torch.from_numpy(probes).to(dev), 1.0)
    ov = (ind @ ind.T).float().cpu().numpy()
    order0 = np.lexsort((pos[probes[:, 1]], pos[probes[:, 0]]))
    left = np.ones(nq, bool)
    out = []
    for s in order0:
        if not left[s]:
            continue
        left[s] = False
        row = np.where(left, ov[s], -1)
        pick = np.argsort(-row)[:7]
        pick = pick[row[pick] >= 0]
        left[pick] = False
        out.extend([s, *pick.tolist()])
    res["greedy_overlap"] = inflation(probes, np.array(out), P)
    print({k: round(v, 3) for k, v in res.items()}, "P", P, "nq", nq, "K", K)


if __name__ == "__main__":
    main()
