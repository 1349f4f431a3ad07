"""Equivalence probe at full size (deep10m, 10k queries): the list-major and the
query-major inverted-index traversals must return identical results (both are
exact); for any query where they differ, which one matches the oracle and how.
(Found the round-2 tie-order bug of list-major keys: 26 of 10k queries.)

    python tools/ivf_traversal_equivalence.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from oracle import ref  # noqa: E402
from synth import generators as gen  # noqa: E402

kind, N, D, M, nlist, nq, topk, n_train, _ = bench.WORKLOADS["deep10m"]
dev = torch.device("cuda", 0)
xt = bench._device_data(kind, 20000, D, dev, 0, gen.STREAM_TRAIN).cpu().numpy()
cb = ref.train(xt, M, n_iter=3, seed=0)
g = rii.Index(D, M, device=0)
g.set_codebook(cb)
x = bench._device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
g.add(x)
g.reconfigure(nlist, n_iter=10, seed=0)
codes = ref.encode_mt(cb, x.cpu().numpy(), M)
del x
q = bench._device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
qh = q.cpu().numpy()
off, ids = g.get_postings()
cen = g.get_centers()
for frac, L in ((0.1, 64), (0.01, 64), (None, 64), (None, 16)):
    S = None if frac is None else gen.subset_torch(N, int(N * frac), dev, seed=0)
    Sh = None if S is None else S.cpu().numpy()
    out = {}
    for mode in ("query", "list"):
        os.environ["RII_IVF_MODE"] = mode
        i, d, _ = g.query(q, topk, S, L=L, path="ivf")
        out[mode] = (i.cpu().numpy(), d.cpu().numpy())
    os.environ.pop("RII_IVF_MODE")
    diff = np.nonzero((out["query"][0] != out["list"][0]).any(1) | (out["query"][1] != out["list"][1]).any(1))[0]
    print(f"frac={frac} L={L}: {len(diff)} of {nq} queries differ", flush=True)
    if len(diff):
        sel = diff[:16]
        oi, od = ref.ivf_mt(cb, codes, cen, off, ids, qh[sel], topk, L, S=Sh)
        for mode in ("query", "list"):
            gi, gd = out[mode][0][sel], out[mode][1][sel]
            eq = [(np.array_equal(gi[r], oi[r]) and np.array_equal(gd[r], od[r])) for r in range(len(sel))]
            print(f"  {mode}: {sum(eq)}/{len(sel)} equal the oracle", flush=True)
            for r in range(min(3, len(sel))):
                if not eq[r]:
                    miss = np.setdiff1d(oi[r], gi[r])
                    extra = np.setdiff1d(gi[r], oi[r])
                    print(f"    q{sel[r]}: missing {miss[:5]} extra {extra[:5]} kth gpu {gd[r][-1]:.7g} oracle {od[r][-1]:.7g}")
                    k = np.nonzero((gi[r] != oi[r]) | (gd[r] != od[r]))[0]
                    for j in k[:4]:
                        print(f"      rank {j}: gpu ({gi[r][j]}, {gd[r][j]!r}) oracle ({oi[r][j]}, {od[r][j]!r})")
