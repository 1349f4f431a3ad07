"""Stress: repeated identical IVF (list-major, several phases) and large-M linear
queries must give identical results.  python tools/nondet_stress_ivf.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402

dev = torch.device("cuda", 0)
reps = int(os.environ.get("REPS", "20"))


def run(tag, g, q, **kw):
    first, bad = None, []
    for r in range(reps):
        i, d, _ = g.query(q, 100, **kw)
        i, d = i.cpu().numpy(), d.cpu().numpy()
        if first is None:
            first = (i, d)
        else:
            diff = np.nonzero((i != first[0]).any(1) | (d != first[1]).any(1))[0]
            if len(diff):
                bad.append((r, diff[:4].tolist()))
    print(f"{tag}: {len(bad)} of {reps - 1} repeats differ {bad[:3]}", flush=True)


for M, N, nq, K in ((32, 2_000_000, 1024, 1414), (16, 2_000_000, 1024, 1414), (8, 2_000_000, 1024, 1414)):
    x = gen.deep_like_torch(N, dev, D=96, seed=M, stream=gen.STREAM_BASE)
    g = rii.Index(96, M, device=0)
    g.train(x[:50_000], n_iter=5, seed=0)
    g.add(x)
    g.reconfigure(K, n_iter=4, seed=0)
    q = gen.deep_like_torch(nq, dev, D=96, seed=M, stream=gen.STREAM_QUERY)
    for L in (64, 16):
        run(f"ivf M={M} L={L}", g, q, L=L, path="ivf")
    S = gen.subset_torch(N, N // 10, dev, seed=1)
    run(f"ivf M={M} L=64 10% subset", g, q, target_ids=S, L=64, path="ivf")
    del g, x
    torch.cuda.empty_cache()
x = gen.deep_like_torch(400_000, dev, D=960, seed=5, stream=gen.STREAM_BASE)
g = rii.Index(960, 240, device=0)
g.train(x[:20_000], n_iter=3, seed=0)
g.add(x)
q = gen.deep_like_torch(1024, dev, D=960, seed=5, stream=gen.STREAM_QUERY)
run("large M=240 linear", g, q, path="linear")
