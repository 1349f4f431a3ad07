"""Stress: repeated identical linear queries must give identical results (and the
oracle's); many chunks per query batch (few queries, many codes) maximise the
cross-CTA bound sharing.  python tools/nondet_stress.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_03969_b200 as rii  # noqa: E402
from oracle import ref  # noqa: E402
from synth import generators as gen  # noqa: E402

dev = torch.device("cuda", 0)
reps = int(os.environ.get("REPS", "30"))
for M, N, nq in ((8, 2_000_000, 64), (8, 2_000_000, 1024), (32, 2_000_000, 64), (32, 2_000_000, 1024), (16, 2_000_000, 256)):
    x = gen.deep_like_torch(N, dev, D=96, seed=M, stream=gen.STREAM_BASE)
    g = rii.Index(96, M, device=0)
    g.train(x[:50_000], n_iter=5, seed=0)
    g.add(x)
    cb = g.get_codebook()
    q = gen.deep_like_torch(nq, dev, D=96, seed=M, stream=gen.STREAM_QUERY)
    first = None
    bad = []
    for r in range(reps):
        i, d, _ = g.query(q, 100, path="linear")
        i, d = i.cpu().numpy(), d.cpu().numpy()
        if first is None:
            first = (i, d)
        else:
            diff = np.nonzero((i != first[0]).any(1) | (d != first[1]).any(1))[0]
            if len(diff):
                bad.append((r, diff[:4].tolist()))
    codes = g.get_codes()
    sel = np.arange(0, nq, max(1, nq // 16))
    oi, od = ref.linear_mt(cb, codes, q.cpu().numpy()[sel], 100)
    ok_first = all(np.array_equal(first[0][s], oi[k]) and np.array_equal(first[1][s], od[k]) for k, s in enumerate(sel))
    print(f"M={M} N={N} nq={nq}: {len(bad)} of {reps - 1} repeats differ {bad[:3]}; first run == oracle on {len(sel)} sampled: {ok_first}",
          flush=True)
    del g, x
    torch.cuda.empty_cache()
