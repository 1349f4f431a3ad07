import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ref
from synth import generators as gen
import paper_1808_03969_b200 as rii
from tests.parity import assert_topk_parity
for (N, K, frac, L, nq) in ((200_000, 447, 0.1, 64, 40), (60_000, 60, 0.1, 8, 30), (300_000, 300, 0.3, 16, 30)):
    x = gen.deep_like(N, 96, seed=N)
    q = gen.deep_like(nq, 96, seed=N, stream=gen.STREAM_QUERY)
    cb = ref.train(x[:5000], 32, n_iter=2, seed=0)
    g = rii.Index(96, 32, device=0); g.set_codebook(cb); g.add(x); g.reconfigure(K, n_iter=2, seed=0)
    codes = ref.encode_mt(cb, x, 32)
    off, ids = g.get_postings(); cen = g.get_centers()
    S = gen.subset(N, int(N * frac), seed=1)
    res = {}
    for mode in ("query", "list"):
        os.environ["RII_IVF_MODE"] = mode
        res[mode] = g.query(q, 100, target_ids=S, L=L, path="ivf")
    os.environ.pop("RII_IVF_MODE")
    orr = ref.ivf_mt(cb, codes, cen, off, ids, q, 100, L, S=S)
    for mode, r in res.items():
        try:
            assert_topk_parity(ref, cb, codes, q, r, orr, S=S, what=f"{N} {mode}")
            print(N, mode, "OK")
        except AssertionError as e:
            print(N, mode, "FAIL", str(e)[:300])
