"""Full-size parity at BASELINE.json configs[2] (10M x 96, M = 32, nlist = 3162, 10k
queries, top-100) in the launch configuration bench.py times (all 10k queries in
one rii_query call, queries resident in HBM).

* Codes: the oracle encodes all 10M raw rows itself (Eq. 1; the C
  oracle on every host core) and the GPU's codes must equal them bit for bit.
* Coarse centres come from the GPU's PQk-means (a full CPU reconfigure at this
  size is hours single-threaded); the posting lists must be a
  partition of the ids with ascending lists, and 100k sampled ids must sit in the
  list of their SDC-nearest centre (oracle assignment).
* Results: for 32 sampled queries, the full top-100 (ids and fp32 distances) of
  the whole-database linear scan, the inverted index at L = 64 and 1 % / 10 %
  subsets on both paths are compared element by element with the oracle's Alg. 1
  / Alg. 2, run on the oracle's codes and the GPU's
  centres / lists.
"""
import numpy as np
import pytest

from synth import generators as gen
from tests.parity import assert_topk_parity

pytestmark = pytest.mark.gpu


def test_deep10m_full_size(ref):
    import torch

    import paper_1808_03969_b200 as rii
    assert torch.cuda.is_available()
    N, D, M, K, nq, topk = 10_000_000, 96, 32, 3162, 10_000, 100
    dev = torch.device("cuda", 0)
    x = gen.deep_like_torch(N, dev, D=D, seed=0, stream=gen.STREAM_BASE)
    xt = gen.deep_like_torch(20_000, dev, D=D, seed=0, stream=gen.STREAM_TRAIN).cpu().numpy()
    cb = ref.train(xt, M, n_iter=3, seed=0)
    g = rii.Index(D, M, device=0)
    g.set_codebook(cb)
    g.add(x)
    g.reconfigure(K, n_iter=10, seed=0)
    xh = x.cpu().numpy()
    del x
    codes = ref.encode_mt(cb, xh, M)                      # all 10M rows, on every host core
    del xh
    assert np.array_equal(g.get_codes(), codes), "codes differ from the oracle (Eq. 1)"
    assert g.info()["bytes"] == (N + K) * M + 4 * N

    # posting lists: a partition into ascending lists; sampled ids in their nearest list
    centers = g.get_centers()
    off, lst = g.get_postings()
    assert off[0] == 0 and off[-1] == N and (np.diff(off) >= 0).all()
    a = np.full(N, -1, np.int32)
    a[lst] = np.repeat(np.arange(K, dtype=np.int32), np.diff(off))
    assert (a >= 0).all() and np.bincount(lst, minlength=N).max() == 1
    inner = np.ones(N, bool)
    inner[off[1:-1]] = False                              # list starts may step down
    assert (np.diff(lst)[inner[1:]] > 0).all(), "posting lists must be ascending (R11)"
    rng = np.random.default_rng(0)
    samp = np.sort(rng.choice(N, 100_000, replace=False))
    T = ref.sdc_tables(cb, D, M)
    want, _ = ref.assign_mt(T, codes[samp], centers)
    assert np.array_equal(a[samp], want), "coarse assignment a(n) differs from the oracle"

    q = gen.deep_like_torch(nq, dev, D=D, seed=0, stream=gen.STREAM_QUERY)
    qh = q.cpu().numpy()
    qi = np.sort(rng.choice(nq, 32, replace=False))
    S1 = gen.subset(N, N // 100, seed=0)
    S10 = gen.subset(N, N // 10, seed=1)
    cases = [("linear", 1, None), ("ivf", 64, None), ("ivf", 16, None),
             ("linear", 1, S1), ("ivf", 1, S1), ("linear", 1, S10), ("ivf", 4, S10)]
    for path, L, S in cases:
        St = None if S is None else torch.from_numpy(S).to(dev)
        ids, dist, used = g.query(q, topk, target_ids=St, L=L, path=path)
        torch.cuda.synchronize()
        ids, dist = ids.cpu().numpy(), dist.cpu().numpy()
        # every row of the whole 10k batch: sorted by (dist, id) (CA4, exact ties by id), unique ids
        lo = np.where(ids >= 0, ids, np.iinfo(np.int64).max)
        bad = ((dist[:, 1:] < dist[:, :-1]) | ((dist[:, 1:] == dist[:, :-1]) & (lo[:, 1:] <= lo[:, :-1]))) & (ids[:, 1:] >= 0)
        assert not bad.any(), f"{path} L={L}: {int(bad.any(1).sum())} rows not in (dist, id) order"
        ids, dist = ids[qi], dist[qi]
        if path == "linear":
            orr = ref.linear_mt(cb, codes, qh[qi], topk, S=S)
        else:
            orr = ref.ivf_mt(cb, codes, centers, off, lst, qh[qi], topk, L, S=S)
        assert_topk_parity(ref, cb, codes, qh[qi], (ids, dist), orr, S=S,
                           what=f"deep10m {path} L={L} |S|={'N' if S is None else len(S)}")
