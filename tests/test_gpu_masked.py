"""IVF mode A executed as a linear scan: the P = K shortcut and the probe-masked
scan (capi.cu decide_exec, DESIGN.md §6 "Masked IVF").

Alg. 2 under reading R2 evaluates every S-member of the P probed lists,
so its candidate set is (union of the probed lists) ∩ S.  With P = K that set is S
and the result must equal Alg. 1's; with many probed lists the library
scans S once and evaluates a code only for the queries whose probed lists contain
it.  Every case is compared element by element with the oracle's Alg. 2
(`rref_ivf`), and the masked scan additionally with the posting-list traversals
(RII_IVF_MODE=list / query), which must give the same bytes.
"""
import numpy as np
import pytest

from synth import generators as gen
from tests.parity import assert_topk_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rii():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1808_03969_b200 as r
    r.load()
    return r


def _pair(rii, ref, kind, N, D, M, K):
    x = gen.base(kind, N, D, seed=N)
    g = rii.Index(D, M, device=0)
    g.train(x[:4000], n_iter=3, seed=0)
    o = ref.OracleIndex(D, M)
    o.train(x[:4000], n_iter=3, seed=0)
    g.add(x)
    o.add(x)
    g.reconfigure(K, n_iter=3, seed=0)
    o.reconfigure(K, n_iter=3, seed=0)
    assert np.array_equal(g.get_codes(), o.codes)
    assert np.array_equal(g.get_centers(), o.centers)
    return g, o


SHAPES = [("deep", 30_011, 96, 32, 40), ("sift", 25_000, 128, 16, 30), ("deep", 20_003, 96, 8, 24),
          ("gaussian", 9_001, 32, 4, 20), ("sift", 12_001, 128, 64, 16)]


@pytest.mark.parametrize("kind,N,D,M,K", SHAPES)
def test_masked_and_all_lists_match_oracle(rii, ref, monkeypatch, kind, N, D, M, K):
    g, o = _pair(rii, ref, kind, N, D, M, K)
    q = gen.base(kind, 37, D, seed=N, stream=gen.STREAM_QUERY)
    S_big = gen.subset(N, N // 3, seed=3)
    S_small = gen.subset(N, 500, seed=4)
    for sub in (None, S_big, S_small):
        nS = N if sub is None else len(sub)
        for L in (1, 2, 5, K):
            P = ref.num_probe(N, K, nS, sub is not None, L)
            orr = o.query(q, 100, S=sub, L=L, path=2)
            res = {}
            for mode in ("masked", "list", "query", None, "canon"):
                monkeypatch.delenv("RII_COARSE_ROT_MINK", raising=False)
                if mode == "canon":  # the coarse top-P kernel's canonical-only pass (the default
                    # is the lane-rotated pass + exact re-check of the candidates)
                    monkeypatch.delenv("RII_IVF_MODE", raising=False)
                    monkeypatch.setenv("RII_COARSE_ROT_MINK", "1000000000")
                elif mode:
                    monkeypatch.setenv("RII_IVF_MODE", mode)
                else:
                    monkeypatch.delenv("RII_IVF_MODE", raising=False)
                gr = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                assert gr[2] == 2  # path_used reports Alg. 2 whatever the execution
                assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub,
                                   what=f"{kind} M={M} K={K} P={P} mode={mode} S={nS}")
                res[mode] = gr
            monkeypatch.delenv("RII_IVF_MODE", raising=False)
            monkeypatch.delenv("RII_COARSE_ROT_MINK", raising=False)
            for mode in ("list", "query", None, "canon"):  # same bytes whichever way Alg. 2 executes
                assert np.array_equal(res["masked"][0], res[mode][0]), (mode, P)
                assert np.array_equal(res["masked"][1], res[mode][1]), (mode, P)
            if P >= K:  # every list probed: Alg. 2's result is Alg. 1's
                lin = g.query(q, 100, target_ids=sub, path="linear")
                assert np.array_equal(lin[0], res[None][0]) and np.array_equal(lin[1], res[None][1])


_cache = {}


def _long_index(rii, ref, kind, N, D, M, K):
    """N codes on the GPU with oracle-encoded codes, centres = K sample codes, the
    GPU's posting lists checked against the oracle's SDC assignment."""
    key = (kind, N, D, M, K)
    if key not in _cache:
        x = gen.base(kind, N, D, seed=N)
        cb = ref.train(x[:20_000], M, n_iter=3, seed=0)
        g = rii.Index(D, M, device=0)
        g.set_codebook(cb)
        g.add(x)
        codes = ref.encode_mt(cb, x, M)
        assert np.array_equal(g.get_codes(), codes)
        rows = np.unique(codes[::997], axis=0)[:K]
        centers = np.ascontiguousarray(rows)
        g.set_centers(centers)
        off, ids = g.get_postings()
        T = ref.sdc_tables(cb, D, M)
        a, _ = ref.assign_mt(T, codes, centers)
        o_off, o_ids = ref.build_postings(a, centers.shape[0])
        assert np.array_equal(off, o_off) and np.array_equal(ids, o_ids), "posting lists differ (SDC assignment)"
        _cache[key] = (g, cb, codes, centers, off, ids)
    return _cache[key]


# (kind, N, D, M, K, nq, subset size or None, L): long scans on the integer-table
# kernels (u6 at M = 32 / 16 / 8 above RII_Q16_MIN) with the masked group-minimum
# bound, ragged query batches
LONG = [("deep", 600_000, 96, 32, 256, 45, None, 64),
        ("deep", 600_000, 96, 32, 256, 40, 60_000, 8),
        ("sift", 600_000, 128, 16, 200, 33, None, 40),
        ("deep", 600_000, 96, 8, 128, 21, 200_000, 16)]


@pytest.mark.parametrize("kind,N,D,M,K,nq,ns,L", LONG)
def test_masked_long_scan_matches_oracle(rii, ref, monkeypatch, kind, N, D, M, K, nq, ns, L):
    g, cb, codes, centers, off, ids = _long_index(rii, ref, kind, N, D, M, K)
    K = centers.shape[0]
    q = gen.base(kind, nq, D, seed=N + 1, stream=gen.STREAM_QUERY)
    sub = None if ns is None else gen.subset(N, ns, seed=ns)
    monkeypatch.setenv("RII_Q16_MIN", "50000")  # the integer tables also for the 60k subset
    monkeypatch.setenv("RII_IVF_MODE", "masked")
    gr = g.query(q, 100, target_ids=sub, L=L, path="ivf")
    monkeypatch.setenv("RII_IVF_MODE", "query")
    gt = g.query(q, 100, target_ids=sub, L=L, path="ivf")
    orr = ref.ivf_mt(cb, codes, centers, off, ids, q, 100, L, S=sub)
    assert_topk_parity(ref, cb, codes, q, gr, orr, S=sub, what=f"masked {kind} M={M} L={L} S={ns}")
    assert np.array_equal(gr[0], gt[0]) and np.array_equal(gr[1], gt[1])


@pytest.mark.parametrize("kind,N,D,M,K,nq,ns,L", LONG)
def test_rank0_query_major_matches_oracle(rii, ref, monkeypatch, kind, N, D, M, K, nq, ns, L):
    """List-major Alg. 2 with the rank-0 phase on the query-major traversal
    (each query's nearest list scanned with its own table, partials written in place,
    their kk-th distance published as the bound of the integer phases) and on list
    items (RII_R0_QMAJOR=0): both equal the oracle and each other byte for byte."""
    g, cb, codes, centers, off, ids = _long_index(rii, ref, kind, N, D, M, K)
    q = gen.base(kind, nq, D, seed=N + 2, stream=gen.STREAM_QUERY)
    sub = None if ns is None else gen.subset(N, ns, seed=ns + 1)
    monkeypatch.setenv("RII_IVF_MODE", "list")
    monkeypatch.setenv("RII_LIST_Q16_MIN", "64")  # integer phases at these list lengths
    orr = ref.ivf_mt(cb, codes, centers, off, ids, q, 100, L, S=sub)
    res = {}
    for v in ("1", "0"):
        monkeypatch.setenv("RII_R0_QMAJOR", v)
        res[v] = g.query(q, 100, target_ids=sub, L=L, path="ivf")
        assert_topk_parity(ref, cb, codes, q, res[v], orr, S=sub, what=f"r0q={v} {kind} M={M} L={L} S={ns}")
    assert np.array_equal(res["0"][0], res["1"][0]) and np.array_equal(res["0"][1], res["1"][1])
