"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs (BASELINE.json north_star tolerances; see
tests/parity.py).  Sizes span several CTAs/tiles and a ragged tail while the
oracle still finishes in seconds."""
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


def _build_pair(rii, ref, x, M, K, n_iter=5, seed=0, train_rows=None, train_iter=5):
    """GPU index and oracle index built the same way: train on the same rows,
    add, reconfigure.  Returns (gpu, oracle)."""
    D = x.shape[1]
    tr = x if train_rows is None else train_rows
    g = rii.Index(D, M)
    g.train(tr, n_iter=train_iter, seed=seed)
    o = ref.OracleIndex(D, M)
    o.train(tr, n_iter=train_iter, seed=seed)
    g.add(x)
    o.add(x)
    if K:
        g.reconfigure(K, n_iter=n_iter, seed=seed)
        o.reconfigure(K, n_iter=n_iter, seed=seed)
    return g, o


def _check_state(g, o):
    assert np.array_equal(g.get_codebook(), o.cb), "code book differs (O-TRAIN)"
    assert np.array_equal(g.get_codes(), o.codes), "codes differ (Eq. 1)"
    if o.K:
        assert np.array_equal(g.get_centers(), o.centers), "PQk-means centres differ (R9)"
        off, ids = g.get_postings()
        assert np.array_equal(off, o.offsets) and np.array_equal(ids, o.ids), "posting lists differ"


# ------------------------------------------------------------------ tiny ----
def test_tiny_config_end_to_end(rii, ref):
    """BASELINE.json configs[0]: N=10k N(0,1) D=32, M=4, 20 k-means iters on the data,
    nlist=100, 100 queries, topk=10, whole search at L=8 and a 1000-id subset."""
    c = gen.CONFIGS["tiny"]
    x = gen.gaussian(c["N"], c["D"], seed=0)
    q = gen.gaussian(c["nq"], c["D"], seed=0, stream=gen.STREAM_QUERY)
    S = gen.subset(c["N"], 1000, seed=0)
    ref.reseed_reset()
    g, o = _build_pair(rii, ref, x, c["M"], c["nlist"], n_iter=10, train_iter=20)
    assert ref.reseed_counts()[1] >= 1  # the bit-exact state check covers a PQk-means re-seed (R9)
    _check_state(g, o)
    for path in ("linear", "ivf", "auto"):
        for sub in (None, S):
            for L in (1, 8, 100):
                gr = g.query(q, 10, target_ids=sub, L=L, path=path)
                orr = o.query(q, 10, S=sub, L=L, path={"linear": 1, "ivf": 2, "auto": 0}[path])
                assert gr[2] == orr[2], f"path_used {gr[2]} != {orr[2]}"
                assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"tiny {path} L={L} S={sub is not None}")


# ------------------------------------------------------- shapes / kernels ---
CASES = [
    # (kind, N, D, M, K, nq, topk)       -- M in {4,8,16,32}: lane-rotated kernel; 12, 6: generic kernel
    ("sift", 23_457, 128, 16, 50, 37, 100),
    ("deep", 19_999, 96, 32, 40, 25, 100),
    ("deep", 17_001, 96, 8, 30, 29, 50),
    ("deep", 9_001, 96, 12, 20, 13, 20),
    ("gaussian", 5_003, 30, 6, 10, 7, 5),
]


@pytest.mark.parametrize("kind,N,D,M,K,nq,topk", CASES)
def test_paths_match_oracle(rii, ref, kind, N, D, M, K, nq, topk):
    x = gen.base(kind, N, D, seed=N)
    q = gen.base(kind, nq, D, seed=N, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, M, K, n_iter=4, train_rows=x[:4000], train_iter=4)
    _check_state(g, o)
    S_small = gen.subset(N, 777, seed=1)
    S_big = gen.subset(N, N // 2 + 3, seed=2)
    for path in ("linear", "ivf"):
        for sub in (None, S_small, S_big):
            for L in (1, 4):
                gr = g.query(q, topk, target_ids=sub, L=L, path=path)
                orr = o.query(q, topk, S=sub, L=L, path=1 if path == "linear" else 2)
                assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"{kind} M={M} {path} L={L}")


@pytest.mark.parametrize("mode", ["list", "query"])
@pytest.mark.parametrize("kind,N,D,M,K", [("deep", 30_011, 96, 32, 20), ("sift", 25_000, 128, 16, 16),
                                          ("sift", 24_001, 128, 64, 12),
                                          ("deep", 20_003, 96, 8, 12), ("deep", 40_000, 96, 32, 2)])
def test_ivf_list_major_and_query_major(rii, ref, monkeypatch, mode, kind, N, D, M, K):
    """Both posting-list traversals (list-major: B queries share a list; query-major:
    one table per query) against the oracle's Alg. 2, whole and subset.  K = 2 makes
    the lists long (20k codes).  List-major variants (two codes per thread for M = 8,
    bf16-packed and group-minimum-bound items, u6 / u7 items) give the same bytes."""
    monkeypatch.setenv("RII_IVF_MODE", mode)
    x = gen.base(kind, N, D, seed=N)
    q = gen.base(kind, 41, D, seed=N, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, M, K, n_iter=3, train_rows=x[:3000], train_iter=3)
    _check_state(g, o)
    # |S| = 7: almost every restricted list is empty (items that find nothing write
    # only their first key; the merge must skip them) and the rows are padded
    for sub in (None, gen.subset(N, N // 3, seed=5), gen.subset(N, 7, seed=6)):
        for L in (1, 3, K):
            gr = g.query(q, 100, target_ids=sub, L=L, path="ivf")
            orr = o.query(q, 100, S=sub, L=L, path=2)
            assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"ivf-{mode} {kind} M={M} L={L}")
            if mode == "list":  # two-phase u16 items (default) == single-phase fp32 / bf16 items
                monkeypatch.setenv("RII_Q16", "0")
                g2 = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                monkeypatch.delenv("RII_Q16")
                assert np.array_equal(gr[0], g2[0]) and np.array_equal(gr[1], g2[1])
                monkeypatch.setenv("RII_LIST_PACKED_MIN", "1")  # bf16-packed fp items (A/B variant, off by default)
                g5 = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                monkeypatch.delenv("RII_LIST_PACKED_MIN")
                assert np.array_equal(gr[0], g5[0]) and np.array_equal(gr[1], g5[1])
                monkeypatch.setenv("RII_LIST_BOUND", "1")  # group-minimum bound items instead of phase A
                g4 = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                monkeypatch.delenv("RII_LIST_BOUND")
                assert np.array_equal(gr[0], g4[0]) and np.array_equal(gr[1], g4[1])
                if M == 8:  # one code per thread and step (two by default)
                    monkeypatch.setenv("RII_LIST_U", "1")
                    g6 = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                    monkeypatch.delenv("RII_LIST_U")
                    assert np.array_equal(gr[0], g6[0]) and np.array_equal(gr[1], g6[1])
                if M == 32:  # u6 items of 8 (RII_LIST_U6=3) and 16 queries (=4); 7-bit items
                    for var, cfg in (("RII_LIST_U6", "3"), ("RII_LIST_U6", "4"), ("RII_LIST_U7", "0"),
                                     ("RII_LIST_NTH", "192"), ("RII_LIST_NTH", "384")):
                        monkeypatch.setenv(var, cfg)
                        g3 = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                        monkeypatch.delenv(var)
                        assert np.array_equal(gr[0], g3[0]) and np.array_equal(gr[1], g3[1]), (var, cfg)


def test_device_memory_path_matches_host_path(rii, ref):
    import torch
    x = gen.deep_like(12_345, 96, seed=3)
    q = gen.deep_like(40, 96, seed=3, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, 32, 0, train_rows=x[:3000], train_iter=3)
    hi, hd, _ = g.query(q, 64, path="linear")
    di, dd, _ = g.query(torch.from_numpy(q).cuda(), 64, path="linear")
    torch.cuda.synchronize()
    assert np.array_equal(hi, di.cpu().numpy()) and np.array_equal(hd, dd.cpu().numpy())
    gx = rii.Index(96, 32)
    gx.set_codebook(g.get_codebook())
    gx.add(torch.from_numpy(x).cuda())
    assert np.array_equal(gx.get_codes(), o.codes)


# ------------------------------------------------------------- edge cases ---
def test_edge_cases(rii, ref):
    x = gen.sift_like(3_001, 128, seed=7)
    q = gen.sift_like(9, 128, seed=7, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, 16, 10, n_iter=3, train_rows=x, train_iter=3)
    # topk > |S| and > N: padding with (-1, +inf) (R18)
    for topk, sub in ((1024, None), (50, np.array([5, 17, 3000], np.int64)), (7, np.array([42], np.int64))):
        for path in ("linear", "ivf"):
            gr = g.query(q, topk, target_ids=sub, L=3, path=path)
            orr = o.query(q, topk, S=sub, L=3, path=1 if path == "linear" else 2)
            assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"edge topk={topk}")
    # empty subset -> all padding
    ids, dist, _ = g.query(q, 5, target_ids=np.zeros(0, np.int64), path="linear")
    assert (ids == -1).all() and np.isinf(dist).all()
    # invalid subsets (R6): unsorted, duplicate, out of range
    for bad in ([3, 2], [4, 4], [0, 3001]):
        with pytest.raises(rii.RiiError) as e:
            g.query(q, 5, target_ids=np.array(bad, np.int64))
        assert e.value.status == 1
    # topk bounds
    with pytest.raises(rii.RiiError):
        g.query(q, 0)
    with pytest.raises(rii.RiiError):
        g.query(q, 1025)
    # nq = 0
    ids, dist, _ = g.query(q[:0], 5)
    assert ids.shape == (0, 5)
    # K = 0 (never reconfigured): LINEAR forced, IVF refused
    g0 = rii.Index(128, 16)
    g0.set_codebook(o.cb)
    g0.add(x)
    assert g0.query(q, 5)[2] == rii.PATH_LINEAR
    with pytest.raises(rii.RiiError) as e:
        g0.query(q, 5, path="ivf")
    assert e.value.status == 2
    # untrained index
    with pytest.raises(rii.RiiError) as e:
        rii.Index(128, 16).add(x)
    assert e.value.status == 2


def test_duplicate_codes_tie_break(rii, ref):
    """Identical codes give identical distances; ties must resolve to the lowest id
    (CA4) even across CTAs and chunks."""
    base = gen.deep_like(300, 96, seed=9)
    x = np.concatenate([base] * 40)  # 12,000 rows, each code repeated 40 times
    q = gen.deep_like(11, 96, seed=9, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, 32, 0, train_rows=x[:3000], train_iter=2)
    gr = g.query(q, 100, path="linear")
    orr = o.query(q, 100, path=1)
    assert np.array_equal(gr[0], orr[0]) and np.array_equal(gr[1], orr[1])


@pytest.mark.parametrize("mode", ["list", "query"])
def test_duplicate_codes_tie_break_ivf(rii, ref, monkeypatch, mode):
    """Exact distance ties in the inverted index resolve to the lowest id (CA4) on
    both traversals -- list-major items stream a list-ordered copy of the codes, so
    their keys must carry ids, not positions -- whole and subset, across many lists
    and the integer (u6 / u16) items."""
    monkeypatch.setenv("RII_IVF_MODE", mode)
    monkeypatch.setenv("RII_LIST_Q16_MIN", "64")
    for kind, D, M in (("deep", 96, 32), ("sift", 128, 16)):
        base = gen.base(kind, 700, D, seed=19)
        x = np.concatenate([base] * 60)  # 42,000 rows, every code 60 times
        q = gen.base(kind, 23, D, seed=19, stream=gen.STREAM_QUERY)
        g, o = _build_pair(rii, ref, x, M, 12, n_iter=2, train_rows=base, train_iter=2)
        S = gen.subset(len(x), len(x) // 2 + 11, seed=7)
        for sub in (None, S):
            for L in (2, 12):
                gr = g.query(q, 100, target_ids=sub, L=L, path="ivf")
                orr = o.query(q, 100, S=sub, L=L, path=2)
                assert np.array_equal(gr[0], orr[0]) and np.array_equal(gr[1], orr[1]), (kind, mode, L, sub is None)


def test_lossless_case_is_exact_knn(rii, ref):
    """C-PIN7 on the GPU: D = M, code book {0..255}, integer data -> exact kNN."""
    x = gen.lossless(6_000, 16, seed=5)
    q = np.random.default_rng(5).integers(0, 256, size=(20, 16)).astype(np.float32)
    cb = np.tile(np.arange(256, dtype=np.float32)[None, :, None], (16, 1, 1))
    g = rii.Index(16, 16)
    g.set_codebook(cb)
    g.add(x)
    ids, dist, _ = g.query(q, 30, path="linear")
    for i in range(len(q)):
        d = ((x.astype(np.int64) - q[i].astype(np.int64)) ** 2).sum(1)
        order = np.lexsort((np.arange(len(x)), d))[:30]
        assert np.array_equal(ids[i], order) and np.array_equal(dist[i], d[order].astype(np.float32))


def test_theta_rule_and_ivf_all_lists(rii, ref):
    x = gen.sift_like(8_000, 128, seed=11)
    q = gen.sift_like(16, 128, seed=11, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, 16, 40, n_iter=3, train_rows=x[:3000], train_iter=3)
    th = ref.default_theta(g.info()["N"], 40, 2)
    for size, want in ((th - 1, rii.PATH_LINEAR), (th, rii.PATH_IVF)):
        S = gen.subset(8_000, size, seed=size)
        assert g.query(q, 5, target_ids=S, L=2)[2] == want
    g.set_theta(10**9)
    assert g.query(q, 5, L=2)[2] == rii.PATH_LINEAR
    g.set_theta(-1)
    lin = g.query(q, 40, path="linear")
    ivf = g.query(q, 40, L=40, path="ivf")     # L = nlist -> linear (BASELINE.json invariant 2)
    assert np.array_equal(lin[0], ivf[0]) and np.array_equal(lin[1], ivf[1])


def test_add_after_reconfigure_and_growth(rii, ref):
    """Data addition with K > 0 then reconfigure again (config 4 in small)."""
    x = gen.sift_like(12_000, 128, seed=13)
    q = gen.sift_like(12, 128, seed=13, stream=gen.STREAM_QUERY)
    ref.reseed_reset()
    g, o = _build_pair(rii, ref, x[:2_000], 16, 20, n_iter=3, train_rows=x[:2_000], train_iter=3)
    assert ref.reseed_counts()[0] >= 1  # training re-seeds (R8) inside the bit-exact code-book check
    _check_state(g, o)
    for s in range(2_000, 12_000, 3_333):
        g.add(x[s:s + 3_333])
        o.add(x[s:s + 3_333])
    _check_state(g, o)
    for L in (1, 5):
        assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 20, L=L, path="ivf"), o.query(q, 20, L=L, path=2))
    ref.reseed_reset()
    g.reconfigure(110, n_iter=3, seed=4)
    o.reconfigure(110, n_iter=3, seed=4)
    assert ref.reseed_counts()[1] >= 1  # PQk-means re-seeds (R9) inside the bit-exact centre check
    _check_state(g, o)
    assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 20, L=2, path="ivf"), o.query(q, 20, L=2, path=2))


def test_logical_shards_equal_single_index(rii, ref, tmp_path):
    """Id-range sharding on one GPU: two detached shards, per-shard
    partial top-k, merge -> the oracle's result on the whole database (C-PIN10) and
    identical to the single index; each shard survives save / load (RIIS layout,
    validated: a corrupted posting offset is rejected)."""
    import struct
    import torch
    x = gen.deep_like(20_001, 96, seed=17)
    q = gen.deep_like(33, 96, seed=17, stream=gen.STREAM_QUERY)
    single, o = _build_pair(rii, ref, x, 32, 0, train_rows=x[:3000], train_iter=2)
    cb = single.get_codebook()
    shards = []
    for r in range(2):
        s = rii.Index(96, 32, rank=r, world=2)
        s.set_codebook(cb)
        for a in range(0, 20_001, 7_000):      # several add batches -> several id ranges per shard
            s.add(x[a:a + 7_000])
        s.add(x[:0])
        shards.append(s)
    qt = torch.from_numpy(q).cuda()
    S = gen.subset(20_001, 5_000, seed=3)
    for sub in (None, S):
        parts = torch.stack([s.query_partial(qt, 50, target_ids=sub, path="linear")[0] for s in shards])
        ids, dist = rii.merge_partials(parts, 50)
        ids, dist = ids.cpu().numpy(), dist.cpu().numpy()
        ref_ids, ref_d, _ = single.query(q, 50, target_ids=sub, path="linear")
        assert np.array_equal(ids, ref_ids) and np.array_equal(dist, ref_d)
        assert_topk_parity(ref, o.cb, o.codes, q, (ids, dist), o.query(q, 50, S=sub, path=1), S=sub, what="shards")
    with pytest.raises(rii.RiiError) as e:
        shards[0].query(q, 5)
    assert e.value.status == 2
    # shard persistence (RIIS): reload both shards, same partials
    for s in shards:
        s.set_centers(ref.reconfigure(o.cb, o.codes, 16, 2, 0)[0])
    loaded = []
    for r, s in enumerate(shards):
        p = str(tmp_path / f"s{r}.rii")
        s.save(p)
        raw = open(p, "rb").read()
        assert raw[:4] == b"RIIS"
        loaded.append(rii.Index.load(p))
        assert loaded[-1].info() == s.info() and (loaded[-1].rank, loaded[-1].world) == (r, 2)
        # corrupt the first posting offset (must be 0)
        nseg = struct.unpack_from("<I", raw, 36)[0]
        n_local, K = struct.unpack_from("<qq", raw, 48)
        off0 = 88 + 256 * 96 * 4 + 24 * nseg + n_local * 32 + K * 32
        assert struct.unpack_from("<q", raw, off0)[0] == 0
        bad = bytearray(raw)
        struct.pack_into("<q", bad, off0, 7)
        (tmp_path / "bad.rii").write_bytes(bytes(bad))
        with pytest.raises(rii.RiiError) as e:
            rii.Index.load(str(tmp_path / "bad.rii"))
        assert e.value.status == 1
    for sub in (None, S):
        for path, L in (("linear", 1), ("ivf", 3)):
            a = [s.query_partial(qt, 50, target_ids=sub, L=L, path=path)[0] for s in shards]
            b = [s.query_partial(qt, 50, target_ids=sub, L=L, path=path)[0] for s in loaded]
            assert all(torch.equal(u, v) for u, v in zip(a, b))


def test_theta_calibration(rii, ref):
    """Alg. 3 threshold fitted from GPU timings: a line theta(L) = aL + b
    whose value is machine-dependent (parity unpinned); checked for sanity and for the
    rule |S| < theta -> linear, applied with the fitted value."""
    import torch
    N, D, M = 200_000, 96, 32
    x = torch.from_numpy(gen.deep_like(N, D, seed=31)).cuda()
    q = torch.from_numpy(gen.deep_like(256, D, seed=31, stream=gen.STREAM_QUERY)).cuda()
    g = rii.Index(D, M)
    g.train(x[:20_000], n_iter=2, seed=0)
    g.add(x)
    g.reconfigure(447, n_iter=3, seed=0)
    a, b, cross = g.calibrate_theta(q, topk=100, L_grid=(1, 4, 16))
    assert np.isfinite(a) and np.isfinite(b)
    assert ((cross >= 0) & (cross <= N)).all()
    for L in (1, 4, 16):
        th = int(max(0.0, np.ceil(a * L + b)))
        if th >= 8:
            S = np.arange(0, N, N // (th // 2))[: th // 2].astype(np.int64)
            assert g.query(q[:4], 10, target_ids=S, L=L)[2] == rii.PATH_LINEAR
        if 2 * th <= N:
            S = np.arange(0, N, max(1, N // (2 * th)))[: 2 * th].astype(np.int64)
            assert g.query(q[:4], 10, target_ids=S, L=L)[2] == rii.PATH_IVF
    g.set_theta(-1)  # back to the analytic default (R3)
    assert g.query(q[:4], 10, L=1)[2] == rii.PATH_IVF


@pytest.mark.parametrize("kind,N,D,M,K", [("deep", 20_011, 96, 32, 30), ("sift", 15_000, 128, 16, 40),
                                          ("deep", 9_001, 96, 12, 10)])
def test_ivf_paper_mode(rii, ref, kind, N, D, M, K):
    """Alg. 2 as printed (RII_IVF_PAPER): L = candidate budget, ceil(KL/|S|) lists in
    (d0, k) order, early stop at |U| = L -- against oracle rref_ivf_paper."""
    x = gen.base(kind, N, D, seed=N + 1)
    q = gen.base(kind, 23, D, seed=N + 1, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, M, K, n_iter=3, train_rows=x[:3000], train_iter=3)
    g.set_ivf_mode("paper")
    for sub in (None, gen.subset(N, N // 4, seed=9), gen.subset(N, 150, seed=10)):
        for L in (1, 50, 700, N):
            gr = g.query(q, 50, target_ids=sub, L=L, path="ivf")
            orr = ref.ivf_paper(o.cb, o.codes, o.centers, o.offsets, o.ids, q, 50, L, S=sub)
            assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"paper {kind} L={L}")
    # AUTO default threshold in paper mode: theta(L) = L + K
    S = gen.subset(N, 200 + K - 1, seed=11)
    assert g.query(q[:2], 5, target_ids=S, L=200)[2] == rii.PATH_LINEAR
    S = gen.subset(N, 200 + K, seed=12)
    assert g.query(q[:2], 5, target_ids=S, L=200)[2] == rii.PATH_IVF
    g.set_ivf_mode("lists")
    assert g.query(q[:2], 5, L=2)[2] == rii.PATH_IVF


@pytest.mark.parametrize("M,K", [(8, 9_000), (16, 8_192), (32, 1_000)])
def test_assignment_paths_large_k(rii, ref, M, K):
    """a(n) = argmin_k d_S for installed centres: K >= 8192 takes the
    SDC-mode packed scan (codes as queries over the centre codes), smaller K the
    rotated-table kernel with canonical near-tie fallback.  Bit-exact vs the oracle."""
    D = 96 if M != 16 else 128
    kind = "deep" if M != 16 else "sift"
    x = gen.base(kind, 20_000, D, seed=K + M)
    g = rii.Index(D, M)
    g.train(x[:4000], n_iter=2, seed=0)
    cb = g.get_codebook()
    g.add(x)
    codes = g.get_codes()
    assert np.array_equal(codes, ref.encode(cb, x, M))
    rng = np.random.default_rng(K)
    centers = codes[rng.choice(len(codes), K, replace=False)].copy()
    centers[1] = centers[0]            # duplicate centre: exact ties must go to the lower k
    g.set_centers(centers)
    T = ref.sdc_tables(cb, D, M)
    a, _ = ref.assign(T, codes, centers)
    off, ids = g.get_postings()
    want_off, want_ids = ref.build_postings(a, K)
    assert np.array_equal(off, want_off) and np.array_equal(ids, want_ids)


def _parse_spec_rii1(raw):
    """SPEC's persistence layout, read independently of the library."""
    import struct
    assert raw[:4] == b"RII1"
    version, D, M, Z, N, K = struct.unpack_from("<6I", raw, 4)
    theta, = struct.unpack_from("<Q", raw, 28)
    default_L, flags = struct.unpack_from("<2I", raw, 36)
    o = 44
    cb = np.frombuffer(raw, "<f4", M * Z * (D // M), o).reshape(M, Z, D // M)
    o += cb.nbytes
    R = None
    if flags & 1:
        R = np.frombuffer(raw, "<f4", D * D, o).reshape(D, D)
        o += R.nbytes
    codes = np.frombuffer(raw, np.uint8, N * M, o).reshape(N, M)
    o += codes.nbytes
    centers = np.frombuffer(raw, np.uint8, K * M, o).reshape(K, M)
    o += centers.nbytes
    lists = []
    for _ in range(K):
        n, = struct.unpack_from("<I", raw, o)
        lists.append(np.frombuffer(raw, "<u4", n, o + 4).astype(np.int64))
        o += 4 + 4 * n
    return dict(version=version, D=D, M=M, Z=Z, N=N, K=K, theta=theta, default_L=default_L, flags=flags, cb=cb,
                R=R, codes=codes, centers=centers, lists=lists, end=o)


def test_save_load_roundtrip(rii, ref, tmp_path):
    """Persistence: a single-GPU index is written in SPEC's RII1 layout bit
    for bit (parsed here independently); load(save(idx)) answers identically; save ->
    load -> save is byte-identical; the payload is (N+K)M + 4N (+4K list lengths)
    bytes plus header and code book; malformed files (truncated, bad magic,
    corrupted posting lists) are rejected before anything reaches the device."""
    import struct
    N, D, M, K = 20_000, 128, 16, 64
    x = gen.sift_like(N, D, seed=51)
    q = gen.sift_like(17, D, seed=51, stream=gen.STREAM_QUERY)
    g = rii.Index(D, M)
    g.train(x[:5000], n_iter=3, seed=0)
    g.add(x)
    g.reconfigure(K, n_iter=3, seed=0)
    g.set_theta(4321)
    p1, p2 = str(tmp_path / "a.rii"), str(tmp_path / "b.rii")
    g.save(p1)
    raw = open(p1, "rb").read()
    f = _parse_spec_rii1(raw)
    assert (f["version"], f["D"], f["M"], f["Z"], f["N"], f["K"], f["theta"], f["flags"]) == (1, D, M, 256, N, K, 4321, 0)
    assert f["end"] == len(raw)  # no extension block: ivf_mode 0, theta not fitted
    assert np.array_equal(f["cb"], g.get_codebook()) and np.array_equal(f["codes"], g.get_codes())
    assert np.array_equal(f["centers"], g.get_centers())
    off, ids = g.get_postings()
    assert all(np.array_equal(f["lists"][k], ids[off[k]:off[k + 1]]) for k in range(K))
    assert len(raw) == 44 + 256 * D * 4 + (N + K) * M + 4 * N + 4 * K
    h = rii.Index.load(p1)
    assert h.info() == g.info()
    for path, L, S in (("linear", 1, None), ("ivf", 3, None), ("auto", 2, gen.subset(N, 4000, seed=1))):
        a, b = g.query(q, 20, S, L=L, path=path), h.query(q, 20, S, L=L, path=path)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    h.save(p2)
    assert open(p2, "rb").read() == raw
    # analytic theta (flags bit 1) and the extension block (paper-mode Alg. 2)
    g.set_theta(-1)
    g.set_ivf_mode("paper")
    g.save(p1)
    raw2 = open(p1, "rb").read()
    f2 = _parse_spec_rii1(raw2)
    assert f2["flags"] == 2 and f2["theta"] == 0 and raw2[f2["end"]:f2["end"] + 4] == b"RIIX"
    h2 = rii.Index.load(p1)
    assert h2.info()["theta"] == -1
    a, b = g.query(q, 20, L=300, path="ivf"), h2.query(q, 20, L=300, path="ivf")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # malformed files
    lists0 = 44 + 256 * D * 4 + (N + K) * M     # first posting list: u32 length, then ids
    n0, = struct.unpack_from("<I", raw, lists0)
    bad = {"t.rii": raw[:-10], "m.rii": b"XXXX" + raw[4:], "x.rii": raw + b"\0"}
    r = bytearray(raw); struct.pack_into("<I", r, lists0 + 4, N + 5); bad["range.rii"] = bytes(r)       # id >= N
    r = bytearray(raw); struct.pack_into("<I", r, lists0 + 8, struct.unpack_from("<I", raw, lists0 + 4)[0])
    bad["dup.rii"] = bytes(r)                                                                             # repeated id
    r = bytearray(raw); struct.pack_into("<I", r, lists0, n0 + 1); bad["len.rii"] = bytes(r)            # lengths != N
    r = bytearray(raw); struct.pack_into("<I", r, 8, 100); bad["shape.rii"] = bytes(r)                    # D % M != 0
    for name, data in bad.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(rii.RiiError) as e:
            rii.Index.load(str(tmp_path / name))
        assert e.value.status == 1, name


# ------------------------------------------------- u16 fixed-point tables ---# ------------------------------------------------- u16 fixed-point tables ---
@pytest.mark.parametrize("kind,N,D,M,nq,topk", [("deep", 40_009, 96, 32, 45, 100), ("sift", 33_333, 128, 16, 19, 64),
                                                ("sift", 30_011, 128, 64, 21, 100),  # two table halves
                                                ("deep", 20_011, 96, 8, 23, 10), ("gaussian", 17_003, 32, 4, 9, 100)])
def test_linear_u16_tables(rii, ref, monkeypatch, kind, N, D, M, nq, topk):
    """The u16 fixed-point SWAR scan (sampled kk-th bound, integer filter, canonical
    rescore) must return exactly the oracle's Alg. 1 result, whole and subset; the
    threshold RII_Q16_MIN=1 forces it onto these small sizes (several chunks, ragged
    tails, query batches not a multiple of 8)."""
    monkeypatch.setenv("RII_Q16_MIN", "1")
    x = gen.base(kind, N, D, seed=N)
    q = gen.base(kind, nq, D, seed=N, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, M, 0, train_rows=x[:4000], train_iter=3)
    for sub in (None, gen.subset(N, N // 2 + 1, seed=3)):
        gr = g.query(q, topk, target_ids=sub, path="linear")
        orr = o.query(q, topk, S=sub, path=1)
        assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"u16 {kind} M={M}")
        monkeypatch.setenv("RII_Q16", "0")  # the bf16 / fp32 path gives the identical answer
        g2 = g.query(q, topk, target_ids=sub, path="linear")
        monkeypatch.delenv("RII_Q16")
        assert np.array_equal(gr[0], g2[0]) and np.array_equal(gr[1], g2[1])
        for cfg in ("0", "4", "9"):  # u16, u6 (8 queries) and u6 (16 queries) tables (the default picks by M)
            monkeypatch.setenv("RII_Q16_CFG", cfg)
            g3 = g.query(q, topk, target_ids=sub, path="linear")
            monkeypatch.delenv("RII_Q16_CFG")
            assert np.array_equal(gr[0], g3[0]) and np.array_equal(gr[1], g3[1]), f"cfg {cfg}"
        if M == 8:  # the L2-prefetching variant of long M = 8 scans (forced onto this size)
            monkeypatch.setenv("RII_LIN_PF_MIN", "1")
            g4 = g.query(q, topk, target_ids=sub, path="linear")
            monkeypatch.delenv("RII_LIN_PF_MIN")
            assert np.array_equal(gr[0], g4[0]) and np.array_equal(gr[1], g4[1])
            # the 384-thread configuration of the 16-query kernel (default: 512), with and without prefetch
            for env in ({"RII_M8_NTH": "384", "RII_Q16_CFG": "9"},
                        {"RII_M8_NTH": "384", "RII_Q16_CFG": "9", "RII_LIN_PF_MIN": "1"},
                        {"RII_Q16_CFG": "9", "RII_LIN_PF_MIN": "1"}):
                for k, v in env.items():
                    monkeypatch.setenv(k, v)
                g5 = g.query(q, topk, target_ids=sub, path="linear")
                for k in env:
                    monkeypatch.delenv(k)
                assert np.array_equal(gr[0], g5[0]) and np.array_equal(gr[1], g5[1]), env
        if M == 64:  # the u6 kernel at 384 threads (A/B variant) equals the default 256
            for env in ({"RII_M64_NTH": "384"},):
                for k, v in env.items():
                    monkeypatch.setenv(k, v)
                g4 = g.query(q, topk, target_ids=sub, path="linear")
                for k in env:
                    monkeypatch.delenv(k)
                assert np.array_equal(gr[0], g4[0]) and np.array_equal(gr[1], g4[1]), env


def test_linear_u16_duplicates_and_zero_distance(rii, ref, monkeypatch):
    """Ties and T = 0: every code repeated 60 times (one 8-query batch sees > NEWCAP
    equal candidates per step window) and queries equal to stored vectors in the
    lossless case (kk-th bound 0, scale clamp)."""
    monkeypatch.setenv("RII_Q16_MIN", "1")
    base = gen.deep_like(300, 96, seed=9)
    x = np.concatenate([base] * 60)
    q = np.concatenate([gen.deep_like(7, 96, seed=9, stream=gen.STREAM_QUERY), base[:5]])
    g, o = _build_pair(rii, ref, x, 32, 0, train_rows=x[:3000], train_iter=2)
    gr = g.query(q, 100, path="linear")
    orr = o.query(q, 100, path=1)
    assert np.array_equal(gr[0], orr[0]) and np.array_equal(gr[1], orr[1])
    xl = np.concatenate([gen.lossless(300, 16, seed=5)] * 200)  # >= 32 zero-distance copies in the sample
    cb = np.tile(np.arange(256, dtype=np.float32)[None, :, None], (16, 1, 1))
    gl = rii.Index(16, 16)
    gl.set_codebook(cb)
    gl.add(xl)
    ql = np.concatenate([xl[:6], np.random.default_rng(5).integers(0, 256, size=(6, 16)).astype(np.float32)])
    ids, dist, _ = gl.query(ql, 10, path="linear")
    for i in range(len(ql)):
        d = ((xl.astype(np.int64) - ql[i].astype(np.int64)) ** 2).sum(1)
        order = np.lexsort((np.arange(len(xl)), d))[:10]
        assert np.array_equal(ids[i], order) and np.array_equal(dist[i], d[order].astype(np.float32))


# ------------------------------------------------------------ OPQ (Rii-OPQ) ---
def _orthogonal(D, seed):
    Q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(D, D)))
    return Q.astype(np.float32)


@pytest.mark.parametrize("D,n", [(96, 1001), (128, 37), (30, 300)])
def test_rotate_kernel_bit_exact(rii, ref, D, n):
    """rotate_kernel (canonical order CR) equals the oracle's rref_rotate bit for bit."""
    import torch
    R = _orthogonal(D, D)
    x = gen.base("deep", n, D, seed=D)
    g = rii.Index(D, 1 if D == 30 else 32 if D == 96 else 16)
    g.set_rotation(R)
    y = g.rotate(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y, ref.rotate(R, x))
    Rg, has = g.get_rotation()
    assert has and np.array_equal(Rg, R)


def test_opq_pipeline_matches_oracle(rii, ref):
    """Rii-OPQ with a given rotation: train, add, reconfigure and every
    query path on R x equal the oracle's, bit for bit where bit-exact is required."""
    D, M, K, N = 96, 32, 12, 20_011
    R = _orthogonal(D, 5)
    x = gen.base("deep", N, D, seed=5)
    q = gen.base("deep", 23, D, seed=5, stream=gen.STREAM_QUERY)
    g = rii.Index(D, M)
    g.set_rotation(R)
    g.train(x[:4000], n_iter=3, seed=0)
    g.add(x)
    g.reconfigure(K, n_iter=3, seed=0)
    o = ref.OracleIndex(D, M)
    o.R = R
    o.train(x[:4000], n_iter=3, seed=0)
    o.add(x)
    o.reconfigure(K, n_iter=3, seed=0)
    assert np.array_equal(g.get_codebook(), o.cb)
    assert np.array_equal(g.get_codes(), o.codes)
    assert np.array_equal(g.get_centers(), o.centers)
    S = gen.subset(N, 3001, seed=1)
    for path in ("linear", "ivf"):
        for sub in (None, S):
            gr = g.query(q, 50, target_ids=sub, L=3, path=path)
            orr = o.query(q, 50, S=sub, L=3, path=1 if path == "linear" else 2)
            assert_topk_parity(ref, o.cb, o.codes, ref.rotate(R, q), gr, orr, S=sub, what=f"opq {path}")


def test_train_opq_properties(rii, ref, tmp_path):
    """rii_train_opq: R orthogonal, deterministic, and the quantisation distortion
    of R x is below plain PQ's on data whose energy is concentrated in a few
    rotated directions (the case OPQ targets); save/load keeps R."""
    D, M, n = 32, 8, 8000
    rng = np.random.default_rng(3)
    scales = (2.0 ** (-np.arange(D) / 3.0)).astype(np.float32)
    x = ((rng.normal(size=(n, D)) * scales) @ _orthogonal(D, 9).T).astype(np.float32) * 10
    g = rii.Index(D, M)
    g.train_opq(x, n_opq_iter=6, n_iter=10, seed=1)
    R, has = g.get_rotation()
    assert has and np.abs(R.astype(np.float64) @ R.T.astype(np.float64) - np.eye(D)).max() < 1e-4
    g2 = rii.Index(D, M)
    g2.train_opq(x, n_opq_iter=6, n_iter=10, seed=1)
    assert np.array_equal(g2.get_rotation()[0], R) and np.array_equal(g2.get_codebook(), g.get_codebook())
    p = rii.Index(D, M)
    p.train(x, n_iter=10, seed=1)

    def distortion(idx, rot):
        cb = idx.get_codebook()
        xr = ref.rotate(rot, x) if rot is not None else x
        rec = ref.decode(cb, ref.encode(cb, xr, M), D)
        return float(((xr.astype(np.float64) - rec) ** 2).sum(1).mean())

    d_opq, d_pq = distortion(g, R), distortion(p, None)
    assert d_opq < 0.9 * d_pq, (d_opq, d_pq)
    g.add(x)
    q = x[:5]
    r1 = g.query(q, 10, path="linear")
    g.save(str(tmp_path / "opq.rii"))
    h = rii.Index.load(str(tmp_path / "opq.rii"))
    assert np.array_equal(h.get_rotation()[0], R)
    r2 = h.query(q, 10, path="linear")
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])


# ------------------------------------------------------- large M (F3) -------
@pytest.mark.parametrize("kind,N,D,M,K,nq,topk", [("deep", 3_001, 960, 240, 6, 7, 20),  # GIST1M shape
                                                  ("sift", 4_003, 384, 192, 8, 9, 50),  # MET-like M = 192
                                                  ("gaussian", 2_503, 140, 70, 5, 5, 10),  # M % 4 != 0
                                                  ("sift", 4_001, 128, 64, 8, 9, 50)])  # SIFT1M Table 2 shape
def test_large_m_shapes(rii, ref, kind, N, D, M, K, nq, topk):
    """M > 64 (the paper's range reaches M = 240): train,
    add, reconfigure (large-M SDC assignment) and every query path (linear whole /
    subset, IVF mode A, IVF paper mode with its early stop) equal the oracle's."""
    x = gen.base(kind, N, D, seed=N)
    q = gen.base(kind, nq, D, seed=N, stream=gen.STREAM_QUERY)
    g, o = _build_pair(rii, ref, x, M, K, n_iter=2, train_rows=x, train_iter=2)
    _check_state(g, o)
    S = gen.subset(N, N // 3, seed=4)
    for path in ("linear", "ivf"):
        for sub in (None, S):
            for L in (1, 3):
                gr = g.query(q, topk, target_ids=sub, L=L, path=path)
                orr = o.query(q, topk, S=sub, L=L, path=1 if path == "linear" else 2)
                assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"M={M} {path} L={L}")
    g.set_ivf_mode("paper")
    Lc = N // K
    gr = g.query(q, topk, L=Lc, path="ivf")
    orr = ref.ivf_paper(o.cb, o.codes, o.centers, o.offsets, o.ids, q, topk, Lc)
    assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, what=f"M={M} paper L={Lc}")


@pytest.mark.parametrize("kind,N,D,M,nq,topk", [("deep", 40_003, 960, 240, 21, 100),   # GIST1M shape
                                                ("sift", 50_001, 384, 192, 13, 50),    # MET-like M = 192
                                                ("deep", 30_011, 384, 96, 9, 10)])
def test_large_m_u6_chunk_kernel(rii, ref, monkeypatch, kind, N, D, M, nq, topk):
    """The large-M linear scan on chunked u6 oct tables (k_large_u6.cu; M > 64,
    M % 16 == 0): whole database and a large subset (both on the chunk kernel) and
    a small subset (the one-query kernel), element by element against the oracle's
    Alg. 1; several code chunks per query batch and a ragged last tile."""
    monkeypatch.setenv("RII_LARGE_U6_MIN", "8000")
    x = gen.base(kind, N, D, seed=N)
    q = gen.base(kind, nq, D, seed=N, stream=gen.STREAM_QUERY)
    cb = ref.train(x[:3000], M, n_iter=2, seed=0)
    g = rii.Index(D, M)
    g.set_codebook(cb)
    g.add(x)
    codes = ref.encode_mt(cb, x, M)
    assert np.array_equal(g.get_codes(), codes)
    lib = rii.load()
    lib.rii_kernel_timing(1)
    for sub in (None, gen.subset(N, N // 2 + 7, seed=3), gen.subset(N, 999, seed=4)):
        gr = g.query(q, topk, target_ids=sub, path="linear")
        assert_topk_parity(ref, cb, codes, q, gr, ref.linear_mt(cb, codes, q, topk, S=sub), S=sub,
                           what=f"large u6 M={M} |S|={'N' if sub is None else len(sub)}")
    import ctypes as C
    ms, n = C.c_double(), C.c_int64()
    lib.rii_kernel_timing_read(6, C.byref(ms), C.byref(n))  # u6 launches: the chunk kernel ran (two passes)
    lib.rii_kernel_timing(0)
    assert n.value == 4
