"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it follows and pins the oracle to something other
than itself: closed forms, invariants, brute force on tiny inputs, special cases
that reduce to textbook routines, and values printed in the paper.
"""
import itertools
import math
import os

import numpy as np
import pytest

from synth import generators as gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _rand_cb(M, Z, ds, seed):
    return np.random.default_rng(seed).standard_normal((M, Z, ds)).astype(np.float32)


# ----------------------------------------------------------------- hashing ---
def test_splitmix64_published_value(ref):
    for state, hexout in _rows("splitmix64.txt"):
        assert ref.splitmix64(int(state)) == int(hexout, 16)


# ------------------------------------------------------------------ encode ---
def test_encode_worked_example(ref):
    rows = {r[0]: [float(v) for v in r[1:]] for r in _rows("encode_worked_example.txt")}
    cb = np.array(rows["cb"], np.float32).reshape(2, 2, 2)
    x = np.array([rows["x"]], np.float32)
    assert ref.encode(cb, x, M=2, Z=2).tolist() == [[int(v) for v in rows["code"]]]


def test_encode_is_exhaustive_argmin(ref):
    """Eq. 1: brute-force nearest code word per sub-vector (fp64 from the
    reconstruction), ties to the lowest index (CA4)."""
    M, Z, ds = 4, 16, 3
    cb = _rand_cb(M, Z, ds, 1)
    x = np.random.default_rng(2).standard_normal((100, M * ds)).astype(np.float32)
    codes = ref.encode(cb, x, M, Z)
    for i in range(len(x)):
        for m in range(M):
            d = ((x[i, m * ds:(m + 1) * ds].astype(np.float64)[None, :] - cb[m].astype(np.float64)) ** 2).sum(1)
            c = codes[i, m]
            assert d[c] <= d.min() * (1 + 1e-6)
            # ties resolve to the lowest index
            assert not any(d[z] < d[c] * (1 - 1e-6) for z in range(Z))


def test_encode_decode_roundtrip_exhaustive(ref):
    """S:87 / S:130: encode(decode(c)) == c for every code (M=2, Z=4, distinct words)."""
    M, Z, ds = 2, 4, 2
    cb = _rand_cb(M, Z, ds, 3)
    codes = np.array(list(itertools.product(range(Z), repeat=M)), np.uint8)
    x = ref.decode(cb, codes, M * ds, Z)
    assert np.array_equal(ref.encode(cb, x, M, Z), codes)


# --------------------------------------------------------------- LUT / ADC ---
def test_lut_closed_forms(ref):
    """A(m,z) = ||q_m - c_{m,z}||^2.  q = 0 gives ||c||^2; q equal to
    a code-word concatenation gives an exact 0 at that code."""
    M, Z, ds = 4, 256, 8
    cb = _rand_cb(M, Z, ds, 4)
    A = ref.lut(cb, np.zeros(M * ds, np.float32), M, Z)
    norms = (cb.astype(np.float64) ** 2).sum(-1)
    assert np.allclose(A, norms, rtol=4e-7 * ds, atol=0)
    code = np.array([[7, 200, 0, 255]], np.uint8)
    q = ref.decode(cb, code, M * ds, Z)[0]
    A = ref.lut(cb, q, M, Z)
    assert all(A[m, code[0, m]] == 0.0 for m in range(M))
    assert ref.adc(A, code[0]) == 0.0


def test_adc_equals_reconstruction_distance(ref):
    """Eq. 2, BASELINE.json invariant 1: d_A(q, xbar) = ||q - decode(xbar)||^2."""
    M, Z, ds = 8, 256, 4
    cb = _rand_cb(M, Z, ds, 5)
    g = np.random.default_rng(6)
    codes = g.integers(0, Z, size=(200, M)).astype(np.uint8)
    rec = ref.decode(cb, codes, M * ds, Z).astype(np.float64)
    for t in range(5):
        q = g.standard_normal(M * ds).astype(np.float32)
        A = ref.lut(cb, q, M, Z)
        A64 = ref.lut64(cb, q, M, Z)
        exact = ((rec - q.astype(np.float64)) ** 2).sum(1)
        for i in range(len(codes)):
            assert abs(ref.adc(A, codes[i]) - exact[i]) <= 1e-5 * exact[i]
            assert abs(ref.adc64(A64, codes[i]) - exact[i]) <= 1e-12 * exact[i]
    A = ref.lut(cb, g.standard_normal(M * ds).astype(np.float32)[None, :][0], M, Z)
    assert ref.adc(A[:1], codes[0, :1]) == A[0, codes[0, 0]]   # M = 1


def test_sdc_tables(ref):
    """d_S: symmetric, zero diagonal, = ||decode(a)-decode(b)||^2."""
    M, Z, ds = 2, 256, 5
    cb = _rand_cb(M, Z, ds, 7)
    T = ref.sdc_tables(cb, M * ds, M, Z)
    assert np.array_equal(T, np.transpose(T, (0, 2, 1)))
    assert all((np.diagonal(T[m]) == 0).all() for m in range(M))
    g = np.random.default_rng(8)
    for _ in range(50):
        a, b = g.integers(0, Z, size=(2, M)).astype(np.uint8)
        ra, rb = ref.decode(cb, np.stack([a, b]), M * ds, Z).astype(np.float64)
        exact = ((ra - rb) ** 2).sum()
        assert abs(ref.sdc(T, a, b) - exact) <= 1e-5 * exact
        assert ref.sdc(T, a, b) == ref.sdc(T, b, a)


# ------------------------------------------------------------ linear scan ----
def _lossless_setup(n=3000, D=8, seed=0):
    """C-PIN7: D = M (ds = 1), Z = 256, code book {0..255} per dimension, integer data:
    PQ is lossless and ADC equals the exact squared distance."""
    x = gen.lossless(n, D, seed)
    cb = np.tile(np.arange(256, dtype=np.float32)[None, :, None], (D, 1, 1))
    return x, cb


def test_linear_lossless_equals_textbook_knn(ref):
    """Alg. 1 + Eq. 3: in the lossless case the PQ linear scan is
    exact kNN; compared with a plain numpy brute force (argsort by (d, id))."""
    x, cb = _lossless_setup()
    D = x.shape[1]
    codes = ref.encode(cb, x, D)
    assert np.array_equal(codes, x.astype(np.uint8))
    q = np.random.default_rng(9).integers(0, 256, size=(20, D)).astype(np.float32)
    ids, dist = ref.linear(cb, codes, q, topk=50)
    for i in range(len(q)):
        d = ((x.astype(np.int64) - q[i].astype(np.int64)) ** 2).sum(1)
        order = np.lexsort((np.arange(len(x)), d))[:50]
        assert np.array_equal(ids[i], order)
        assert np.array_equal(dist[i], d[order].astype(np.float32))


def test_subset_equals_filtered_whole(ref):
    """Eq. 3 with S, BASELINE.json invariant 3: subset search = whole ranking
    filtered to S; singleton S; containment; padding when topk > |S| (R18)."""
    M, Z, ds, N = 4, 256, 4, 2000
    cb = _rand_cb(M, Z, ds, 10)
    codes = np.random.default_rng(11).integers(0, Z, size=(N, M)).astype(np.uint8)
    q = np.random.default_rng(12).standard_normal((5, M * ds)).astype(np.float32)
    wid, wd = ref.linear(cb, codes, q, topk=N)
    for size in (1, 10, 1000):
        S = gen.subset(N, size, seed=size)
        sid, sd = ref.linear(cb, codes, q, topk=20, S=S)
        for i in range(len(q)):
            keep = np.isin(wid[i], S)
            exp_ids, exp_d = wid[i][keep][:20], wd[i][keep][:20]
            k = len(exp_ids)
            assert np.array_equal(sid[i, :k], exp_ids) and np.array_equal(sd[i, :k], exp_d)
            assert (sid[i, k:] == -1).all() and np.isinf(sd[i, k:]).all()
    with pytest.raises(ref.OracleError):
        ref.linear(cb, codes, q, topk=5, S=np.array([3, 3], np.int64))   # R6: strictly ascending


# ---------------------------------------------------------------------- IVF --
def _small_index(ref, N=2000, M=4, K=20, seed=13):
    ds = 4
    x = gen.gaussian(N, M * ds, seed=seed)
    idx = ref.OracleIndex(M * ds, M)
    idx.train(x, n_iter=5, seed=seed)
    idx.add(x)
    idx.reconfigure(K, n_iter=5, seed=seed)
    return idx, x


def test_num_probe_formula(ref):
    """P:492-502 (budget ceil(K L / |S|), capped at K) under reading R1 (L in lists)."""
    assert ref.num_probe(10_000, 100, 10_000, False, 8) == 8
    assert ref.num_probe(10_000, 100, 10_000, False, 500) == 100
    assert ref.num_probe(10_000, 100, 1_000, True, 8) == 80           # ceil(8*1e4/1e3)
    assert ref.num_probe(10_000, 100, 3_000, True, 8) == 27           # ceil(26.67)
    assert ref.num_probe(10_000, 100, 10, True, 8) == 100             # capped at K
    assert ref.default_theta(10_000, 100, 8) == 900                   # R3


def test_ivf_all_lists_equals_linear(ref):
    """BASELINE.json invariant 2 / S:326: L = nlist probes every list -> linear scan."""
    idx, _ = _small_index(ref)
    q = gen.gaussian(10, idx.D, seed=14, stream=gen.STREAM_QUERY)
    lid, ld = ref.linear(idx.cb, idx.codes, q, topk=30)
    vid, vd = ref.ivf(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, topk=30, L=idx.K)
    assert np.array_equal(lid, vid) and np.array_equal(ld, vd)
    S = gen.subset(idx.N, 300, seed=15)
    lid, ld = ref.linear(idx.cb, idx.codes, q, topk=30, S=S)
    vid, vd = ref.ivf(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, topk=30, L=idx.K, S=S)
    assert np.array_equal(lid, vid) and np.array_equal(ld, vd)


def test_ivf_single_list_degenerates(ref):
    """K = 1 -> the one posting list holds every id -> linear scan."""
    idx, _ = _small_index(ref, K=1)
    q = gen.gaussian(5, idx.D, seed=16, stream=gen.STREAM_QUERY)
    assert np.array_equal(ref.linear(idx.cb, idx.codes, q, 10)[0],
                          ref.ivf(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, 10, L=1)[0])


def test_ivf_is_linear_over_nearest_lists(ref):
    """Alg. 2 L2-L13 (mode A, R2): the result is the linear scan restricted to the members
    of the P lists whose centres are nearest by ADC; the nearest lists are found here
    from the reconstruction distance ||q - decode(cbar_k)||^2 in fp64 (Eq. 2), and
    cases with a near-tie at the P-th list are skipped."""
    idx, _ = _small_index(ref, K=40)
    rec = ref.decode(idx.cb, idx.centers, idx.D).astype(np.float64)
    q = gen.gaussian(30, idx.D, seed=17, stream=gen.STREAM_QUERY)
    checked = 0
    for L in (1, 3, 7):
        for S in (None, gen.subset(idx.N, 500, seed=L)):
            P = ref.num_probe(idx.N, idx.K, 0 if S is None else len(S), S is not None, L)
            vid, vd = ref.ivf(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, 25, L=L, S=S)
            for i in range(len(q)):
                d0 = ((rec - q[i].astype(np.float64)) ** 2).sum(1)
                order = np.argsort(d0, kind="stable")
                if P < idx.K and abs(d0[order[P]] - d0[order[P - 1]]) < 1e-5 * d0[order[P]]:
                    continue
                members = np.sort(np.concatenate([idx.ids[idx.offsets[k]:idx.offsets[k + 1]] for k in order[:P]]))
                if S is not None:
                    members = members[np.isin(members, S)]
                lid, ld = ref.linear(idx.cb, idx.codes, q[i:i + 1], 25, S=members)
                assert np.array_equal(lid[0], vid[i]) and np.array_equal(ld[0], vd[i])
                assert np.isin(vid[i][vid[i] >= 0], S if S is not None else np.arange(idx.N)).all()
                checked += 1
    assert checked > 100


def test_query_path_rule(ref):
    """Alg. 3: |S| < theta -> linear, else inverted index; K = 0 -> linear."""
    idx, _ = _small_index(ref)
    q = gen.gaussian(3, idx.D, seed=18, stream=gen.STREAM_QUERY)
    th = ref.default_theta(idx.N, idx.K, 2)
    for size, want in ((th - 1, ref.PATH_LINEAR), (th, ref.PATH_IVF)):
        S = gen.subset(idx.N, size, seed=size)
        assert idx.query(q, 5, S=S, L=2)[2] == want
    assert idx.query(q, 5, L=2)[2] == ref.PATH_IVF            # S = ALL, N >= theta
    idx.theta = idx.N + 1
    assert idx.query(q, 5, L=2)[2] == ref.PATH_LINEAR
    empty = ref.OracleIndex(idx.D, idx.M)
    empty.cb = idx.cb
    empty.add(gen.gaussian(50, idx.D, seed=19))
    assert empty.query(q, 5, L=2)[2] == ref.PATH_LINEAR


# -------------------------------------------------- assignment / postings ----
def test_assignment_is_exhaustive_nearest_center(ref):
    """a(n) = argmin_k d_S(xbar_n, cbar_k), brute force (fp64 reconstruction
    distance), N <= 2000; W partitions the ids, ascending (Eq. 4, R11)."""
    idx, _ = _small_index(ref, K=25)
    rx = ref.decode(idx.cb, idx.codes, idx.D).astype(np.float64)
    rc = ref.decode(idx.cb, idx.centers, idx.D).astype(np.float64)
    d = ((rx[:, None, :] - rc[None, :, :]) ** 2).sum(-1)
    chosen = d[np.arange(idx.N), idx.assign]
    assert (chosen <= d.min(1) * (1 + 1e-6) + 1e-12).all()
    assert np.array_equal(np.sort(idx.ids), np.arange(idx.N))
    for k in range(idx.K):
        lst = idx.ids[idx.offsets[k]:idx.offsets[k + 1]]
        assert (np.diff(lst) > 0).all() and (idx.assign[lst] == k).all()


def test_add_appends_and_assigns(ref):
    """PushBack(Xbar, ybar); PushBack(W_a(N+1), N+1); existing ids unchanged."""
    idx, _ = _small_index(ref, K=10)
    before = idx.codes.copy()
    y = gen.gaussian(100, idx.D, seed=20, stream=gen.STREAM_QUERY)
    first = idx.add(y)
    assert first == len(before) and np.array_equal(idx.codes[:first], before)
    T = ref.sdc_tables(idx.cb, idx.D, idx.M)
    for n in range(first, idx.N):
        dd = [ref.sdc(T, idx.codes[n], c) for c in idx.centers]
        assert idx.assign[n] == int(np.argmin(dd))
        k = idx.assign[n]
        assert n in idx.ids[idx.offsets[k]:idx.offsets[k + 1]]
    q = y[:1]
    ids, dist, _ = idx.query(q, 1, S=np.array([first], np.int64), path=ref.PATH_LINEAR)
    assert ids[0, 0] == first                                # S:241 singleton subset


def test_memory_formula_matches_paper(ref):
    """(N+K) M log2 Z + 32 N bits; the paper prints 68 MB and 244 MB."""
    for N, K, M, printed in _rows("memory_footprint.txt"):
        N, K, M = int(N), int(K), int(M)
        bits = (N + K) * M * math.log2(256) + 32 * N
        assert round(bits / 8 / 1e6) == int(printed)
    idx, _ = _small_index(ref, K=20)
    assert idx.memory_bytes() == (idx.N + idx.K) * idx.M + 4 * idx.N


# ---------------------------------------------------------------- PQk-means --
def test_pqkmeans_recovers_distinct_values(ref):
    """codes with exactly K' distinct values -> centres = those values, objective 0."""
    M, Z, ds, K = 4, 256, 2, 6
    cb = _rand_cb(M, Z, ds, 21)
    T = ref.sdc_tables(cb, M * ds, M, Z)
    g = np.random.default_rng(22)
    vals = g.integers(0, Z, size=(K, M)).astype(np.uint8)
    X = vals[g.integers(0, K, size=300)]
    C, obj = ref.pqkmeans(T, X, K, n_iter=5)
    assert {tuple(c) for c in C} == {tuple(v) for v in vals}
    assert obj[-1] == 0.0


def test_pqkmeans_single_center_enumeration(ref):
    """K' = 1 -> per subspace the symbol minimising the summed squared distance
    to the members' code words, by enumeration over all Z (fp64 reconstruction)."""
    M, Z, ds = 3, 256, 3
    cb = _rand_cb(M, Z, ds, 23)
    T = ref.sdc_tables(cb, M * ds, M, Z)
    X = np.random.default_rng(24).integers(0, Z, size=(200, M)).astype(np.uint8)
    C, _ = ref.pqkmeans(T, X, 1, n_iter=1)
    for m in range(M):
        w = cb[m].astype(np.float64)
        cost = ((w[:, None, :] - w[X[:, m]][None, :, :]) ** 2).sum(-1).sum(1)
        assert cost[C[0, m]] <= cost.min() * (1 + 1e-9)


def test_pqkmeans_monotone_and_deterministic(ref):
    """S:257, S:268 (objective non-increasing), P:682 (deterministic for K')
    (better than K' random codes as centres)."""
    idx, _ = _small_index(ref)
    T = ref.sdc_tables(idx.cb, idx.D, idx.M)
    X = idx.codes[:1500]
    C1, obj = ref.pqkmeans(T, X, 30, n_iter=8)
    C2, obj2 = ref.pqkmeans(T, X, 30, n_iter=8)
    assert np.array_equal(C1, C2) and np.array_equal(obj, obj2)
    assert (np.diff(obj) <= 1e-6 * obj[:-1]).all()
    rnd = X[np.random.default_rng(25).choice(len(X), 30, replace=False)]
    a, _ = ref.assign(T, X, rnd)
    base = sum(ref.sdc(T, X[i], rnd[a[i]]) for i in range(len(X)))
    assert obj[-1] <= base


def test_sample_is_smallest_keys(ref):
    """Reading R10 ("a subset ... min(N, 100K')"): the sample is exactly the
    n_s ids with the smallest splitmix64(seed ^ id), in key order."""
    N, ns, seed = 5000, 700, 1234
    s = ref.sample_ids(N, ns, seed)
    keys = np.array([ref.splitmix64(seed ^ i) for i in range(N)], dtype=np.uint64)
    assert len(set(s.tolist())) == ns
    assert all(int(keys[s[i]]) < int(keys[s[i + 1]]) for i in range(ns - 1))
    rest = np.setdiff1d(np.arange(N), s)
    assert min(int(k) for k in keys[rest]) > int(keys[s[-1]])


def test_reconfigure_deterministic_and_partition(ref):
    """Alg. 4: deterministic for K' and seed; W partitions the ids."""
    idx, _ = _small_index(ref, K=15)
    c1 = ref.reconfigure(idx.cb, idx.codes, 15, 5, 99)
    c2 = ref.reconfigure(idx.cb, idx.codes, 15, 5, 99)
    for a, b in zip(c1, c2):
        assert np.array_equal(a, b)
    centers, a, off, ids, _ = c1
    assert off[-1] == idx.N and np.array_equal(np.sort(ids), np.arange(idx.N))


# -------------------------------------------------------------------- train --
def test_train_two_point_masses(ref):
    """{(0,0),(0,0),(1,1),(1,1)}, M=1, Z=2 -> code words {(0,0),(1,1)}."""
    x = np.array([[0, 0], [0, 0], [1, 1], [1, 1]], np.float32)
    cb = ref.train(x, M=1, n_iter=5, seed=0, Z=2)
    assert {tuple(r) for r in cb[0]} == {(0.0, 0.0), (1.0, 1.0)}


def test_train_zero_distortion_fixed_point(ref):
    """the training set = Z distinct vectors -> the code book is that set; and the
    lossless case (integer data, ds=1) trains to exactly {0..255} per dimension."""
    x = np.random.default_rng(26).standard_normal((16, 3)).astype(np.float32)
    cb = ref.train(x, M=1, n_iter=3, seed=5, Z=16)
    assert {tuple(r) for r in cb[0]} == {tuple(r) for r in x}
    x, _ = _lossless_setup(n=1000, D=4)
    cb = ref.train(x, M=4, n_iter=2, seed=1)
    for m in range(4):
        assert np.array_equal(np.sort(cb[m, :, 0]), np.arange(256, dtype=np.float32))


def test_train_beats_random_codewords_and_is_deterministic(ref):
    """per-subspace distortion <= that of Z randomly chosen training rows;
    deterministic for a fixed seed."""
    M, Z = 4, 8
    x = np.random.default_rng(27).standard_normal((1000, 16)).astype(np.float32)
    cb = ref.train(x, M, n_iter=10, seed=3, Z=Z)
    assert np.array_equal(cb, ref.train(x, M, n_iter=10, seed=3, Z=Z))
    rnd = x[np.random.default_rng(28).choice(1000, Z, replace=False)]
    for m in range(M):
        sub = x[:, m * 4:(m + 1) * 4].astype(np.float64)
        dist = lambda W: ((sub[:, None, :] - W[None].astype(np.float64)) ** 2).sum(-1).min(1).sum()
        assert dist(cb[m]) <= dist(rnd[:, m * 4:(m + 1) * 4])


def test_train_rejects_too_few_rows(ref):
    with pytest.raises(ref.OracleError) as e:
        ref.train(np.zeros((10, 4), np.float32), M=2, n_iter=1, seed=0)
    assert e.value.status == 6


# ------------------------------------------------------ paper-exact Alg. 2 ---
def test_ivf_paper_budget_and_early_stop(ref):
    """Alg. 2 as printed: L = candidates, ceil(KL/|S|) lists,
    early stop at |U| = L.  Pinned by: (a) an unlimited budget over every list equals
    the linear scan; (b) K = 1: the first L members of S in id order (R11),
    ranked — i.e. the linear scan over exactly those ids; (c) the returned ids are
    always within the traversal prefix."""
    idx, _ = _small_index(ref, K=1)
    q = gen.gaussian(8, idx.D, seed=41, stream=gen.STREAM_QUERY)
    for S in (None, gen.subset(idx.N, 900, seed=42)):
        members = np.arange(idx.N) if S is None else S
        for L in (1, 37, 500):
            pid, pd = ref.ivf_paper(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, 20, L, S=S)
            lid, ld = ref.linear(idx.cb, idx.codes, q, 20, S=members[:L])
            assert np.array_equal(pid, lid) and np.array_equal(pd, ld)
    idx, _ = _small_index(ref, K=25)
    q = gen.gaussian(8, idx.D, seed=43, stream=gen.STREAM_QUERY)
    pid, pd = ref.ivf_paper(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, 30, L=idx.N)
    lid, ld = ref.linear(idx.cb, idx.codes, q, 30)
    assert np.array_equal(pid, lid) and np.array_equal(pd, ld)
    # traversal prefix: ranks by fp64 reconstruction distance of the centres (skip near-ties)
    rec = ref.decode(idx.cb, idx.centers, idx.D).astype(np.float64)
    L = 150
    P = -(-idx.K * L // idx.N)
    pid, _ = ref.ivf_paper(idx.cb, idx.codes, idx.centers, idx.offsets, idx.ids, q, 30, L)
    for i in range(len(q)):
        d0 = ((rec - q[i].astype(np.float64)) ** 2).sum(1)
        order = np.argsort(d0, kind="stable")
        if np.min(np.diff(np.sort(d0))[: P + 1]) < 1e-6 * d0.max():
            continue
        prefix = np.concatenate([idx.ids[idx.offsets[k]:idx.offsets[k + 1]] for k in order[:P]])[:L]
        assert np.isin(pid[i][pid[i] >= 0], prefix).all()


# --------------------------------------------------------------- OPQ rotation --
def test_rotate_closed_forms(ref):
    """rref_rotate (canonical order CR): identity, permutations and sign
    flips are exact; a 3-4-5 rotation matches its fp64 value to fp32 rounding; an
    orthogonal R preserves norms and R^T undoes R (within fp32 accumulation error)."""
    rng = np.random.default_rng(11)
    D = 24
    x = rng.normal(size=(50, D)).astype(np.float32)
    assert np.array_equal(ref.rotate(np.eye(D, dtype=np.float32), x), x)
    perm = rng.permutation(D)
    P = np.zeros((D, D), np.float32)
    P[np.arange(D), perm] = 1.0                      # (P x)_i = x_perm[i]
    assert np.array_equal(ref.rotate(P, x), x[:, perm])
    S = np.diag(np.where(rng.random(D) < 0.5, -1.0, 1.0)).astype(np.float32)
    assert np.array_equal(ref.rotate(S, x), x * np.diag(S)[None, :])
    G = np.array([[0.6, -0.8], [0.8, 0.6]], np.float32)  # cos/sin of the 3-4-5 triangle
    y = ref.rotate(G, np.array([[5.0, 10.0]], np.float32))[0]
    exact = np.array([-5.0, 10.0])
    assert np.all(np.abs(y - exact) <= 4e-6 * np.abs(exact)), y
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    Q = Q.astype(np.float32)
    yq = ref.rotate(Q, x).astype(np.float64)
    assert np.allclose(np.linalg.norm(yq, axis=1), np.linalg.norm(x.astype(np.float64), axis=1), rtol=2e-5)
    back = ref.rotate(np.ascontiguousarray(Q.T), ref.rotate(Q, x))
    assert np.allclose(back, x, atol=2e-5 * np.abs(x).max())


def test_rotated_index_is_pq_on_rotated_data(ref):
    """Rii-OPQ "remaining process is exactly the same as PQ": an oracle
    index with rotation R returns what a plain index over R x returns for R q."""
    rng = np.random.default_rng(12)
    D, M = 16, 4
    x = rng.normal(size=(3000, D)).astype(np.float32)
    q = rng.normal(size=(5, D)).astype(np.float32)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    Q = Q.astype(np.float32)
    a = ref.OracleIndex(D, M)
    a.R = Q
    a.train(x, n_iter=3)
    a.add(x)
    b = ref.OracleIndex(D, M)
    xr = ref.rotate(Q, x)
    b.train(xr, n_iter=3)
    b.add(xr)
    assert np.array_equal(a.codes, b.codes) and np.array_equal(a.cb, b.cb)
    ra, rb = a.query(q, 7, path=ref.PATH_LINEAR), b.query(ref.rotate(Q, q), 7, path=ref.PATH_LINEAR)
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])


# ------------------------------------------------ empty-cluster re-seeding ---
def test_train_reseed_worked_example(ref):
    """R8 / SPEC S:138 ("empty clusters re-seeded from the farthest point"): a hand-
    traced 1-D Lloyd run (tests/golden/train_reseed_worked_example.txt) in which a
    code word loses all its rows in iteration 2 and is re-seeded with the unused
    row of largest assignment distance.  The instrumented oracle shows the branch
    ran exactly once; the other plausible readings give other code books."""
    rows = {r[0]: [float(v) for v in r[1:]] for r in _rows("train_reseed_worked_example.txt")}
    x = np.array(rows["rows"], np.float32)[:, None]
    Z, seed, n_iter = int(rows["Z"][0]), int(rows["seed"][0]), int(rows["n_iter"][0])
    init = ref.train(x, 1, 0, seed, Z=Z)
    assert init[0, :, 0].tolist() == rows["init"]
    ref.reseed_reset()
    cb = ref.train(x, 1, n_iter, seed, Z=Z)
    assert ref.reseed_counts() == (1, 0)
    assert cb[0, :, 0].tolist() == np.array(rows["result"], np.float32).tolist()
    ref.reseed_reset()
    ref.train(x, 1, 1, seed, Z=Z)  # one iteration: nothing is empty yet
    assert ref.reseed_counts() == (0, 0)


def test_pqkmeans_reseed_worked_example(ref):
    """R9 / SPEC S:273 ("empty clusters re-seeded with the member of the largest
    cluster farthest from its center"): a hand-traced PQk-means run on symbols
    placed on a line (tests/golden/pqkmeans_reseed_worked_example.txt).  Cluster 1
    empties in iteration 1; the largest cluster is a tie (lowest k wins) and its
    farthest members tie (lowest sample index wins).  The instrumented oracle
    shows the branch ran once; other readings give other centres."""
    rows = {r[0]: [float(v) for v in r[1:]] for r in _rows("pqkmeans_reseed_worked_example.txt")}
    p = np.array(rows["positions"], np.float64)
    T = ((p[:, None] - p[None, :]) ** 2).astype(np.float32)[None]
    X = np.array(rows["sample"], np.uint8)[:, None]
    K, n_iter = int(rows["K"][0]), int(rows["n_iter"][0])
    ref.reseed_reset()
    C, obj = ref.pqkmeans(T, X, K, n_iter)
    assert ref.reseed_counts() == (0, 1)
    assert C[:, 0].tolist() == [int(v) for v in rows["result"]]
    ref.reseed_reset()
    ref.pqkmeans(T, X, K, 1)  # re-seeding after the first update only: nothing is empty yet
    assert ref.reseed_counts() == (0, 0)


def test_reseed_branches_run_at_config_scale(ref):
    """The re-seeding branches are not only reachable on hand-made inputs: the tiny
    config's build (BASELINE configs[0]: 20 Lloyd iterations, reconfigure to 100
    lists) re-seeds one PQk-means cluster, and the small growth build of
    tests/test_gpu_parity.py (test_add_after_reconfigure_and_growth) re-seeds two
    training code words and six PQk-means clusters -- the GPU tests compare those
    builds' code books and centres bit for bit, so the GPU's re-seeding is checked
    against the pinned rule."""
    c = gen.CONFIGS["tiny"]
    x = gen.gaussian(c["N"], c["D"], seed=0)
    ref.reseed_reset()
    o = ref.OracleIndex(c["D"], c["M"])
    o.train(x, n_iter=20, seed=0)
    o.add(x)
    o.reconfigure(c["nlist"], n_iter=10, seed=0)
    assert ref.reseed_counts() == (0, 1)
    x = gen.sift_like(12_000, 128, seed=13)
    ref.reseed_reset()
    o = ref.OracleIndex(128, 16)
    o.train(x[:2_000], n_iter=3, seed=0)
    o.add(x[:2_000])
    o.reconfigure(20, n_iter=3, seed=0)
    for s in range(2_000, 12_000, 3_333):
        o.add(x[s:s + 3_333])
    o.reconfigure(110, n_iter=3, seed=4)
    assert ref.reseed_counts() == (2, 6)
