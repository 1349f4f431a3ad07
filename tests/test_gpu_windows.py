"""Multi-window parity of the headline u6 / u16 linear-scan kernels.

At full size every CTA of the headline kernel scans ~25 barrier windows
(128 steps x 384 codes = 49,152 codes each), and three mechanisms only act across
windows: the mid-chunk tightening of a query's filter by the bound another CTA
published (window-end read of gthr), the re-quantisation of the integer tables at
a tighter bound (maybe_rescale), and the publication of each CTA's kk-th distance
(atomicMin on gthr).  These cases force long chunks (RII_CHUNK_CODES) over
600k codes -- 8 to 12 windows per CTA, ragged chunk ends -- count the events
with the kernels' debug counters (rii_debug_counters) to prove each mechanism
fired, and compare every result element by element with the oracle's Alg. 1
(P:423-440).
"""
import numpy as np
import pytest

from synth import generators as gen
from tests.parity import assert_topk_parity

pytestmark = pytest.mark.gpu

_cache = {}


def _index(rii, ref, kind, N, D, M):
    key = (kind, N, D, M)
    if key not in _cache:
        x = gen.base(kind, N, D, seed=N)
        cb = ref.train(x[:20_000], M, n_iter=3, seed=0)
        g = rii.Index(D, M, device=0)
        g.set_codebook(cb)
        g.add(x)
        codes = ref.encode_mt(cb, x, M)
        assert np.array_equal(g.get_codes(), codes), "codes differ from the oracle (Eq. 1)"
        _cache[key] = (g, cb, codes)
    return _cache[key]


# (kind, N, D, M, nq, chunk, sample, expect): expect = counters that must be > 0
CASES = [
    # one long chunk (12.2 windows) + a one-code ragged tail chunk
    ("deep", 600_000, 96, 32, 48, 599_999, None, ("publishes",)),
    # ragged chunks (8.1 + 4.1 windows): the short chunk's CTAs publish while the long
    # ones are still scanning -> window-end tightening; a loose sampled bound (4,096
    # codes) -> re-quantisation at the tighter bound
    ("deep", 600_000, 96, 32, 48, 400_000, 4_096, ("gthr_tightenings", "rescales", "publishes")),
    # the u16 kernel (M = 16) under the same schedule
    ("sift", 600_000, 128, 16, 40, 400_000, 4_096, ("gthr_tightenings", "rescales", "publishes")),
    # M = 64 (the paper's SIFT1M shape, Table 2): two table halves
    ("sift", 600_000, 128, 64, 24, 400_000, 4_096, ("gthr_tightenings", "rescales", "publishes")),
]


@pytest.mark.parametrize("kind,N,D,M,nq,chunk,sample,expect", CASES)
def test_multi_window_scan_matches_oracle(monkeypatch, ref, kind, N, D, M, nq, chunk, sample, expect):
    import paper_1808_03969_b200 as rii
    rii.load()
    g, cb, codes = _index(rii, ref, kind, N, D, M)
    q = gen.base(kind, nq, D, seed=N, stream=gen.STREAM_QUERY)
    monkeypatch.setenv("RII_CHUNK_CODES", str(chunk))
    if sample:
        monkeypatch.setenv("RII_Q16_SAMPLE", str(sample))
    rii.debug_counters(True)
    try:
        gr = g.query(q, 100, path="linear")
        c = rii.read_debug_counters()
    finally:
        rii.debug_counters(False)
    print(kind, M, chunk, sample, c)
    B = 16 if M == 32 else 8
    n_cta = -(-nq // B)
    assert c["windows"] >= n_cta * (chunk // 49_152), c     # every CTA of the long chunk ran its windows
    for k in expect:
        assert c[k] > 0, (k, c)
    orr = ref.linear_mt(cb, codes, q, 100)
    assert_topk_parity(ref, cb, codes, q, gr, orr, what=f"{kind} M={M} chunk={chunk} sample={sample}")


def test_multi_window_subset_and_duplicates(monkeypatch, ref):
    """A 10 % subset scanned in long chunks (gathered codes, ids mapped through S)
    and a database of repeated codes (ties across windows and chunks resolve to the
    lowest id, CA4)."""
    import paper_1808_03969_b200 as rii
    rii.load()
    g, cb, codes = _index(rii, ref, "deep", 600_000, 96, 32)
    q = gen.deep_like(32, 96, seed=5, stream=gen.STREAM_QUERY)
    S = gen.subset(600_000, 60_000, seed=6)
    monkeypatch.setenv("RII_CHUNK_CODES", "40_000".replace("_", ""))
    monkeypatch.setenv("RII_Q16_MIN", "50000")
    gr = g.query(q, 100, target_ids=S, path="linear")
    assert_topk_parity(ref, cb, codes, q, gr, ref.linear_mt(cb, codes, q, 100, S=S), S=S, what="subset windows")
    base = gen.deep_like(5_000, 96, seed=7)
    x = np.concatenate([base] * 120)                       # 600k rows, every code 120 times
    h = rii.Index(96, 32, device=0)
    h.set_codebook(cb)
    h.add(x)
    dcodes = ref.encode_mt(cb, x, 32)
    monkeypatch.setenv("RII_CHUNK_CODES", "250000")
    gr = h.query(q, 100, path="linear")
    orr = ref.linear_mt(cb, dcodes, q, 100)
    assert np.array_equal(gr[0], orr[0]) and np.array_equal(gr[1], orr[1])
