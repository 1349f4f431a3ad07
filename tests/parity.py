"""Comparator of GPU results against the oracle (BASELINE.json north_star tolerances).

* Codes / assignments / centres / posting lists: bit-exact (checked directly).
* Result lists: the GPU returns canonical (CA2) fp32 distances, so each returned
  distance must equal the oracle's fp32 ADC of the returned id exactly, and stay
  within 1e-5 relative of the oracle's distance at the same rank.  Ids must equal
  the oracle's except where the oracle's distances at the swapped ranks differ by
  less than 1e-5 relative (near-ties, including the k-th boundary).
"""
import numpy as np

REL = 1e-5


def _ref_adc(ref, cb, codes, q, ids, M):
    A = ref.lut(cb, q, M)
    return np.array([ref.adc(A, codes[i]) if i >= 0 else np.inf for i in ids], np.float32)


def assert_topk_parity(ref, cb, codes, q, gpu, oracle, S=None, max_fallback_frac=0.02, what=""):
    gid, gd = (np.asarray(a) for a in gpu[:2])
    rid, rd = (np.asarray(a) for a in oracle[:2])
    assert gid.shape == rid.shape, (gid.shape, rid.shape)
    M = codes.shape[1]
    nq = gid.shape[0]
    fallback = 0
    allowed = None if S is None else set(np.asarray(S).tolist())
    for i in range(nq):
        if np.array_equal(gid[i], rid[i]) and np.array_equal(gd[i], rd[i]):
            continue
        fallback += 1
        # padding identical
        assert np.array_equal(gid[i] < 0, rid[i] < 0), f"{what} q{i}: padding differs"
        valid = gid[i] >= 0
        g_ids, g_d = gid[i][valid], gd[i][valid]
        r_d = rd[i][valid]
        # sorted by (dist, id), unique, contained in S
        order = np.lexsort((g_ids, g_d))
        assert np.array_equal(order, np.arange(len(order))), f"{what} q{i}: not sorted"
        assert len(set(g_ids.tolist())) == len(g_ids), f"{what} q{i}: duplicate ids"
        if allowed is not None:
            assert all(int(v) in allowed for v in g_ids), f"{what} q{i}: id outside S"
        # returned distances are the canonical ADC of the returned ids
        exact = _ref_adc(ref, cb, codes, q[i], g_ids, M)
        assert np.array_equal(exact, g_d), f"{what} q{i}: distance is not the CA2 ADC of its id"
        # rank-wise within tolerance of the oracle
        tol = REL * np.maximum(r_d, 1e-30)
        assert (np.abs(g_d.astype(np.float64) - r_d) <= tol).all(), f"{what} q{i}: distance off by > 1e-5 rel"
    assert fallback <= max(1, int(max_fallback_frac * nq)), f"{what}: {fallback}/{nq} queries needed the near-tie rule"
    return fallback
