"""ctypes front end of the CPU oracle (oracle/rii_ref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py.  The product package
(paper_1808_03969_b200) never imports this module.

Every function marshals numpy arrays into the plain C oracle; the arithmetic
lives in rii_ref.c, which cites the paper passage each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rii_ref.c")
_LIB = os.path.join(_HERE, "librii_ref.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]

PATH_AUTO, PATH_LINEAR, PATH_IVF = 0, 1, 2
Z_DEFAULT = 256


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        p = C.c_void_p
        i64, i32, u64 = C.c_int64, C.c_int32, C.c_uint64
        sig = {
            "rref_splitmix64": (u64, [u64]),
            "rref_encode": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, p]),
            "rref_decode": (None, [p, C.c_int, C.c_int, C.c_int, p, i64, p]),
            "rref_rotate": (None, [p, C.c_int, p, i64, p]),
            "rref_lut": (None, [p, C.c_int, C.c_int, C.c_int, p, p]),
            "rref_lut64": (None, [p, C.c_int, C.c_int, C.c_int, p, p]),
            "rref_adc": (C.c_float, [p, C.c_int, C.c_int, p]),
            "rref_adc64": (C.c_double, [p, C.c_int, C.c_int, p]),
            "rref_sdc_tables": (None, [p, C.c_int, C.c_int, C.c_int, p]),
            "rref_sdc": (C.c_float, [p, C.c_int, C.c_int, p, p]),
            "rref_linear": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, p, i64, C.c_int, p, i64, p, p]),
            "rref_num_probe": (i64, [i64, i64, i64, C.c_int, i64]),
            "rref_ivf": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, p, i64, p, p, p, i64, C.c_int,
                                   p, i64, i64, p, p]),
            "rref_ivf_paper": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, p, i64, p, p, p, i64, C.c_int,
                                         p, i64, i64, p, p]),
            "rref_default_theta": (i64, [i64, i64, i64]),
            "rref_query": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, p, i64, p, p, p, i64, C.c_int,
                                     p, i64, i64, i64, C.c_int, p, p, p]),
            "rref_assign": (C.c_int, [p, C.c_int, C.c_int, p, i64, p, i64, p, p]),
            "rref_build_postings": (C.c_int, [p, i64, i64, p, p]),
            "rref_sample_ids": (C.c_int, [i64, i64, u64, p]),
            "rref_pqkmeans": (C.c_int, [p, C.c_int, C.c_int, p, i64, i64, C.c_int, p, p]),
            "rref_reconfigure": (C.c_int, [p, C.c_int, C.c_int, C.c_int, p, i64, i64, C.c_int, u64,
                                           p, p, p, p, p]),
            "rref_train": (C.c_int, [p, i64, C.c_int, C.c_int, C.c_int, C.c_int, u64, p]),
            "rref_reseed_count": (i64, [C.c_int]),
            "rref_reseed_reset": (None, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _chk(st, what):
    if st != 0:
        raise OracleError(st, what)


def reseed_counts() -> tuple[int, int]:
    """(training, PQk-means) empty-cluster re-seeds since the last reset (instrumentation)."""
    return int(lib().rref_reseed_count(0)), int(lib().rref_reseed_count(1))


def reseed_reset() -> None:
    lib().rref_reseed_reset()


def splitmix64(x: int) -> int:
    return int(lib().rref_splitmix64(x))


def encode(cb, x, M, Z=Z_DEFAULT):
    x = _c(x, np.float32)
    cb = _c(cb, np.float32)
    n, D = x.shape
    out = np.empty((n, M), np.uint8)
    _chk(lib().rref_encode(_p(cb), D, M, Z, _p(x), n, _p(out)), "encode")
    return out


def decode(cb, codes, D, Z=Z_DEFAULT):
    codes = _c(codes, np.uint8)
    cb = _c(cb, np.float32)
    n, M = codes.shape
    out = np.empty((n, D), np.float32)
    lib().rref_decode(_p(cb), D, M, Z, _p(codes), n, _p(out))
    return out


def rotate(R, x):
    """OPQ input rotation y = R x, canonical fp32 order CR."""
    R = _c(R, np.float32)
    x = _c(np.atleast_2d(x), np.float32)
    D = R.shape[0]
    assert R.shape == (D, D) and x.shape[1] == D
    y = np.empty_like(x)
    lib().rref_rotate(_p(R), D, _p(x), x.shape[0], _p(y))
    return y


def lut(cb, q, M, Z=Z_DEFAULT):
    q = _c(q, np.float32)
    cb = _c(cb, np.float32)
    D = q.shape[-1]
    A = np.empty((M, Z), np.float32)
    lib().rref_lut(_p(cb), D, M, Z, _p(q), _p(A))
    return A


def lut64(cb, q, M, Z=Z_DEFAULT):
    q = _c(q, np.float32)
    cb = _c(cb, np.float32)
    D = q.shape[-1]
    A = np.empty((M, Z), np.float64)
    lib().rref_lut64(_p(cb), D, M, Z, _p(q), _p(A))
    return A


def adc(A, code):
    A = _c(A, np.float32)
    code = _c(code, np.uint8)
    M, Z = A.shape
    return float(lib().rref_adc(_p(A), M, Z, _p(code)))


def adc64(A, code):
    A = _c(A, np.float64)
    code = _c(code, np.uint8)
    M, Z = A.shape
    return float(lib().rref_adc64(_p(A), M, Z, _p(code)))


def sdc_tables(cb, D, M, Z=Z_DEFAULT):
    cb = _c(cb, np.float32)
    T = np.empty((M, Z, Z), np.float32)
    lib().rref_sdc_tables(_p(cb), D, M, Z, _p(T))
    return T


def sdc(T, a, b):
    T = _c(T, np.float32)
    M, Z, _ = T.shape
    return float(lib().rref_sdc(_p(T), M, Z, _p(_c(a, np.uint8)), _p(_c(b, np.uint8))))


def _targets(S):
    if S is None:
        return None, 0
    S = _c(S, np.int64)
    return S, S.shape[0]


def linear(cb, codes, q, topk, S=None, Z=Z_DEFAULT):
    cb, codes, q = _c(cb, np.float32), _c(codes, np.uint8), _c(q, np.float32)
    N, M = codes.shape
    nq, D = q.shape
    S, nS = _targets(S)
    ids = np.empty((nq, topk), np.int64)
    dist = np.empty((nq, topk), np.float32)
    _chk(lib().rref_linear(_p(cb), D, M, Z, _p(codes), N, _p(q), nq, topk, _p(S), nS, _p(ids), _p(dist)),
         "linear")
    return ids, dist


def num_probe(N, K, nS, has_S, L):
    return int(lib().rref_num_probe(N, K, nS, 1 if has_S else 0, L))


def ivf(cb, codes, centers, offsets, ids_csr, q, topk, L, S=None, Z=Z_DEFAULT):
    cb, codes, q = _c(cb, np.float32), _c(codes, np.uint8), _c(q, np.float32)
    centers, offsets, ids_csr = _c(centers, np.uint8), _c(offsets, np.int64), _c(ids_csr, np.int64)
    N, M = codes.shape
    K = centers.shape[0]
    nq, D = q.shape
    S, nS = _targets(S)
    ids = np.empty((nq, topk), np.int64)
    dist = np.empty((nq, topk), np.float32)
    _chk(lib().rref_ivf(_p(cb), D, M, Z, _p(codes), N, _p(centers), K, _p(offsets), _p(ids_csr), _p(q), nq,
                        topk, _p(S), nS, L, _p(ids), _p(dist)), "ivf")
    return ids, dist


def ivf_paper(cb, codes, centers, offsets, ids_csr, q, topk, L, S=None, Z=Z_DEFAULT):
    """Alg. 2 as printed: L = candidate budget with the early stop (R2 mode B)."""
    cb, codes, q = _c(cb, np.float32), _c(codes, np.uint8), _c(q, np.float32)
    centers, offsets, ids_csr = _c(centers, np.uint8), _c(offsets, np.int64), _c(ids_csr, np.int64)
    N, M = codes.shape
    K = centers.shape[0]
    nq, D = q.shape
    S, nS = _targets(S)
    ids = np.empty((nq, topk), np.int64)
    dist = np.empty((nq, topk), np.float32)
    _chk(lib().rref_ivf_paper(_p(cb), D, M, Z, _p(codes), N, _p(centers), K, _p(offsets), _p(ids_csr), _p(q), nq,
                              topk, _p(S), nS, L, _p(ids), _p(dist)), "ivf_paper")
    return ids, dist


def default_theta(N, K, L):
    return int(lib().rref_default_theta(N, K, L))


def query(cb, codes, centers, offsets, ids_csr, q, topk, L, S=None, theta=-1, path=PATH_AUTO, Z=Z_DEFAULT):
    cb, codes, q = _c(cb, np.float32), _c(codes, np.uint8), _c(q, np.float32)
    N, M = codes.shape
    nq, D = q.shape
    if centers is None or len(centers) == 0:
        K = 0
        centers = np.zeros((1, M), np.uint8)
        offsets = np.zeros(1, np.int64)
        ids_csr = np.zeros(1, np.int64)
    else:
        K = centers.shape[0]
    centers, offsets, ids_csr = _c(centers, np.uint8), _c(offsets, np.int64), _c(ids_csr, np.int64)
    S, nS = _targets(S)
    ids = np.empty((nq, topk), np.int64)
    dist = np.empty((nq, topk), np.float32)
    used = C.c_int(0)
    _chk(lib().rref_query(_p(cb), D, M, Z, _p(codes), N, _p(centers), K, _p(offsets), _p(ids_csr), _p(q), nq,
                          topk, _p(S), nS, L, theta, path, _p(ids), _p(dist), C.byref(used)), "query")
    return ids, dist, used.value


def assign(T, codes, centers):
    T, codes, centers = _c(T, np.float32), _c(codes, np.uint8), _c(centers, np.uint8)
    M, Z, _ = T.shape
    n = codes.shape[0]
    K = centers.shape[0]
    a = np.empty(n, np.int32)
    d = np.empty(n, np.float32)
    _chk(lib().rref_assign(_p(T), M, Z, _p(codes), n, _p(centers), K, _p(a), _p(d)), "assign")
    return a, d


def build_postings(a, K):
    a = _c(a, np.int32)
    N = a.shape[0]
    off = np.empty(K + 1, np.int64)
    ids = np.empty(N, np.int64)
    _chk(lib().rref_build_postings(_p(a), N, K, _p(off), _p(ids)), "build_postings")
    return off, ids


def sample_ids(N, ns, seed):
    out = np.empty(ns, np.int64)
    _chk(lib().rref_sample_ids(N, ns, seed, _p(out)), "sample_ids")
    return out


def pqkmeans(T, X, K, n_iter):
    T, X = _c(T, np.float32), _c(X, np.uint8)
    M, Z, _ = T.shape
    ns = X.shape[0]
    Cc = np.empty((K, M), np.uint8)
    obj = np.empty(n_iter + 1, np.float64)
    _chk(lib().rref_pqkmeans(_p(T), M, Z, _p(X), ns, K, n_iter, _p(Cc), _p(obj)), "pqkmeans")
    return Cc, obj


def reconfigure(cb, codes, K, n_iter, seed, Z=Z_DEFAULT):
    cb, codes = _c(cb, np.float32), _c(codes, np.uint8)
    N, M = codes.shape
    D = cb.size // Z
    centers = np.empty((K, M), np.uint8)
    a = np.empty(N, np.int32)
    off = np.empty(K + 1, np.int64)
    ids = np.empty(N, np.int64)
    obj = np.empty(n_iter + 1, np.float64)
    _chk(lib().rref_reconfigure(_p(cb), D, M, Z, _p(codes), N, K, n_iter, seed, _p(centers), _p(a), _p(off),
                                _p(ids), _p(obj)), "reconfigure")
    return centers, a, off, ids, obj


def train(x, M, n_iter, seed, Z=Z_DEFAULT):
    x = _c(x, np.float32)
    n, D = x.shape
    cb = np.empty((M, Z, D // M), np.float32)
    _chk(lib().rref_train(_p(x), n, D, M, Z, n_iter, seed, _p(cb)), "train")
    return cb


class OracleIndex:
    """The paper's data structure (Sec. 4.1) held as numpy arrays:
    codebook, linear codes Xbar, centres Cbar, posting lists W (CSR), theta."""

    def __init__(self, D, M, Z=Z_DEFAULT):
        self.D, self.M, self.Z = D, M, Z
        self.cb = None
        self.codes = np.zeros((0, M), np.uint8)
        self.centers = np.zeros((0, M), np.uint8)
        self.assign = np.zeros(0, np.int32)
        self.offsets = np.zeros(1, np.int64)
        self.ids = np.zeros(0, np.int64)
        self.theta = -1
        self.R = None  # OPQ rotation; inputs become R x

    def _in(self, x):
        return x if self.R is None else rotate(self.R, x)

    @property
    def N(self):
        return self.codes.shape[0]

    @property
    def K(self):
        return self.centers.shape[0]

    def train(self, x, n_iter=20, seed=0):
        self.cb = train(self._in(x), self.M, n_iter, seed, self.Z)

    def add(self, x):
        """Data addition: PushBack codes; PushBack(W_a(n), n)."""
        first = self.N
        new = encode(self.cb, self._in(x), self.M, self.Z)
        self.codes = np.concatenate([self.codes, new])
        if self.K > 0:
            T = sdc_tables(self.cb, self.D, self.M, self.Z)
            a, _ = assign(T, new, self.centers)
            self.assign = np.concatenate([self.assign, a])
            self.offsets, self.ids = build_postings(self.assign, self.K)
        return first

    def reconfigure(self, K, n_iter=10, seed=0):
        self.centers, self.assign, self.offsets, self.ids, obj = reconfigure(
            self.cb, self.codes, K, n_iter, seed, self.Z)
        return obj

    def query(self, q, topk, S=None, L=1, path=PATH_AUTO):
        return query(self.cb, self.codes, self.centers if self.K else None, self.offsets, self.ids, self._in(q), topk, L,
                     S, self.theta, path, self.Z)

    def memory_bytes(self):
        """Theoretical footprint (N+K) M log2 Z + 32 N bits in bytes, Z = 256."""
        return self.codes.nbytes + self.centers.nbytes + 4 * self.N


# ------------------------------------------------------------- all cores ---
def cores() -> int:
    """Host threads available to this process."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def parallel_rows(fn, rows, *args, threads=None, **kw):
    """Run the single-threaded oracle function fn(..., rows_slice, ...) on contiguous
    slices of `rows` (queries, or vectors to encode) in a thread pool and
    concatenate the results along axis 0.  The C oracle releases the GIL (ctypes),
    so the slices run on separate cores; every slice computes exactly what the
    single call would (the oracle has no cross-row state).  `rows` is passed as the
    argument named by fn's signature position: fn(rows_slice, *args, **kw)."""
    import concurrent.futures as cf
    threads = threads or cores()
    n = len(rows)
    if n == 0 or threads <= 1:
        return fn(rows, *args, **kw)
    bounds = np.linspace(0, n, min(threads * 4, n) + 1).astype(int)
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(lambda ab: fn(rows[ab[0]:ab[1]], *args, **kw), zip(bounds[:-1], bounds[1:])))
    if isinstance(parts[0], tuple):
        return tuple(np.concatenate([p[i] for p in parts]) for i in range(len(parts[0])))
    return np.concatenate(parts)


def encode_mt(cb, x, M, threads=None):
    return parallel_rows(lambda xs: encode(cb, xs, M), x, threads=threads)


def linear_mt(cb, codes, q, topk, S=None, threads=None):
    return parallel_rows(lambda qs: linear(cb, codes, qs, topk, S=S), q, threads=threads)


def ivf_mt(cb, codes, centers, offsets, ids_csr, q, topk, L, S=None, threads=None):
    return parallel_rows(lambda qs: ivf(cb, codes, centers, offsets, ids_csr, qs, topk, L, S=S), q, threads=threads)


def assign_mt(T, codes, centers, threads=None):
    return parallel_rows(lambda cs: assign(T, cs, centers), codes, threads=threads)
