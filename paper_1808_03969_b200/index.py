"""Python binding of the C ABI (include/rii.h): argument marshalling only.

Every step of the method runs in the CUDA kernels of librii_b200.so; this module
only converts numpy arrays / torch tensors into pointers.  Torch CUDA tensors
are passed as device memory (RII_MEM_DEVICE) on torch's current stream; numpy
arrays and CPU tensors as host memory (RII_MEM_HOST).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib as _rl

_PATHS = {"auto": _rl.PATH_AUTO, "linear": _rl.PATH_LINEAR, "ivf": _rl.PATH_IVF,
          _rl.PATH_AUTO: _rl.PATH_AUTO, _rl.PATH_LINEAR: _rl.PATH_LINEAR, _rl.PATH_IVF: _rl.PATH_IVF}


def _torch():
    import torch
    return torch


def _is_cuda_tensor(a) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor) and a.is_cuda


def _stream_ptr(stream):
    if stream is not None:
        return C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _host(a, dtype):
    """Contiguous host array of `dtype` (numpy or CPU tensor in)."""
    try:
        torch = _torch()
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(a, dtype=dtype)


def _dev(a, dtype):
    torch = _torch()
    tdt = {np.float32: torch.float32, np.int64: torch.int64, np.uint64: torch.uint64}[dtype]
    if a.dtype != tdt or not a.is_contiguous():
        a = a.to(tdt).contiguous()
    return a


def _ptr(a):
    if _is_cuda_tensor(a) or (hasattr(a, "data_ptr") and not isinstance(a, np.ndarray)):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * _rl.NCCL_ID_BYTES)()
    _rl.check(_rl.load().rii_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of an n-row add batch stored by `rank` of `world` (host-only)."""
    lo, hi = C.c_int64(), C.c_int64()
    _rl.check(_rl.load().rii_shard_range(n, rank, world, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


DEBUG_COUNTERS = ("windows", "compactions", "rollbacks", "gthr_tightenings", "rescales", "publishes", "pushed",
                  "cycles_fill", "cycles_scan", "cycles_tail", "ctas")


def debug_counters(enable: bool) -> None:
    """Start (clear) or stop the scan kernels' diagnostic event counters."""
    _rl.check(_rl.load().rii_debug_counters(1 if enable else 0))


def read_debug_counters() -> dict:
    out = (C.c_int64 * len(DEBUG_COUNTERS))()
    _rl.check(_rl.load().rii_debug_counters_read(out, len(DEBUG_COUNTERS)))
    return dict(zip(DEBUG_COUNTERS, (int(v) for v in out)))


def launch_count() -> int:
    return int(_rl.load().rii_launch_count())


def partial_width(topk: int) -> int:
    return int(_rl.load().rii_partial_width(topk))


def torch_allgather(group=None):
    """A host all-gather over torch.distributed (e.g. the gloo backend) for
    Index(..., transport=...): maps this rank's bytes to every rank's bytes."""
    def allgather(send: np.ndarray) -> np.ndarray:
        torch = _torch()
        import torch.distributed as dist
        world = dist.get_world_size(group)
        t = torch.from_numpy(send)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return torch.cat(out).numpy()
    return allgather


def _transport(fn, world: int):
    """struct rii_transport whose callback marshals host bytes through fn."""
    def cb(ctx, send, recv, nbytes):
        try:
            src = np.ctypeslib.as_array((C.c_uint8 * max(int(nbytes), 1)).from_address(send))[:nbytes].copy()
            out = np.ascontiguousarray(fn(src), dtype=np.uint8)
            if out.size != world * nbytes:
                return 1
            C.memmove(recv, out.ctypes.data, out.size)
            return 0
        except Exception:  # reported to the library as a failed exchange (RII_ERR_NCCL)
            return 1
    fp = _rl.TRANSPORT_FN(cb)
    return _rl.Transport(None, fp), fp


class Index:
    """Rii index (Sec. 4.1) on one GPU, or one shard of a multi-GPU job.

    world > 1: pass the NCCL id (nccl_id, from nccl_unique_id() on rank 0) or a host
    all-gather (transport=fn, fn(bytes of this rank) -> bytes of all ranks, e.g.
    torch_allgather() over gloo); with neither the index is a detached shard."""

    def __init__(self, D: int, M: int, Ks: int = 256, device: int | None = None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, transport=None):
        self._lib = _rl.load()
        if device is None:
            try:
                device = _torch().cuda.current_device()
            except Exception:
                device = 0
        self.D, self.M, self.Ks, self.device, self.rank, self.world = D, M, Ks, device, rank, world
        h = C.c_void_p()
        if transport is not None:
            self._tr, self._tr_fn = _transport(transport, world)  # kept alive with the index
            _rl.check(self._lib.rii_create_with_transport(D, M, Ks, device, rank, world, C.byref(self._tr),
                                                          C.byref(h)))
        else:
            idbuf = None
            if nccl_id is not None:
                idbuf = (C.c_uint8 * _rl.NCCL_ID_BYTES).from_buffer_copy(nccl_id)
            _rl.check(self._lib.rii_create(D, M, Ks, device, rank, world,
                                         C.cast(idbuf, C.c_void_p) if idbuf is not None else None, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.rii_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- build ---
    def _rows(self, x):
        if _is_cuda_tensor(x):
            x = _dev(x, np.float32)
            return x, x.shape[0], _rl.MEM_DEVICE, _stream_ptr(None)
        x = _host(x, np.float32)
        return x, x.shape[0], _rl.MEM_HOST, None

    def train(self, x, n_iter: int = 20, seed: int = 0):
        x, n, where, st = self._rows(x)
        _rl.check(self._lib.rii_train(self._h, _ptr(x), n, n_iter, seed, where, st))

    # --------------------------------------------------------------- OPQ ---
    def set_rotation(self, R):
        """OPQ rotation: every later train / add / query input x becomes R x."""
        if R is None:
            _rl.check(self._lib.rii_set_rotation(self._h, None))
            return
        R = _host(R, np.float32)
        if R.shape != (self.D, self.D):
            raise ValueError(f"R must be {self.D} x {self.D}")
        _rl.check(self._lib.rii_set_rotation(self._h, _ptr(R)))

    def get_rotation(self):
        """(R, has_rotation); R is the identity when the index has no rotation."""
        R = np.empty((self.D, self.D), np.float32)
        has = C.c_int32(0)
        _rl.check(self._lib.rii_get_rotation(self._h, _ptr(R), C.byref(has)))
        return R, bool(has.value)

    def rotate(self, x):
        """R x for device rows (a torch CUDA tensor); returns a new tensor."""
        torch = _torch()
        x = _dev(x, np.float32)
        out = torch.empty_like(x)
        _rl.check(self._lib.rii_rotate(self._h, _ptr(x), x.shape[0], _ptr(out), _stream_ptr(None)))
        return out

    def train_opq(self, x, n_opq_iter: int = 8, n_iter: int = 20, seed: int = 0):
        """Non-parametric OPQ: rotation + code book (rii_train_opq)."""
        x, n, where, st = self._rows(x)
        _rl.check(self._lib.rii_train_opq(self._h, _ptr(x), n, n_opq_iter, n_iter, seed, where, st))

    def add(self, x) -> int:
        x, n, where, st = self._rows(x)
        first = C.c_int64(0)
        _rl.check(self._lib.rii_add(self._h, _ptr(x), n, where, st, C.byref(first)))
        return first.value

    def reconfigure(self, nlist: int, n_iter: int = 10, seed: int = 0, stream=None):
        st = _stream_ptr(stream) if stream is not None else None
        _rl.check(self._lib.rii_reconfigure(self._h, nlist, n_iter, seed, st))

    # ------------------------------------------------------------- query ---
    def query(self, q, topk: int, target_ids=None, L: int = 1, path="auto", out=None, stream=None):
        """Alg. 3 Query.  Returns (ids [nq, topk] int64, dist [nq, topk] fp32, path_used)."""
        Lp = L
        used = C.c_int32(0)
        if _is_cuda_tensor(q):
            torch = _torch()
            q = _dev(q, np.float32)
            nq = q.shape[0]
            S = None if target_ids is None else _dev(torch.as_tensor(target_ids, device=q.device), np.int64)
            if out is None:
                ids = torch.empty((nq, topk), dtype=torch.int64, device=q.device)
                dist = torch.empty((nq, topk), dtype=torch.float32, device=q.device)
            else:
                ids, dist = out
            _rl.check(self._lib.rii_query(self._h, _ptr(q), nq, topk, _ptr(S) if S is not None else None,
                                        0 if S is None else S.numel(), Lp, _PATHS[path], _rl.MEM_DEVICE,
                                        _stream_ptr(stream), _ptr(ids), _ptr(dist), C.byref(used)))
            return ids, dist, used.value
        q = _host(q, np.float32)
        nq = q.shape[0]
        S = None if target_ids is None else _host(target_ids, np.int64)
        if out is None:
            ids = np.empty((nq, topk), np.int64)
            dist = np.empty((nq, topk), np.float32)
        else:
            ids, dist = out
        _rl.check(self._lib.rii_query(self._h, _ptr(q), nq, topk, _ptr(S) if S is not None else None,
                                    0 if S is None else S.shape[0], Lp, _PATHS[path], _rl.MEM_HOST,
                                    _stream_ptr(stream) if stream is not None else None, _ptr(ids), _ptr(dist),
                                    C.byref(used)))
        return ids, dist, used.value

    def query_partial(self, q, topk: int, target_ids=None, L: int = 1, path="auto", stream=None):
        """This shard's top candidates as packed uint64 keys [nq, partial_width(topk)] (device)."""
        torch = _torch()
        q = _dev(q, np.float32)
        nq = q.shape[0]
        S = None if target_ids is None else _dev(torch.as_tensor(target_ids, device=q.device), np.int64)
        keys = torch.empty((nq, partial_width(topk)), dtype=torch.uint64, device=q.device)
        used = C.c_int32(0)
        _rl.check(self._lib.rii_query_partial(self._h, _ptr(q), nq, topk, _ptr(S) if S is not None else None,
                                            0 if S is None else S.numel(), L, _PATHS[path], _stream_ptr(stream),
                                            _ptr(keys), C.byref(used)))
        return keys, used.value

    # ------------------------------------------------------------- state ---
    def get_codebook(self) -> np.ndarray:
        out = np.empty((self.M, self.Ks, self.D // self.M), np.float32)
        _rl.check(self._lib.rii_get_codebook(self._h, _ptr(out)))
        return out

    def set_codebook(self, cb):
        cb = _host(cb, np.float32)
        assert cb.size == self.M * self.Ks * (self.D // self.M)
        _rl.check(self._lib.rii_set_codebook(self._h, _ptr(cb)))

    def get_codes(self, first: int = 0, n: int | None = None) -> np.ndarray:
        if n is None:
            n = self.info()["N"] - first
        out = np.empty((n, self.M), np.uint8)
        _rl.check(self._lib.rii_get_codes(self._h, first, n, _ptr(out)))
        return out

    def get_centers(self) -> np.ndarray:
        out = np.empty((self.info()["K"], self.M), np.uint8)
        _rl.check(self._lib.rii_get_centers(self._h, _ptr(out)))
        return out

    def save(self, path: str):
        """Write the index (SPEC's RII1 layout) or this rank's shard (RIIS), include/rii.h."""
        _rl.check(self._lib.rii_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, device: int | None = None, nccl_id: bytes | None = None) -> "Index":
        """Create an index from an RII1 / RIIS file written by save()."""
        lib = _rl.load()
        if device is None:
            try:
                device = _torch().cuda.current_device()
            except Exception:
                device = 0
        h = C.c_void_p()
        idbuf = None if nccl_id is None else (C.c_uint8 * _rl.NCCL_ID_BYTES).from_buffer_copy(nccl_id)
        _rl.check(lib.rii_load(os.fsencode(path), device, C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                               C.byref(h)))
        self = cls.__new__(cls)
        self._lib, self._h, self.device = lib, h, device
        with open(path, "rb") as f:
            hdr = np.frombuffer(f.read(40), dtype="<u4")
        if bytes(hdr[:1].tobytes()) == b"RII1":  # SPEC layout: D, M, Z, N, K (single GPU)
            self.D, self.M, self.Ks = (int(v) for v in hdr[2:5])
            self.world, self.rank = 1, 0
        else:  # RIIS shard: D, M, Ks, world, rank
            self.D, self.M, self.Ks, self.world, self.rank = (int(v) for v in hdr[2:7])
        return self

    def set_centers(self, centers):
        """Install coarse centres (K x M codes): assigns every code, rebuilds W."""
        c = _host(centers, np.uint8)
        assert c.ndim == 2 and c.shape[1] == self.M
        _rl.check(self._lib.rii_set_centers(self._h, _ptr(c), c.shape[0], None))

    def get_postings(self):
        inf = self.info()
        off = np.empty(inf["K"] + 1, np.int64)
        ids = np.empty(inf["n_local"], np.int64)
        _rl.check(self._lib.rii_get_postings(self._h, _ptr(off), _ptr(ids)))
        return off, ids

    def calibrate_theta(self, q, topk: int = 100, L_grid=(1, 4, 16, 64)):
        """Fit theta(L) = a L + b from GPU timings of both paths (Alg. 3).
        Returns (a, b, crossovers per L)."""
        Lg = np.ascontiguousarray(L_grid, dtype=np.int32)
        cross = np.empty(len(Lg), np.float64)
        a, b = C.c_double(), C.c_double()
        if _is_cuda_tensor(q):
            q = _dev(q, np.float32)
            where, st = _rl.MEM_DEVICE, _stream_ptr(None)
        else:
            q = _host(q, np.float32)
            where, st = _rl.MEM_HOST, None
        _rl.check(self._lib.rii_calibrate_theta(self._h, _ptr(q), q.shape[0], topk, _ptr(Lg), len(Lg), where, st,
                                                C.byref(a), C.byref(b), _ptr(cross)))
        return a.value, b.value, cross

    def set_ivf_mode(self, mode):
        """'lists' (L = nearest lists, every member evaluated; default) or 'paper'
        (Alg. 2 as printed: L = candidate budget with the early stop)."""
        m = {"lists": _rl.IVF_LISTS, "paper": _rl.IVF_PAPER}.get(mode, mode)
        _rl.check(self._lib.rii_set_ivf_mode(self._h, int(m)))

    def set_theta(self, theta: int):
        _rl.check(self._lib.rii_set_theta(self._h, theta))

    def info(self) -> dict:
        N, K, th, nl, b = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
        _rl.check(self._lib.rii_get_info(self._h, C.byref(N), C.byref(K), C.byref(th), C.byref(nl), C.byref(b)))
        return {"N": N.value, "K": K.value, "theta": th.value, "n_local": nl.value, "bytes": b.value}


def merge_partials(keys, topk: int, stream=None):
    """Merge [parts, nq, kk] device keys from rii_query_partial into the final top-k."""
    torch = _torch()
    keys = keys.contiguous()
    parts, nq = keys.shape[0], keys.shape[1]
    ids = torch.empty((nq, topk), dtype=torch.int64, device=keys.device)
    dist = torch.empty((nq, topk), dtype=torch.float32, device=keys.device)
    _rl.check(_rl.load().rii_merge_partials(C.c_void_p(keys.data_ptr()), parts, nq, topk, _stream_ptr(stream),
                                        C.c_void_p(ids.data_ptr()), C.c_void_p(dist.data_ptr())))
    return ids, dist
