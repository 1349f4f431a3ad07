"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method (no PQ, no distances, no selection):
it only draws random numbers.  Both the oracle-side tests and the CUDA path
consume what it produces, so it is the one module the two sides share.

Stand-ins (the paper's datasets are not in this container):
  * "tiny"   (BASELINE.json configs[0]) : N(0,1) vectors.
  * "sift"   (configs[1], configs[3])   : SIFT1M-like 64-component Gaussian mixture,
    means U[0,100)^D, isotropic sd 10, clipped to [0,255], rounded half-to-even.
  * "deep"   (configs[2], configs[4])   : Deep1B-like L2-normalised mixture,
    256 unit-norm means, sd 0.1, normalised after the noise.
Seed streams: 0 base data, 1 queries, 2 target subsets, 3 code-book training
sample, 5 mixture parameters.
"""
from __future__ import annotations

import math

import numpy as np

STREAM_BASE, STREAM_QUERY, STREAM_SUBSET, STREAM_TRAIN, STREAM_MIXTURE = 0, 1, 2, 3, 5


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(stream), int(seed)]))


def gaussian(n: int, D: int, seed: int = 0, stream: int = STREAM_BASE) -> np.ndarray:
    """i.i.d. N(0,1) float32 (BASELINE.json configs[0]); stream 0 with seed 0 is the
    literal `default_rng(0)` draw the config names."""
    g = np.random.default_rng(seed) if stream == STREAM_BASE else rng(seed, stream)
    return g.standard_normal((n, D), dtype=np.float32)


def _sift_means(D: int, n_comp: int, seed: int) -> np.ndarray:
    return rng(seed, STREAM_MIXTURE).uniform(0.0, 100.0, size=(n_comp, D))


def sift_like(n: int, D: int = 128, n_comp: int = 64, seed: int = 0, stream: int = STREAM_BASE,
              chunk: int = 1 << 20) -> np.ndarray:
    """SIFT1M stand-in: x = rint(clip(mu_c + 10 N(0,I), 0, 255)), c uniform over components."""
    mu = _sift_means(D, n_comp, seed)
    g = rng(seed, stream)
    out = np.empty((n, D), np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        comp = g.integers(0, n_comp, size=e - s)
        v = mu[comp] + 10.0 * g.standard_normal((e - s, D))
        out[s:e] = np.rint(np.clip(v, 0.0, 255.0))
    return out


def _deep_means(D: int, n_comp: int, seed: int) -> np.ndarray:
    m = rng(seed, STREAM_MIXTURE).standard_normal((n_comp, D))
    return m / np.linalg.norm(m, axis=1, keepdims=True)


def deep_like(n: int, D: int = 96, n_comp: int = 256, seed: int = 0, stream: int = STREAM_BASE,
              chunk: int = 1 << 20) -> np.ndarray:
    """Deep1B stand-in: x = normalise(mu_c + 0.1 N(0,I)), unit-norm means."""
    mu = _deep_means(D, n_comp, seed)
    g = rng(seed, stream)
    out = np.empty((n, D), np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        comp = g.integers(0, n_comp, size=e - s)
        v = mu[comp] + 0.1 * g.standard_normal((e - s, D))
        out[s:e] = v / np.linalg.norm(v, axis=1, keepdims=True)
    return out


def subset(N: int, size: int, seed: int = 0, stream: int = STREAM_SUBSET) -> np.ndarray:
    """|S| unique ids drawn uniformly from [0, N), sorted ascending."""
    size = min(size, N)
    return np.sort(rng(seed, stream).choice(N, size=size, replace=False)).astype(np.int64)


def lossless(n: int, D: int, seed: int = 0, stream: int = STREAM_BASE) -> np.ndarray:
    """Integer data in [0,255] whose first 256 rows enumerate every value in every
    dimension (so a trained ds=1 code book is exactly {0..255}); the rest uniform."""
    g = rng(seed, stream)
    x = g.integers(0, 256, size=(n, D)).astype(np.float32)
    base = np.stack([g.permutation(256) for _ in range(D)], axis=1).astype(np.float32)
    x[: min(n, 256)] = base[: min(n, 256)]
    return x


# --------------------------------------------------------------------------- #
# Device-side generators (torch Philox) for sizes the host should not draw:
# the same recipes, a different (but seeded and reproducible) random stream.
def _torch():
    import torch
    return torch


def sift_like_torch(n: int, device, D: int = 128, n_comp: int = 64, seed: int = 0, stream: int = STREAM_BASE,
                    out=None, chunk: int = 1 << 22):
    torch = _torch()
    mu = torch.from_numpy(_sift_means(D, n_comp, seed)).to(device=device, dtype=torch.float32)
    gen = torch.Generator(device=device)
    gen.manual_seed((int(seed) << 8) | int(stream))
    if out is None:
        out = torch.empty((n, D), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        comp = torch.randint(0, n_comp, (e - s,), generator=gen, device=device)
        v = mu[comp] + 10.0 * torch.randn((e - s, D), generator=gen, device=device)
        out[s:e] = torch.round(torch.clamp(v, 0.0, 255.0))
    return out


def deep_like_torch(n: int, device, D: int = 96, n_comp: int = 256, seed: int = 0, stream: int = STREAM_BASE,
                    out=None, chunk: int = 1 << 22, batch: int | None = None):
    """Device-side Deep1B stand-in (the recipe of deep_like).  `seed` fixes the mixture
    (its means) and the random stream; `batch` (streamed databases, configs[4]) draws
    batch b of the SAME mixture from its own stream, so that the base vectors of every
    batch, the training sample and the queries share one set of means."""
    torch = _torch()
    mu = torch.from_numpy(_deep_means(D, n_comp, seed)).to(device=device, dtype=torch.float32)
    gen = torch.Generator(device=device)
    gen.manual_seed((int(seed) << 8) | int(stream) if batch is None else
                    (((int(seed) << 8) | int(stream)) << 24) + 1 + int(batch))
    if out is None:
        out = torch.empty((n, D), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        comp = torch.randint(0, n_comp, (e - s,), generator=gen, device=device)
        v = mu[comp] + 0.1 * torch.randn((e - s, D), generator=gen, device=device)
        out[s:e] = v / torch.linalg.vector_norm(v, dim=1, keepdim=True)
    return out


def subset_torch(N: int, size: int, device, seed: int = 0, stream: int = STREAM_SUBSET):
    torch = _torch()
    gen = torch.Generator(device=device)
    gen.manual_seed((int(seed) << 8) | int(stream))
    perm = torch.randperm(N, generator=gen, device=device)[: min(size, N)]
    return torch.sort(perm).values.to(torch.int64)


# --------------------------------------------------------------------------- #
# BASELINE.json configs (recipes in DESIGN.md; readings R12-R15 for the gaps).
CONFIGS = {
    "tiny": dict(kind="gaussian", N=10_000, D=32, M=4, nlist=100, nq=100, topk=10, L=[8],
                 subsets=[1_000], n_train=None, train_iter=20),
    "sift1m": dict(kind="sift", N=1_000_000, D=128, M=16, nlist=1000, nq=10_000, topk=100, L=[1, 4, 16, 64],
                   subsets=[100, 1_000, 10_000, 100_000, 1_000_000], n_train=100_000, train_iter=20),
    "deep10m": dict(kind="deep", N=10_000_000, D=96, M=32, nlist=3162, nq=10_000, topk=100, L=[1, 4, 16, 64],
                    subsets=[100_000, 1_000_000], n_train=100_000, train_iter=20),
    "growth": dict(kind="sift", N=10_000, D=128, M=16, nlist=100, nq=10_000, topk=100, L=[1, 8],
                   add_batches=9, add_size=1_111_111, n_train=100_000, train_iter=20),
    "scale1b": dict(kind="deep", N=1_000_000_000, D=96, M=8, nlist=31_623, nq=10_000, q_batch=1_024, topk=100,
                    L=[64], subsets=[1_000_000], n_train=1_000_000, train_iter=20),
}


def nlist_for(N: int) -> int:
    """K' = sqrt(N) rounded to nearest (reading R12)."""
    return int(math.floor(math.sqrt(N) + 0.5))


def base(kind: str, n: int, D: int, seed: int = 0, stream: int = STREAM_BASE) -> np.ndarray:
    if kind == "gaussian":
        return gaussian(n, D, seed, stream)
    if kind == "sift":
        return sift_like(n, D, seed=seed, stream=stream)
    if kind == "deep":
        return deep_like(n, D, seed=seed, stream=stream)
    raise ValueError(kind)
