"""Seeded synthetic workloads for BASELINE.json's five configurations.

The paper's inputs (Qwen2.5-0.5B / Mistral-7B / GPT-2 logits on arXiv
abstracts) are not available; these generators stand in
with the shapes and value distributions BASELINE.json names:

  C1  1 x 32768 fp64, N(0, 3^2), T=4, p=3, c=5, polynomial invsqrt/inv settings
  C2  256 x 32768 fp64 (+fp32), T in {3,4}, N(0, 3^2) with a planted maximiser
      whose gap over the runner-up is log-uniform in [1e-3, 1]
  C3  64 x 151936 fp64, T=4, LLM-like logits: -1.1 ln(rank) + N(0, 0.5^2),
      randomly permuted per row
  C4  128 x 32768 fp64 nucleus sampling, p in {0.9, 0.95}, Zipf(1.1)-shaped logits
  C5  B in {1,16,256,4096} x n in {1024,32768,151936}, fp64/fp32, T=4, N(0, 3^2)

c is not given by BASELINE.json; c = 5 with p = 3 is pinned.
"""
from __future__ import annotations

import numpy as np

C5_B = (1, 16, 256, 4096)
C5_N = (1024, 32768, 151936)


def gaussian(B: int, n: int, seed: int, sigma: float = 3.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, sigma, size=(B, n))


def planted(B: int, n: int, seed: int, sigma: float = 3.0):
    """N(0, sigma^2) rows with a planted unique maximiser; returns (x, istar, gap)."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, sigma, size=(B, n))
    istar = rng.integers(0, n, size=B)
    gap = 10.0 ** rng.uniform(-3.0, 0.0, size=B)
    for r in range(B):
        row = x[r]
        row[istar[r]] = -np.inf
        row[istar[r]] = row.max() + gap[r]
    return x, istar, gap


def zipf_logits(B: int, n: int, seed: int, s: float = 1.1, noise: float = 0.5) -> np.ndarray:
    rng = np.random.default_rng(seed)
    base = -s * np.log(np.arange(1, n + 1, dtype=np.float64))
    x = np.empty((B, n))
    for r in range(B):
        x[r] = rng.permutation(base + rng.normal(0.0, noise, size=n))
    return x


def peaked_logits(B: int, n: int, seed: int, min_gap: float = 0.05) -> np.ndarray:
    """SPEC.md:606's "peaked fixture vectors": the LLM-like Zipf rows above with
    the top-1 logit margin raised to at least `min_gap` (nats) where the noise
    left a near-tie; the paper's logits (QWEN, Table 1) are not available."""
    x = zipf_logits(B, n, seed)
    for r in range(B):
        i = int(np.argmax(x[r]))
        second = np.partition(x[r], -2)[-2]
        if x[r, i] - second < min_gap:
            x[r, i] = second + min_gap
    return x


def torch_gaussian(B: int, n: int, seed: int, dtype=None, device="cuda", sigma: float = 3.0):
    """Device-side N(0, sigma^2) generator for bench-scale inputs (GBs)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.empty((B, n), dtype=torch.float64, device=device)
    for r0 in range(0, B, 256):  # bounded temporaries
        r1 = min(B, r0 + 256)
        x[r0:r1].normal_(0.0, sigma, generator=g)
    return x if dtype is None or dtype == torch.float64 else x.to(dtype)


def shard_rows(B: int, rank: int, world: int):
    """Contiguous row shard [r0, r1) of rank `rank` out of `world` (rows are
    independent: no collective on the data path)."""
    q, r = divmod(B, world)
    r0 = rank * q + min(rank, r)
    r1 = r0 + q + (1 if rank < r else 0)
    return r0, r1
