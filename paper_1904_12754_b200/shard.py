"""Multi-GPU partitioning (one process per GPU).

Two exact schemes:

* **Row sharding** (`row_shard`): components are independent MLMC problems; rank r of N solves
  every N-th component of a fixed permutation.  No data-path collective.  Used by bench.py.
* **Sample sharding** (`owned_chunks`, `combine_ordered`; device side in context.cu): every rank
  runs the same components, but a batch's 512-sample chunk g is sampled only on rank
  g % N; the per-chunk partials are summed across ranks (NCCL all-reduce on the GPU) and
  combined per request in ascending chunk order (SumAcc::combine, parallel.hpp:52).  Each chunk
  is non-zero on exactly one rank, so the sum is exact and every rank gets the single-GPU
  totals bit for bit -- and with them the same driver decisions.
"""
from __future__ import annotations

import numpy as np

PERM_SEED = 20190429


def row_shard(n: int, rank: int, world: int, seed: int = PERM_SEED) -> np.ndarray:
    """Sorted components of `rank`: round-robin over a fixed permutation of range(n)."""
    if not (0 <= rank < world):
        raise ValueError("bad rank / world")
    perm = np.random.default_rng(seed).permutation(n).astype(np.int64)
    return np.sort(perm[rank::world])


def owned_chunks(g_begin: int, g_end: int, rank: int, world: int) -> np.ndarray:
    """Global chunk ids of the window [g_begin, g_end) that `rank` samples (g % world == rank)."""
    own0 = g_begin + (rank - g_begin % world) % world
    return np.arange(own0, g_end, world, dtype=np.int64)


def combine_ordered(sums, sums_sq, costs):
    """SumAcc::combine over chunk partials in ascending order, from zero (parallel.hpp:52)."""
    s = s2 = 0.0
    c = 0
    for a, b, k in zip(sums, sums_sq, costs):
        s += float(a)
        s2 += float(b)
        c += int(k)
    return s, s2, c
