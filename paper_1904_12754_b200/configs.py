"""Synthetic inputs of the BASELINE configs (host-side input generation, not the hot path).

C1 / C2 (BASELINE.json configs[0], configs[1]): 2-D 5-point Laplacian on a g x g
grid of interior nodes (row = y*g + x, diag -4, off-diagonal +1, Dirichlet boundary
eliminated), v_i uniform in [0,1) drawn from the reference's own Philox stream
stream_for(seed, 0, i, lane 6) (rng.hpp:76-79; lanes 0-3 and 7 are taken by the reference),
t = 1 (C1) / 0.5 (C2), eps = 1e-3.  Per-row driver seed = 1000 + row.
There is no public dataset behind these configs: everything is generated from seeds.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import SparseMatrix

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox_first_uniform(seed: int, level: int, samples: np.ndarray, lane: int) -> np.ndarray:
    """First next_uniform() of stream_for(seed, level, s, lane) for every s (rng.hpp:21-66),
    vectorised: block 0, words (c2, c3) of the Philox4x32-10 output."""
    s = np.asarray(samples, np.uint64)
    c0 = np.zeros_like(s, dtype=np.uint64)
    c1 = s & _MASK
    c2 = s >> np.uint64(32)
    c3 = np.full_like(s, (level & 0xFFFFFF) | (lane << 24), dtype=np.uint64)
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        c0, c1, c2, c3 = n0, p1 & _MASK, n2, p0 & _MASK
        k0 = (k0 + np.uint64(_W0)) & _MASK
        k1 = (k1 + np.uint64(_W1)) & _MASK
    bits = (c2 << np.uint64(32)) | c3
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def grid_laplacian(g: int) -> SparseMatrix:
    """5-point Laplacian on g x g interior nodes; columns ascending within each row."""
    n = g * g
    r = np.arange(n, dtype=np.int64)
    x, y = r % g, r // g
    cols = np.stack([r - g, r - 1, r, r + 1, r + g], axis=1)
    vals = np.tile(np.array([1.0, 1.0, -4.0, 1.0, 1.0]), (n, 1))
    ok = np.stack([y > 0, x > 0, np.ones(n, bool), x + 1 < g, y + 1 < g], axis=1)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(ok.sum(axis=1))
    return SparseMatrix(n, rp, cols[ok].astype(np.int64), vals[ok].astype(np.float64))


def grid_vector(seed: int, n: int) -> np.ndarray:
    return philox_first_uniform(seed, 0, np.arange(n, dtype=np.uint64), 6)


def row_seeds(rows) -> np.ndarray:
    return (np.asarray(rows, np.uint64) + np.uint64(1000)).astype(np.uint64)


@dataclass
class Config:
    name: str
    a: SparseMatrix
    u: np.ndarray
    beta: float
    epsilon: float
    description: str


VECTOR_SEED = 12345  # v = stream_for(12345, 0, i, 6), as in the survey probes


def make_config(name: str) -> Config:
    if name in ("c1", "C1"):
        a = grid_laplacian(64)
        return Config("c1", a, grid_vector(VECTOR_SEED, a.n), 1.0, 1e-3,
                      "2D 5-point Laplacian 64x64 (n=4096), t=1, eps=1e-3, all components")
    if name in ("c2", "C2"):
        a = grid_laplacian(1024)
        return Config("c2", a, grid_vector(VECTOR_SEED, a.n), 0.5, 1e-3,
                      "2D 5-point Laplacian 1024x1024 (n=1,048,576), t=0.5, eps=1e-3, all components")
    if name.startswith("grid"):
        g = int(name[4:])
        a = grid_laplacian(g)
        return Config(name, a, grid_vector(VECTOR_SEED, a.n), 1.0, 1e-3, f"2D 5-point Laplacian {g}x{g}")
    raise ValueError(f"unknown config {name!r}")
