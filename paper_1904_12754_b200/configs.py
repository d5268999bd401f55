"""Synthetic inputs of the BASELINE configs (host-side input generation, not the hot path).

C1 / C2 (BASELINE.json configs[0], configs[1]): 2-D 5-point Laplacian on a g x g
grid of interior nodes (row = y*g + x, diag -4, off-diagonal +1, Dirichlet boundary
eliminated), v_i uniform in [0,1) drawn from the reference's own Philox stream
stream_for(seed, 0, i, lane 6) (rng.hpp:76-79; lanes 0-3 and 7 are taken by the reference),
t = 1 (C1) / 0.5 (C2), eps = 1e-3.  Per-row driver seed = 1000 + row.
There is no public dataset behind these configs: everything is generated from seeds.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import SparseMatrix, _check, _ptr, _take_matrix

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
    sampler: str = "reference"         # the path sampler the config is run with
    rows: np.ndarray | None = None     # components to estimate (None: all)
    max_levels_above_l0: int = 30      # MlmcOptions.max_levels_above_l0
    extra: dict = field(default_factory=dict)


VECTOR_SEED = 12345  # v = stream_for(12345, 0, i, 6), as in the survey probes
GRAPH_SEED = 1       # BA / R-MAT seed (SURVEY §8d probes used seed 1 for C3)


# ---------------------------------------------------------------- native generators (csrc/gen.cpp)
def _take(h) -> SparseMatrix:
    return _take_matrix(h)


def gen_ba(n: int, d: int, seed: int) -> SparseMatrix:
    """Barabasi-Albert adjacency, the reference's pref(n, d, seed) (netgen.cpp:61-107)."""
    h = C.c_void_p()
    _check(L.lib.expmc_gen_ba(n, d, seed, C.byref(h)))
    return _take(h)


def gen_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
             seed: int = GRAPH_SEED) -> SparseMatrix:
    """Symmetrised unit-weight R-MAT graph on 2^scale nodes (BASELINE config 4)."""
    h = C.c_void_p()
    _check(L.lib.expmc_gen_rmat(scale, edge_factor, a, b, c, seed, C.byref(h)))
    return _take(h)


def gen_convdiff3d(g: int, peclet: float = 10.0, axis: int = 0) -> SparseMatrix:
    """3-D 7-point convection-diffusion on g^3 nodes (BASELINE config 5): diag -6, off 1,
    upwind/downwind 1 +/- Pe/2 along `axis` (x by default: Pe = 10 gives +6 / -4)."""
    h = C.c_void_p()
    _check(L.lib.expmc_gen_convdiff3d(g, peclet, axis, C.byref(h)))
    return _take(h)


def power_iteration(a: SparseMatrix, iters: int = 50) -> float:
    rp = np.ascontiguousarray(a.row_ptr, np.int64)
    col = np.ascontiguousarray(a.col, np.int64)
    val = np.ascontiguousarray(a.val, np.float64)
    csr = L.Csr(a.n, int(rp[-1]), _ptr(rp), _ptr(col), _ptr(val))
    lam = C.c_double()
    _check(L.lib.expmc_power_iteration(C.byref(csr), iters, C.byref(lam)))
    return lam.value


def seeded_rows(n: int, k: int, seed: int = 4242) -> np.ndarray:
    """k distinct seed-chosen components, sorted."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(k, n), replace=False)).astype(np.int64)


def _graph_config(name, a, desc, rows=None) -> Config:
    # e^{A / lambda} 1 = e^{beta A} 1 with beta = 1 / lambda: the unscaled 0/1 adjacency keeps every
    # row's CDF exactly uniform (kUniformRow); both arms are run on the same (A, beta).
    lam = power_iteration(a, 50)
    return Config(name, a, np.ones(a.n), 1.0 / lam, 1e-3, desc + f"; lambda_max~{lam:.4g} (50 power iterations), "
                  "beta = 1/lambda, v = 1 (total communicability)", sampler="event", rows=rows,
                  extra={"lambda": lam})


def make_config(name: str) -> Config:
    name = name.lower()
    if name == "c1":
        a = grid_laplacian(64)
        return Config("c1", a, grid_vector(VECTOR_SEED, a.n), 1.0, 1e-3,
                      "2D 5-point Laplacian 64x64 (n=4096), t=1, eps=1e-3, all components")
    if name == "c2":
        a = grid_laplacian(1024)
        return Config("c2", a, grid_vector(VECTOR_SEED, a.n), 0.5, 1e-3,
                      "2D 5-point Laplacian 1024x1024 (n=1,048,576), t=0.5, eps=1e-3, all components")
    if name.startswith("grid"):
        g = int(name[4:])
        a = grid_laplacian(g)
        return Config(name, a, grid_vector(VECTOR_SEED, a.n), 1.0, 1e-3, f"2D 5-point Laplacian {g}x{g}")
    if name == "c3" or name.startswith("c3-"):
        n = int(name[3:]) if "-" in name else 1_000_000
        return _graph_config(name, gen_ba(n, 5, GRAPH_SEED),
                             f"Barabasi-Albert n={n}, m=5 (reference pref algorithm, seed {GRAPH_SEED})")
    if name == "c4" or name.startswith("c4-"):
        scale = int(name[3:]) if "-" in name else 24
        a = gen_rmat(scale, 16)
        return _graph_config(name, a, f"R-MAT scale {scale} (a=0.57, b=c=0.19, d=0.05), 16*2^{scale} edges, "
                             "symmetrised, unit weights", rows=seeded_rows(a.n, min(a.n, 1 << 20)))
    if name == "c5" or name.startswith("c5-"):
        g = int(name[3:]) if "-" in name else 256
        a = gen_convdiff3d(g, 10.0, 0)
        u = 2.0 * philox_first_uniform(VECTOR_SEED, 0, np.arange(a.n, dtype=np.uint64), 6) - 1.0
        return Config(name, a, u, 0.1, 1e-4,
                      f"3D 7-point convection-diffusion {g}^3 (cell Peclet 10 along x: off-diagonals +6/-4/1), "
                      "t=0.1, v uniform [-1,1), eps=1e-4, 5 MLMC levels", max_levels_above_l0=4,
                      sampler="event")  # alias picks on its non-uniform rows (tests/test_alias.py)
    raise ValueError(f"unknown config {name!r}")
