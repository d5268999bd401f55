"""Benchmark workloads, package-free (numpy only).

The BASELINE configs' inputs and the `config` dict that both arms of `bench.py` print.  This
module must not import `paper_1904_12754_b200`: the reference arm (`bench.py --impl reference`)
builds its inputs here so that its process never loads the product library.  The product side
builds the same inputs through `paper_1904_12754_b200.configs`; `tests/test_workloads.py` pins the
two bit for bit.

Inputs (no dataset is involved, everything is generated from seeds):
  C1/C2  2-D 5-point Laplacian on g x g interior nodes (row = y*g + x, diag -4, off +1, Dirichlet
         eliminated), v_i = first uniform of stream_for(12345, 0, i, lane 6) (rng.hpp:21-79).
  C3     the reference's own pref(1e6, 5, seed 1) (netgen.cpp:61-107), beta = 1/lambda, lambda from
         50 power iterations started at 1; v = 1.
  C4     R-MAT scale 24 (csrc/gen.cpp); beta = 1/lambda; v = 1; 2^20 seed-chosen components.
  C5     3-D 7-point convection-diffusion on 256^3, cell Peclet 10 along x, t = 0.1,
         v = 2 u - 1 with u from the C1/C2 stream; eps = 1e-4.
Row seed of component r: 1000 + r.
"""
from __future__ import annotations

import numpy as np

VECTOR_SEED = 12345
GRAPH_SEED = 1
ROW_SEED_BASE = 1000

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)

# name -> workload description, eps, t (text), components per job
WORKLOADS = {
    "c1": ("C1: 2D 5-point Laplacian 64x64 (n=4096), t=1, v uniform [0,1) from seed, eps=1e-3, "
           "all 4096 components, reference MLMC driver per component", 1e-3, "1", 4096),
    "c2": ("C2: 2D 5-point Laplacian 1024x1024 (n=1,048,576, 5,238,784 nnz, fp64), t=0.5, v uniform [0,1) from "
           "seed, eps=1e-3, all 1,048,576 components, reference MLMC driver per component", 1e-3, "0.5", 1 << 20),
    "c3": ("C3: Barabasi-Albert n=1,000,000, m=5 (reference pref, seed 1), beta=1/lambda_max (50 power "
           "iterations), v=1, eps=1e-3, all components", 1e-3, "1/lambda_max", 1_000_000),
    "c4": ("C4: R-MAT scale 24 (a=0.57, b=c=0.19), 16*2^24 edges symmetrised, unit weights, beta=1/lambda_max, "
           "v=1, eps=1e-3, 1,048,576 seed-chosen components", 1e-3, "1/lambda_max", 1 << 20),
    "c5": ("C5: 3D 7-point convection-diffusion 256^3 (cell Peclet 10 along x), t=0.1, v uniform [-1,1), "
           "eps=1e-4, 5 MLMC levels, all components", 1e-4, "0.1", 256 ** 3),
}


def config_dict(name: str) -> dict:
    """The `config` object of both bench arms: the workload only (no sample sizes, no
    parallelism, nothing either arm measures) so the two lines compare equal."""
    base = name.split("-")[0]
    if base not in WORKLOADS or name != base:
        return {"workload": f"{name} (scaled-down variant, not a BASELINE config)"}
    desc, eps, t, comps = WORKLOADS[base]
    return {"workload": desc, "epsilon": eps, "t": t, "components_per_job": comps,
            "row_seed": f"{ROW_SEED_BASE} + row"}


def philox_first_uniform(seed: int, level: int, samples, lane: int) -> np.ndarray:
    """First next_uniform() of stream_for(seed, level, s, lane) for every s (rng.hpp:21-66):
    block 0, words (c2, c3) of the Philox4x32-10 output."""
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
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    bits = (c2 << np.uint64(32)) | c3
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def grid_laplacian(g: int):
    """(n, row_ptr, col, val) of the 5-point Laplacian on g x g interior nodes, columns ascending."""
    n = g * g
    r = np.arange(n, dtype=np.int64)
    x, y = r % g, r // g
    cols = np.stack([r - g, r - 1, r, r + 1, r + g], axis=1)
    vals = np.tile(np.array([1.0, 1.0, -4.0, 1.0, 1.0]), (n, 1))
    ok = np.stack([y > 0, x > 0, np.ones(n, bool), x + 1 < g, y + 1 < g], axis=1)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(ok.sum(axis=1))
    return n, rp, cols[ok].astype(np.int64), vals[ok].astype(np.float64)


def convdiff3d(g: int, peclet: float = 10.0, axis: int = 0):
    """(n, row_ptr, col, val): 7-point convection-diffusion on g^3 nodes, diag -6, off 1, upwind /
    downwind 1 +/- Pe/2 along `axis`; columns ascending (-z, -y, -x, self, +x, +y, +z)."""
    n = g ** 3
    r = np.arange(n, dtype=np.int64)
    c3 = (r % g, (r // g) % g, r // (g * g))
    stride = (1, g, g * g)
    up, down = 1.0 + 0.5 * peclet, 1.0 - 0.5 * peclet
    cols, vals, oks = [], [], []
    for dim in (2, 1, 0):
        cols.append(r - stride[dim])
        vals.append(np.full(n, up if dim == axis else 1.0))
        oks.append(c3[dim] > 0)
    cols.append(r)
    vals.append(np.full(n, -6.0))
    oks.append(np.ones(n, bool))
    for dim in (0, 1, 2):
        cols.append(r + stride[dim])
        vals.append(np.full(n, down if dim == axis else 1.0))
        oks.append(c3[dim] + 1 < g)
    cols, vals, ok = np.stack(cols, 1), np.stack(vals, 1), np.stack(oks, 1)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(ok.sum(axis=1))
    return n, rp, cols[ok].astype(np.int64), vals[ok].astype(np.float64)


def power_iteration(n, row_ptr, col, val, iters: int = 50) -> float:
    """lambda_max estimate, the arithmetic of csrc/gen.cpp expmc_power_iteration: x0 = 1, per
    iteration y = A x (row sums in column order), |y|_2 by a SEQUENTIAL sum (np.cumsum), x = y/|y|."""
    x = np.ones(n)
    xn = np.sqrt(float(n))
    lam = 0.0
    for _ in range(iters):
        # row sums in column order: a stable segmented cumulative sum per row
        prod = val * x[col]
        y = _segmented_sequential_sum(prod, row_ptr, n)
        s = float(np.cumsum(y * y)[-1]) if n else 0.0
        yn = np.sqrt(s)
        lam = yn / xn
        if not yn > 0.0:
            break
        x = y / yn
        xn = 1.0
    return float(lam)


def _segmented_sequential_sum(v, row_ptr, n):
    """Per-row sequential left-to-right sum (acc = 0; acc += v[k]) of v over CSR segments, exact
    in the same order as a scalar loop: rows are summed position by position across rows."""
    deg = np.diff(row_ptr)
    out = np.zeros(n)
    if n == 0:
        return out
    order = np.argsort(-deg, kind="stable")
    sdeg = deg[order]
    start = row_ptr[:-1][order]
    acc = np.zeros(n)
    band = min(int(sdeg[0]), 256)  # positions summed across rows; the few wider rows continue below
    for k in range(band):
        cnt = int(np.searchsorted(-sdeg, -k, side="left"))  # rows with deg > k form a prefix
        acc[:cnt] += v[start[:cnt] + k]
    wide = int(np.searchsorted(-sdeg, -band, side="left"))  # rows with deg > band
    for i in range(wide):  # sequential continuation: acc + v[band] + v[band + 1] + ...
        b0 = int(start[i]) + band
        seg = np.empty(int(sdeg[i]) - band + 1)
        seg[0] = acc[i]
        seg[1:] = v[b0:int(start[i]) + int(sdeg[i])]
        acc[i] = np.cumsum(seg)[-1]
    out[order] = acc
    return out


def seeded_rows(n: int, k: int, seed: int = 4242) -> np.ndarray:
    """k distinct seed-chosen components, sorted (configs.seeded_rows)."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(k, n), replace=False)).astype(np.int64)


def row_seeds(rows) -> np.ndarray:
    return (np.asarray(rows, np.uint64) + np.uint64(ROW_SEED_BASE)).astype(np.uint64)
