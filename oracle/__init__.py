"""TEST INFRASTRUCTURE ONLY -- ctypes front end for the CPU oracle.

Two interchangeable back ends with one Python surface:

* ``Oracle``     -- ``oracle/_build/liboracle.so``: the plain-C restatement
                    (``oracle/expmc_oracle.c``), always available (built by ``make -C oracle``
                    or ``__graft_entry__.build()``).
* ``Reference``  -- ``oracle/_ref/libexpmc_ref.so``: the UNMODIFIED reference library
                    (``/root/reference/proj/core``) compiled in place plus the extern "C" shim
                    ``oracle/ref_capi.cpp``.  Present wherever it was built (it is git-ignored
                    but travels to the GPU box with the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package, and only as the checker / CPU baseline.  The
product (``paper_1904_12754_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "_build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libexpmc_ref.so")

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_U32 = C.c_uint32
_D = C.c_double
_INT = C.c_int


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    """std::invalid_argument"""


class OutOfRange(OracleError, IndexError):
    """std::out_of_range"""


class DomainError(OracleError, ArithmeticError):
    """std::domain_error"""


_ERR = {1: InvalidArgument, 2: OutOfRange, 3: DomainError}


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray  # int64[nnz]
    val: np.ndarray  # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @staticmethod
    def from_dense(d) -> "CSR":
        d = np.asarray(d, dtype=np.float64)
        n = d.shape[0]
        rp = [0]
        cols, vals = [], []
        for i in range(n):
            for j in range(n):
                if d[i, j] != 0.0:
                    cols.append(j)
                    vals.append(d[i, j])
            rp.append(len(cols))
        return CSR(n, np.array(rp, np.int64), np.array(cols, np.int64), np.array(vals, np.float64))

    @staticmethod
    def from_triplets(n, trips) -> "CSR":
        """SparseMatrix::from_triplets semantics (sparse.cpp:12-49): sort, sum duplicates in
        input order, drop zero sums."""
        acc: dict = {}
        for (i, j, v) in trips:
            if (i, j) in acc:
                acc[(i, j)] += float(v)
            else:
                acc[(i, j)] = float(v)
        keys = sorted(k for k, v in acc.items() if v != 0.0)
        rp = np.zeros(n + 1, np.int64)
        for (i, _j) in keys:
            rp[i + 1] += 1
        rp = np.cumsum(rp).astype(np.int64)
        col = np.array([j for (_i, j) in keys], np.int64)
        val = np.array([acc[k] for k in keys], np.float64)
        return CSR(n, rp, col, val)

    def transpose(self) -> "CSR":
        """A^T in canonical CSR (SparseMatrix::transpose; forward mode decomposes A^T,
        mlmc.hpp:47-49)."""
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        order = np.lexsort((rows, self.col))  # by new row (= old col), then new col (= old row)
        rp = np.zeros(self.n + 1, np.int64)
        np.add.at(rp, self.col + 1, 1)
        return CSR(self.n, np.cumsum(rp).astype(np.int64), rows[order].copy(), self.val[order].copy())


LEVEL_DT = np.dtype([("level", np.int32), ("pad", np.int32), ("sum", np.float64),
                     ("sum_sq", np.float64), ("samples", np.uint64), ("cost", np.uint64)])


class _Options(C.Structure):
    _fields_ = [("epsilon", _D), ("seed", _U64), ("threads", C.c_int32), ("l0_override", C.c_int32),
                ("warmup", _U64), ("max_levels_above_l0", C.c_int32), ("max_iterations", C.c_int32)]


class _OrcResult(C.Structure):
    _fields_ = [("estimate", _D), ("statistical_error", _D), ("bias_estimate", _D), ("l0", C.c_int32),
                ("L", C.c_int32), ("total_cost", _U64), ("converged", C.c_int32), ("nlevels", C.c_int32),
                ("total_jumps", _U64), ("total_samples", _U64)]


class _RefResult(C.Structure):
    _fields_ = [("estimate", _D), ("statistical_error", _D), ("bias_estimate", _D), ("l0", C.c_int32),
                ("L", C.c_int32), ("total_cost", _U64), ("converged", C.c_int32), ("nlevels", C.c_int32)]


class _Mc(C.Structure):
    _fields_ = [("estimate", _D), ("std_error", _D), ("samples", _U64), ("dt", _D), ("steps", _I64),
                ("wall_cost", _U64)]


class _OrcMc(C.Structure):
    _fields_ = [("estimate", _D), ("std_error", _D), ("samples", _U64), ("dt", _D), ("steps", _I64),
                ("wall_cost", _U64), ("jumps", _U64)]


def _mc_dict(r):
    return dict(estimate=r.estimate, std_error=r.std_error, samples=r.samples, dt=r.dt, steps=r.steps,
                wall_cost=r.wall_cost)


class _OrcStats(C.Structure):
    _fields_ = [("sum", _D), ("sum_sq", _D), ("samples", _U64), ("cost", _U64), ("jumps", _U64)]


def _options(epsilon=1e-3, seed=0, threads=0, l0_override=-1, warmup=1000, max_levels_above_l0=30,
             max_iterations=200):
    return _Options(epsilon, seed, threads, l0_override, warmup, max_levels_above_l0, max_iterations)


class _Backend:
    """Common numpy surface over liboracle.so / libexpmc_ref.so."""

    kind = "?"

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.path = path
        self.lib = C.CDLL(path)

    def _check(self, rc):
        if rc != 0:
            msg = self._last_error()
            raise _ERR.get(rc, OracleError)(msg)

    def uniforms(self, seed, level, sample, lane, count):
        out = np.empty(count, np.float64)
        self._uniforms(_U64(seed), _U32(level), _U64(sample), _U32(lane), _I64(count), _ptr(out))
        return out


class Oracle(_Backend):
    kind = "port"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_chain_n.restype = _I64
        L.orc_chain_edges.restype = _I64
        L.orc_grid_nnz.restype = _I64
        self._uniforms = L.orc_uniforms

    def _last_error(self):
        return self.lib.orc_last_error().decode()

    # ---- inputs
    def grid_laplacian(self, g) -> CSR:
        n = g * g
        nnz = int(self.lib.orc_grid_nnz(_I64(g)))
        rp = np.empty(n + 1, np.int64)
        col = np.empty(nnz, np.int64)
        val = np.empty(nnz, np.float64)
        self.lib.orc_grid_laplacian(_I64(g), _ptr(rp), _ptr(col), _ptr(val))
        return CSR(n, rp, col, val)

    def grid_vector(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.orc_grid_vector(_U64(seed), _I64(n), _ptr(out))
        return out

    def chain(self, a: CSR) -> "OracleChain":
        return OracleChain(self, a)

    def initial_level(self, beta, d_max):
        out = C.c_int()
        self._check(self.lib.orc_initial_level(_D(beta), _D(d_max), C.byref(out)))
        return out.value

    def optimal_allocation(self, v, c, eps):
        v = np.ascontiguousarray(v, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        if v.shape != c.shape:
            raise InvalidArgument("variance and cost arrays differ in length")
        out = np.empty(len(v), np.uint64)
        self._check(self.lib.orc_optimal_allocation(_I64(len(v)), _ptr(v), _ptr(c), _D(eps), _ptr(out)))
        return out

    def bias_estimate(self, means):
        m = np.ascontiguousarray(means, np.float64)
        out = _D()
        self._check(self.lib.orc_bias_estimate(_I64(len(m)), _ptr(m), C.byref(out)))
        return out.value

    def dense_expmv(self, a: CSR, u, beta, threads=0):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(a.n, np.float64)
        threads = threads or os.cpu_count() or 1
        self._check(self.lib.orc_dense_expmv(_I64(a.n), _ptr(a.row_ptr), _ptr(a.col), _ptr(a.val), _ptr(u),
                                             _D(beta), _INT(threads), _ptr(out)))
        return out


class _Chain:
    def decomposition(self):
        n, e = self.n, self.edges
        d = np.empty(n, np.float64)
        rate = np.empty(n, np.float64)
        rp = np.empty(n + 1, np.int64)
        cdf = np.empty(e, np.float64)
        tgt = np.empty(e, np.int64)
        sign = np.empty(e, np.uint8)
        w = np.empty(e, np.float64)
        dmax, dbar = _D(), _D()
        self._export(_ptr(d), _ptr(rate), _ptr(rp), _ptr(cdf), _ptr(tgt), _ptr(sign), _ptr(w),
                     C.byref(dmax), C.byref(dbar))
        return dict(d=d, rate=rate, row_ptr=rp, jump_cdf=cdf, jump_target=tgt, sign=sign,
                    jump_weight=w, d_max=dmax.value, d_bar=dbar.value)


class OracleChain(_Chain):
    def __init__(self, be: Oracle, a: CSR):
        self.be = be
        self.a = a
        h = C.c_void_p()
        be._check(be.lib.orc_decompose(_I64(a.n), _ptr(a.row_ptr), _ptr(a.col), _ptr(a.val), C.byref(h)))
        self.h = h
        self.n = int(be.lib.orc_chain_n(h))
        self.edges = int(be.lib.orc_chain_edges(h))
        self.d_max = self.decomposition()["d_max"]

    def __del__(self):
        try:
            self.be.lib.orc_chain_free(self.h)
        except Exception:
            pass

    def _export(self, *args):
        self.be.lib.orc_chain_export(self.h, *args)

    def samples(self, u, entry, beta, level, base, seed, sample_idx, lane=0):
        idx = np.ascontiguousarray(sample_idx, np.uint64)
        k = len(idx)
        u = np.ascontiguousarray(u, np.float64)
        fine, coarse = np.empty(k), np.empty(k)
        cost, jumps = np.empty(k, np.uint64), np.empty(k, np.uint64)
        end = np.empty(k, np.int64)
        self.be._check(self.be.lib.orc_samples(self.h, _ptr(u), _I64(entry), _D(beta), _INT(level), _INT(int(base)),
                                               _U64(seed), _U32(lane), _I64(k), _ptr(idx), _ptr(fine), _ptr(coarse),
                                               _ptr(cost), _ptr(jumps), _ptr(end)))
        return dict(fine=fine, coarse=coarse, cost=cost, jumps=jumps, end_state=end)

    def run_level(self, u, entry, beta, level, base, first, count, seed, threads=1, lane=0):
        u = np.ascontiguousarray(u, np.float64)
        st = _OrcStats()
        self.be._check(self.be.lib.orc_run_level(self.h, _ptr(u), _I64(entry), _D(beta), _INT(level), _INT(int(base)),
                                                 _U64(first), _U64(count), _U64(seed), _U32(lane), _INT(threads),
                                                 C.byref(st)))
        return dict(sum=st.sum, sum_sq=st.sum_sq, samples=st.samples, cost=st.cost, jumps=st.jumps)

    def driver_rows(self, u, beta, rows, row_seeds, max_levels=40, **opt):
        rows = np.ascontiguousarray(rows, np.int64)
        seeds = np.ascontiguousarray(row_seeds, np.uint64)
        u = np.ascontiguousarray(u, np.float64)
        res = (_OrcResult * len(rows))()
        lv = np.zeros((len(rows), max_levels), LEVEL_DT)
        o = _options(**opt)
        self.be._check(self.be.lib.orc_mlmc_driver_rows(self.h, _ptr(u), _D(beta), C.byref(o), _I64(len(rows)),
                                                        _ptr(rows), _ptr(seeds), res, _ptr(lv), C.c_int32(max_levels)))
        return [dict(estimate=r.estimate, statistical_error=r.statistical_error, bias_estimate=r.bias_estimate,
                     l0=r.l0, L=r.L, total_cost=r.total_cost, converged=bool(r.converged), nlevels=r.nlevels,
                     total_jumps=r.total_jumps, total_samples=r.total_samples, levels=lv[i, :r.nlevels].copy())
                for i, r in enumerate(res)]

    # ---- forward mode (lane 1): this chain must be the decomposition of A^T
    def forward_samples(self, u, beta, level, base, seed, sample_idx):
        r = self.samples(u, 0, beta, level, base, seed, sample_idx, lane=1)
        return r

    def forward_run_level(self, u, beta, level, base, first, count, seed, threads=1):
        return self.run_level(u, 0, beta, level, base, first, count, seed, threads=threads, lane=1)

    def forward_driver(self, u, beta, seeds=None, max_levels=40, **opt):
        """One forward mlmc_driver run per seed (default: opt['seed'] or 0)."""
        seeds = np.ascontiguousarray([opt.get("seed", 0)] if seeds is None else seeds, np.uint64)
        u = np.ascontiguousarray(u, np.float64)
        res = (_OrcResult * len(seeds))()
        lv = np.zeros((len(seeds), max_levels), LEVEL_DT)
        o = _options(**opt)
        self.be._check(self.be.lib.orc_mlmc_driver_forward(self.h, _ptr(u), _D(beta), C.byref(o), _I64(len(seeds)),
                                                           _ptr(seeds), res, _ptr(lv), C.c_int32(max_levels)))
        return [dict(estimate=r.estimate, statistical_error=r.statistical_error, bias_estimate=r.bias_estimate,
                     l0=r.l0, L=r.L, total_cost=r.total_cost, converged=bool(r.converged), nlevels=r.nlevels,
                     total_jumps=r.total_jumps, total_samples=r.total_samples, levels=lv[i, :r.nlevels].copy())
                for i, r in enumerate(res)]

    # ---- fem mode (lane 2): the chain of -M^{-1}K, load = M^{-1}F
    def fem_samples(self, u, load, entry, beta, level, base, seed, sample_idx):
        idx = np.ascontiguousarray(sample_idx, np.uint64)
        k = len(idx)
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        out = {x: np.empty(k) for x in ("value", "eta_f", "eta_c", "integ_f", "integ_c")}
        end = np.empty(k, np.int64)
        cost, jumps = np.empty(k, np.uint64), np.empty(k, np.uint64)
        self.be._check(self.be.lib.orc_fem_samples(
            self.h, _ptr(u), _ptr(load), _I64(entry), _D(beta), _INT(level), _INT(int(base)), _U64(seed), _I64(k),
            _ptr(idx), _ptr(out["value"]), _ptr(out["eta_f"]), _ptr(out["eta_c"]), _ptr(out["integ_f"]),
            _ptr(out["integ_c"]), _ptr(end), _ptr(cost), _ptr(jumps)))
        out.update(end_state=end, cost=cost, jumps=jumps)
        return out

    def fem_run_level(self, u, load, entry, beta, level, base, first, count, seed, threads=1):
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        st = _OrcStats()
        ig = _D()
        self.be._check(self.be.lib.orc_fem_run_level(self.h, _ptr(u), _ptr(load), _I64(entry), _D(beta), _INT(level),
                                                     _INT(int(base)), _U64(first), _U64(count), _U64(seed),
                                                     _INT(threads), C.byref(st), C.byref(ig)))
        return dict(sum=st.sum, sum_sq=st.sum_sq, samples=st.samples, cost=st.cost, jumps=st.jumps,
                    integ_sum=ig.value)

    def fem_driver_rows(self, u, load, beta, rows, row_seeds, max_levels=40, **opt):
        rows = np.ascontiguousarray(rows, np.int64)
        seeds = np.ascontiguousarray(row_seeds, np.uint64)
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        res = (_OrcResult * len(rows))()
        quad = np.zeros(len(rows))
        lv = np.zeros((len(rows), max_levels), LEVEL_DT)
        o = _options(**opt)
        self.be._check(self.be.lib.orc_mlmc_driver_fem(self.h, _ptr(u), _ptr(load), _D(beta), C.byref(o),
                                                       _I64(len(rows)), _ptr(rows), _ptr(seeds), res, _ptr(quad),
                                                       _ptr(lv), C.c_int32(max_levels)))
        return [dict(estimate=r.estimate, statistical_error=r.statistical_error, bias_estimate=r.bias_estimate,
                     quadrature_bound=float(quad[i]), l0=r.l0, L=r.L, total_cost=r.total_cost,
                     converged=bool(r.converged), nlevels=r.nlevels, total_jumps=r.total_jumps,
                     total_samples=r.total_samples, levels=lv[i, :r.nlevels].copy())
                for i, r in enumerate(res)]

    # ---- classical MC (mc.cpp:42-76)
    def mc_single_entry(self, u, entry, beta, dt, samples, seed, threads=4):
        return self._mc(u, entry, beta, dt, samples, seed, 0, threads)

    def mc_forward_scalar(self, u, beta, dt, samples, seed, threads=4):
        return self._mc(u, 0, beta, dt, samples, seed, 1, threads)

    def _mc(self, u, entry, beta, dt, samples, seed, lane, threads):
        u = np.ascontiguousarray(u, np.float64)
        r = _OrcMc()
        self.be._check(self.be.lib.orc_mc(self.h, _ptr(u), _I64(entry), _D(beta), _D(dt), _U64(samples), _U64(seed),
                                          _U32(lane), _INT(threads), C.byref(r)))
        d = _mc_dict(r)
        d["jumps"] = r.jumps
        return d

    def transposed(self) -> "OracleChain":
        return OracleChain(self.be, self.a.transpose())


class Reference(_Backend):
    kind = "reference"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        self._uniforms = L.ref_uniforms

    def _last_error(self):
        return self.lib.ref_last_error().decode()

    def chain(self, a: CSR) -> "RefChain":
        return RefChain(self, a)

    def pref(self, n, d, seed) -> "RefChain":
        h = C.c_void_p()
        self._check(self.lib.ref_pref(_I64(n), _I64(d), _U64(seed), C.byref(h)))
        return RefChain(self, None, handle=h)

    def smallw(self, n, k, p, seed) -> "RefChain":
        h = C.c_void_p()
        self._check(self.lib.ref_smallw(_I64(n), _I64(k), _D(p), _U64(seed), C.byref(h)))
        return RefChain(self, None, handle=h)

    def chain_scaled(self, a: CSR, row_scale) -> "RefChain":
        """decompose_scaled (chain.cpp:80-85)."""
        sc = np.ascontiguousarray(row_scale, np.float64)
        h = C.c_void_p()
        self._check(self.lib.ref_matrix_create_scaled(_I64(a.n), _ptr(a.row_ptr), _ptr(a.col), _ptr(a.val), _ptr(sc),
                                                      C.byref(h)))
        return RefChain(self, None, handle=h)

    def read_matrix_market(self, path) -> "RefChain":
        h = C.c_void_p()
        self._check(self.lib.ref_read_matrix_market(os.fsencode(path), C.byref(h)))
        return RefChain(self, None, handle=h)

    def from_triplets(self, n, rows, cols, vals) -> "RefChain":
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(cols, np.int64)
        v = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        self._check(self.lib.ref_from_triplets(_I64(n), _I64(r.size), _ptr(r), _ptr(c), _ptr(v), C.byref(h)))
        return RefChain(self, None, handle=h)

    def fit_slope(self, x, y, loglog=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = _D()
        self._check(self.lib.ref_fit_slope(_INT(int(loglog)), _I64(x.size), _ptr(x), _ptr(y), C.byref(out)))
        return out.value

    def read_vector(self, path):
        n = _I64()
        self._check(self.lib.ref_read_vector(os.fsencode(path), _I64(0), None, C.byref(n)))
        out = np.empty(n.value)
        self._check(self.lib.ref_read_vector(os.fsencode(path), _I64(n.value), _ptr(out), C.byref(n)))
        return out

    def load_fem_system(self, mass, stiffness, load, u0):
        """load_fem_system (fem.cpp:12-37) -> dict(mass_diag, stiffness: CSR, load, u0)."""
        n, nnz = _I64(), _I64()
        args = [os.fsencode(x) for x in (mass, stiffness, load, u0)]
        self._check(self.lib.ref_load_fem_system(*args, C.byref(n), C.byref(nnz), None, None, None, None, None, None))
        md, ld, u0v = np.empty(n.value), np.empty(n.value), np.empty(n.value)
        rp, col, val = np.empty(n.value + 1, np.int64), np.empty(nnz.value, np.int64), np.empty(nnz.value)
        self._check(self.lib.ref_load_fem_system(*args, C.byref(n), C.byref(nnz), _ptr(md), _ptr(rp), _ptr(col),
                                                 _ptr(val), _ptr(ld), _ptr(u0v)))
        return dict(mass_diag=md, stiffness=CSR(n.value, rp, col, val), load=ld, u0=u0v)

    def solve_convdiff_point(self, mass_diag, stiffness: CSR, load, u0, node, t, max_levels=40, **opt):
        """solve_convdiff_point (fem.cpp:51-73)."""
        md = np.ascontiguousarray(mass_diag, np.float64)
        ld = np.ascontiguousarray(load, np.float64)
        u0 = np.ascontiguousarray(u0, np.float64)
        res = _RefResult()
        lv = np.zeros(max_levels, LEVEL_DT)
        q = _D()
        o = _options(**opt)
        a = stiffness
        self._check(self.lib.ref_solve_convdiff_point(_I64(a.n), _ptr(md), _ptr(a.row_ptr), _ptr(a.col), _ptr(a.val),
                                                      _ptr(ld), _ptr(u0), _I64(node), _D(t), C.byref(o), C.byref(res),
                                                      _ptr(lv), C.c_int32(max_levels), C.byref(q)))
        return _ref_result(res, lv, quadrature_bound=q.value)

    def initial_level(self, beta, d_max):
        out = C.c_int()
        self._check(self.lib.ref_initial_level(_D(beta), _D(d_max), C.byref(out)))
        return out.value

    def optimal_allocation(self, v, c, eps):
        v = np.ascontiguousarray(v, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        out = np.empty(len(v), np.uint64)
        self._check(self.lib.ref_optimal_allocation(_I64(len(v)), _ptr(v), _ptr(c), _D(eps), _ptr(out)))
        return out

    def bias_estimate(self, means):
        m = np.ascontiguousarray(means, np.float64)
        out = _D()
        self._check(self.lib.ref_bias_estimate(_I64(len(m)), _ptr(m), C.byref(out)))
        return out.value


class RefChain(_Chain):
    def __init__(self, be: Reference, a: CSR | None, handle=None):
        self.be = be
        if handle is None:
            h = C.c_void_p()
            be._check(be.lib.ref_matrix_create(_I64(a.n), _ptr(a.row_ptr), _ptr(a.col), _ptr(a.val), C.byref(h)))
            handle = h
        self.h = handle
        n, nnz, e = _I64(), _I64(), _I64()
        be.lib.ref_matrix_sizes(self.h, C.byref(n), C.byref(nnz), C.byref(e))
        self.n, self.nnz, self.edges = n.value, nnz.value, e.value
        if a is None:
            rp = np.empty(self.n + 1, np.int64)
            col = np.empty(self.nnz, np.int64)
            val = np.empty(self.nnz, np.float64)
            be.lib.ref_matrix_csr(self.h, _ptr(rp), _ptr(col), _ptr(val))
            a = CSR(self.n, rp, col, val)
        self.a = a
        self.d_max = self.decomposition()["d_max"]

    def __del__(self):
        try:
            self.be.lib.ref_matrix_destroy(self.h)
        except Exception:
            pass

    def _export(self, *args):
        self.be.lib.ref_matrix_decomposition(self.h, *args)

    def samples(self, u, entry, beta, level, base, seed, sample_idx, lane=0):
        idx = np.ascontiguousarray(sample_idx, np.uint64)
        k = len(idx)
        u = np.ascontiguousarray(u, np.float64)
        fine, coarse = np.empty(k), np.empty(k)
        cost = np.empty(k, np.uint64)
        self.be._check(self.be.lib.ref_samples(self.h, _ptr(u), _I64(entry), _D(beta), _INT(level), _INT(int(base)),
                                               _U64(seed), _U32(lane), _I64(k), _ptr(idx), _ptr(fine), _ptr(coarse),
                                               _ptr(cost)))
        return dict(fine=fine, coarse=coarse, cost=cost)

    def run_level(self, u, entry, beta, level, base, first, count, seed, threads=1, lane=0):
        assert lane == 0
        u = np.ascontiguousarray(u, np.float64)
        s, s2 = _D(), _D()
        m, c = _U64(), _U64()
        self.be._check(self.be.lib.ref_run_level(self.h, _ptr(u), _I64(entry), _D(beta), _INT(level), _INT(int(base)),
                                                 _U64(first), _U64(count), _U64(seed), _INT(threads), C.byref(s),
                                                 C.byref(s2), C.byref(m), C.byref(c)))
        # the reference's RunLevelStats has no jump counter: every fine step of a non-absorbing row ends
        # with one rejected draw, so cost = (jumps + M 2^l) + M 2^l (paths.hpp:22-23, paths.cpp:50-53)
        return dict(sum=s.value, sum_sq=s2.value, samples=m.value, cost=c.value,
                    jumps=max(0, c.value - 2 * m.value * (1 << level)))

    def driver_rows(self, u, beta, rows, row_seeds, max_levels=40, **opt):
        rows = np.ascontiguousarray(rows, np.int64)
        seeds = np.ascontiguousarray(row_seeds, np.uint64)
        u = np.ascontiguousarray(u, np.float64)
        res = (_RefResult * len(rows))()
        lv = np.zeros((len(rows), max_levels), LEVEL_DT)
        o = _options(**opt)
        self.be._check(self.be.lib.ref_mlmc_driver_rows(self.h, _ptr(u), _D(beta), C.byref(o), _I64(len(rows)),
                                                        _ptr(rows), _ptr(seeds), res, _ptr(lv), C.c_int32(max_levels)))
        out = []
        for i, r in enumerate(res):
            levels = lv[i, :r.nlevels].copy()
            steps = np.array([1 << int(l) for l in levels["level"]], np.uint64)
            # transitions = sum_l (cost_l - 2 M_l 2^l): exact for chains without absorbing rows
            jumps = int(np.sum(levels["cost"].astype(np.int64) - 2 * levels["samples"].astype(np.int64) * steps.astype(np.int64)))
            out.append(dict(estimate=r.estimate, statistical_error=r.statistical_error, bias_estimate=r.bias_estimate,
                            l0=r.l0, L=r.L, total_cost=r.total_cost, converged=bool(r.converged), nlevels=r.nlevels,
                            total_jumps=jumps, total_samples=int(levels["samples"].sum()), levels=levels))
        return out

    # ---- forward mode (SampleMode::forward): this chain must hold A^T
    def forward_samples(self, u, beta, level, base, seed, sample_idx):
        idx = np.ascontiguousarray(sample_idx, np.uint64)
        k = len(idx)
        u = np.ascontiguousarray(u, np.float64)
        fine, coarse = np.empty(k), np.empty(k)
        cost = np.empty(k, np.uint64)
        self.be._check(self.be.lib.ref_forward_samples(self.h, _ptr(u), _D(beta), _INT(level), _INT(int(base)),
                                                       _U64(seed), _I64(k), _ptr(idx), _ptr(fine), _ptr(coarse),
                                                       _ptr(cost)))
        return dict(fine=fine, coarse=coarse, cost=cost)

    def forward_run_level(self, u, beta, level, base, first, count, seed, threads=1):
        u = np.ascontiguousarray(u, np.float64)
        s, s2 = _D(), _D()
        m, c = _U64(), _U64()
        self.be._check(self.be.lib.ref_forward_run_level(self.h, _ptr(u), _D(beta), _INT(level), _INT(int(base)),
                                                         _U64(first), _U64(count), _U64(seed), _INT(threads),
                                                         C.byref(s), C.byref(s2), C.byref(m), C.byref(c)))
        return dict(sum=s.value, sum_sq=s2.value, samples=m.value, cost=c.value)

    def forward_driver(self, u, beta, seeds=None, max_levels=40, **opt):
        """One forward mlmc_driver run per seed (the reference takes options.seed)."""
        seeds = [opt.pop("seed", 0)] if seeds is None else list(seeds)
        u = np.ascontiguousarray(u, np.float64)
        out = []
        for sd in seeds:
            res = _RefResult()
            lv = np.zeros(max_levels, LEVEL_DT)
            o = _options(seed=int(sd), **opt)
            self.be._check(self.be.lib.ref_forward_driver(self.h, _ptr(u), _D(beta), C.byref(o), C.byref(res),
                                                          _ptr(lv), C.c_int32(max_levels)))
            out.append(dict(estimate=res.estimate, statistical_error=res.statistical_error,
                            bias_estimate=res.bias_estimate, l0=res.l0, L=res.L, total_cost=res.total_cost,
                            converged=bool(res.converged), nlevels=res.nlevels, levels=lv[:res.nlevels].copy()))
        return out

    def transposed(self) -> "RefChain":
        h = C.c_void_p()
        self.be._check(self.be.lib.ref_transpose(self.h, C.byref(h)))
        return RefChain(self.be, None, handle=h)

    # ---- fem mode (SampleMode::fem)
    def fem_samples(self, u, load, entry, beta, level, base, seed, sample_idx):
        idx = np.ascontiguousarray(sample_idx, np.uint64)
        k = len(idx)
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        out = {x: np.empty(k) for x in ("value", "eta_f", "eta_c", "integ_f", "integ_c")}
        end = np.empty(k, np.int64)
        cost = np.empty(k, np.uint64)
        self.be._check(self.be.lib.ref_fem_samples(
            self.h, _ptr(u), _ptr(load), _I64(entry), _D(beta), _INT(level), _INT(int(base)), _U64(seed), _I64(k),
            _ptr(idx), _ptr(out["value"]), _ptr(out["eta_f"]), _ptr(out["eta_c"]), _ptr(out["integ_f"]),
            _ptr(out["integ_c"]), _ptr(end), _ptr(cost)))
        out.update(end_state=end, cost=cost)
        return out

    def fem_run_level(self, u, load, entry, beta, level, base, first, count, seed, threads=1):
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        s, s2 = _D(), _D()
        m, c = _U64(), _U64()
        self.be._check(self.be.lib.ref_fem_run_level(self.h, _ptr(u), _ptr(load), _I64(entry), _D(beta), _INT(level),
                                                     _INT(int(base)), _U64(first), _U64(count), _U64(seed),
                                                     _INT(threads), C.byref(s), C.byref(s2), C.byref(m), C.byref(c)))
        return dict(sum=s.value, sum_sq=s2.value, samples=m.value, cost=c.value)

    def fem_driver_rows(self, u, load, beta, rows, row_seeds, max_levels=40, **opt):
        u = np.ascontiguousarray(u, np.float64)
        load = np.ascontiguousarray(load, np.float64)
        out = []
        for row, sd in zip(rows, row_seeds):
            res = _RefResult()
            lv = np.zeros(max_levels, LEVEL_DT)
            q = _D()
            o = _options(seed=int(sd), **opt)
            self.be._check(self.be.lib.ref_fem_driver(self.h, _ptr(u), _ptr(load), _I64(int(row)), _D(beta),
                                                      C.byref(o), C.byref(res), _ptr(lv), C.c_int32(max_levels),
                                                      C.byref(q)))
            out.append(_ref_result(res, lv, quadrature_bound=q.value))
        return out

    # ---- classical MC (mc.cpp:42-113)
    def mc_single_entry(self, u, entry, beta, dt, samples, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        r = _Mc()
        self.be._check(self.be.lib.ref_mc_single_entry(self.h, _ptr(u), _I64(entry), _D(beta), _D(dt), _U64(samples),
                                                       _U64(seed), _INT(threads), C.byref(r)))
        return _mc_dict(r)

    def mc_forward_scalar(self, u, beta, dt, samples, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        r = _Mc()
        self.be._check(self.be.lib.ref_mc_forward_scalar(self.h, _ptr(u), _D(beta), _D(dt), _U64(samples),
                                                         _U64(seed), _INT(threads), C.byref(r)))
        return _mc_dict(r)

    def mc_auto(self, u, entry, beta, epsilon, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        r = _Mc()
        self.be._check(self.be.lib.ref_mc_auto(self.h, _ptr(u), _I64(entry), _D(beta), _D(epsilon), _U64(seed),
                                               _INT(threads), C.byref(r)))
        return _mc_dict(r)

    # ---- paper-figure harness (harness.cpp:61-144)
    def bench_levels(self, u, entry, beta, l0, count, samples, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        rows = np.zeros((count, 5))
        slopes = np.zeros(3)
        self.be._check(self.be.lib.ref_bench_levels(self.h, _ptr(u), _I64(entry), _D(beta), _INT(l0), _INT(count),
                                                    _U64(samples), _U64(seed), _INT(threads), _ptr(rows),
                                                    _ptr(slopes)))
        return rows, slopes

    def bench_l0(self, u, entry, beta, l0_min, l0_max, epsilon, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        costs = np.zeros(l0_max - l0_min + 1)
        best, heur = C.c_int(), C.c_int()
        self.be._check(self.be.lib.ref_bench_l0(self.h, _ptr(u), _I64(entry), _D(beta), _INT(l0_min), _INT(l0_max),
                                                _D(epsilon), _U64(seed), _INT(threads), _ptr(costs), C.byref(best),
                                                C.byref(heur)))
        return costs, best.value, heur.value

    def bench_complexity(self, u, entry, beta, epsilons, seed, threads=4):
        u = np.ascontiguousarray(u, np.float64)
        eps = np.ascontiguousarray(epsilons, np.float64)
        ml, mc, sl = np.zeros(eps.size), np.zeros(eps.size), np.zeros(2)
        self.be._check(self.be.lib.ref_bench_complexity(self.h, _ptr(u), _I64(entry), _D(beta), _I64(eps.size),
                                                        _ptr(eps), _U64(seed), _INT(threads), _ptr(ml), _ptr(mc),
                                                        _ptr(sl)))
        return ml, mc, sl

    def dense_expmv(self, u, beta):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.n, np.float64)
        self.be._check(self.be.lib.ref_dense_expmv(self.h, _ptr(u), _D(beta), _ptr(out)))
        return out

    def strang_reference(self, u, beta, steps):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.n, np.float64)
        self.be._check(self.be.lib.ref_strang_reference(self.h, _ptr(u), _D(beta), _I64(steps), _ptr(out)))
        return out


def _ref_result(res, lv, **extra):
    d = dict(estimate=res.estimate, statistical_error=res.statistical_error, bias_estimate=res.bias_estimate,
             l0=res.l0, L=res.L, total_cost=res.total_cost, converged=bool(res.converged), nlevels=res.nlevels,
             levels=lv[:res.nlevels].copy())
    d.update(extra)
    return d


def have_reference() -> bool:
    return os.path.exists(REF_SO)
