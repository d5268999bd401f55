"""Host API mirroring the reference's C++ interface for the MLMC path (names, argument
meaning and error behaviour of expmc::run_level / mlmc_driver, mlmc.hpp:15-98), backed by the
CUDA library through the C-ABI (include/expmc_b200.h).

    reference (C++)                               here (Python over the C-ABI)
    ---------------------------------------       -------------------------------------------
    SparseMatrix::from_triplets (sparse.cpp:12)   SparseMatrix.from_triplets
    decompose(A) (chain.cpp:75)                   Context(A, u, device)  (tables built on GPU)
    MlmcProblem{dec, u, entry, beta, mode}         MlmcProblem(ctx, entry, beta, mode)
      (mlmc.hpp:45-57; forward: dec of A^T)         (forward: Context(A.transpose(), u))
    run_level(p, l, base, first, add, seed)       run_level(p, l, base, first, add, seed)
    mlmc_driver(p, opts) (mlmc.cpp:170)           mlmc_driver(p, opts)
    --                                            mlmc_driver_rows(ctx, beta, rows, seeds, opts)
    --                                            mlmc_driver_forward(ctx, beta, seeds, opts)
    initial_level / optimal_allocation /          initial_level / optimal_allocation /
      bias_estimate (mlmc.cpp:19-51)                bias_estimate (same host C++ as the driver)

Exceptions: std::invalid_argument -> InvalidArgument(ValueError), std::out_of_range ->
OutOfRange(IndexError), std::domain_error -> DomainError(ArithmeticError); CUDA failures ->
CudaError.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


LANE_ENTRY, LANE_FORWARD, LANE_FEM = L.LANE_ENTRY, L.LANE_FORWARD, L.LANE_FEM  # Philox lanes (mlmc.cpp:94-96)


class ExpmcError(RuntimeError):
    pass


class InvalidArgument(ExpmcError, ValueError):
    pass


class OutOfRange(ExpmcError, IndexError):
    pass


class DomainError(ExpmcError, ArithmeticError):
    pass


class CudaError(ExpmcError):
    pass


class NotImplementedMode(ExpmcError, NotImplementedError):
    pass


class IoError(ExpmcError):
    """std::runtime_error of the readers: "path:line: what" (io.cpp)."""


class StepOverflowError(ExpmcError, OverflowError):
    """std::overflow_error (mc_auto)."""


_ERR = {L.EXPMC_EINVAL: InvalidArgument, L.EXPMC_ERANGE: OutOfRange, L.EXPMC_EDOMAIN: DomainError,
        L.EXPMC_ECUDA: CudaError, L.EXPMC_ENOTIMPL: NotImplementedMode, L.EXPMC_EIO: IoError,
        L.EXPMC_EOVERFLOW: StepOverflowError}


def _check(rc: int) -> None:
    if rc != L.EXPMC_OK:
        raise _ERR.get(rc, ExpmcError)(L.lib.expmc_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def version() -> str:
    return L.lib.expmc_version().decode()


def device_count() -> int:
    n = C.c_int()
    _check(L.lib.expmc_device_count(C.byref(n)))
    return n.value


# --------------------------------------------------------------------------------- matrices
@dataclass
class SparseMatrix:
    """Canonical CSR as expmc::SparseMatrix stores it (sparse.hpp:21-75)."""

    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0

    @staticmethod
    def from_triplets(n: int, rows, cols, vals) -> "SparseMatrix":
        """sparse.cpp:12-49 in the native builder (csrc/io.cpp): indices checked (out_of_range),
        values finite (invalid_argument), sorted by (row, col), duplicates summed exactly as the
        reference sums them, zero sums dropped."""
        r = np.ascontiguousarray(rows, np.int64).ravel()
        c = np.ascontiguousarray(cols, np.int64).ravel()
        v = np.ascontiguousarray(vals, np.float64).ravel()
        if not (r.size == c.size == v.size):
            raise InvalidArgument("triplet arrays differ in length")
        h = C.c_void_p()
        _check(L.lib.expmc_csr_from_triplets(int(n), r.size, _ptr(r), _ptr(c), _ptr(v), C.byref(h)))
        return _take_matrix(h)

    @staticmethod
    def from_dense(d) -> "SparseMatrix":
        d = np.asarray(d, np.float64)
        r, c = np.nonzero(d)
        return SparseMatrix.from_triplets(d.shape[0], r, c, d[r, c])

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        i = np.arange(n)
        return SparseMatrix.from_triplets(n, i, i, np.ones(n))

    def transposed(self) -> "SparseMatrix":
        r = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        return SparseMatrix.from_triplets(self.n, self.col, r, self.val)

    def multiply(self, x):
        x = np.asarray(x, np.float64)
        r = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        y = np.zeros(self.n)
        np.add.at(y, r, self.val * x[self.col])
        return y


def _take_matrix(h) -> SparseMatrix:
    """Copy a library-owned expmc_matrix into a SparseMatrix and free it."""
    n, nnz = C.c_int64(), C.c_int64()
    try:
        _check(L.lib.expmc_matrix_info(h, C.byref(n), C.byref(nnz)))
        rp = np.empty(n.value + 1, np.int64)
        col = np.empty(nnz.value, np.int64)
        val = np.empty(nnz.value, np.float64)
        _check(L.lib.expmc_matrix_copy(h, _ptr(rp), _ptr(col), _ptr(val)))
    finally:
        L.lib.expmc_matrix_destroy(h)
    return SparseMatrix(n.value, rp, col, val)


def read_matrix_market(path) -> SparseMatrix:
    """io.cpp:69-128 (native, multi-threaded): coordinate real general|symmetric."""
    h = C.c_void_p()
    _check(L.lib.expmc_read_matrix_market(os.fsencode(path), C.byref(h)))
    return _take_matrix(h)


def read_vector(path) -> np.ndarray:
    """io.cpp:154-167: every whitespace-separated real of every non-comment line."""
    n = C.c_int64()
    _check(L.lib.expmc_read_vector(os.fsencode(path), 0, None, C.byref(n)))
    out = np.empty(n.value)
    _check(L.lib.expmc_read_vector(os.fsencode(path), out.size, _ptr(out), C.byref(n)))
    return out


# --------------------------------------------------------------------------------- stats
@dataclass
class LevelStats:
    """mlmc.hpp:18-31 (+ jumps: accepted CTMC transitions)."""

    level: int = 0
    sum: float = 0.0
    sum_sq: float = 0.0
    samples: int = 0
    cost: int = 0
    jumps: int = 0

    def mean(self) -> float:
        return self.sum / self.samples if self.samples else 0.0

    def variance(self) -> float:  # mlmc.cpp:13-17
        if self.samples < 2:
            return 0.0
        m = self.mean()
        return max(0.0, self.sum_sq / self.samples - m * m)

    def unit_cost(self) -> float:
        return self.cost / self.samples if self.samples else 0.0


@dataclass
class MlmcOptions:
    """mlmc.hpp:59-67."""

    epsilon: float = 1e-3
    seed: int = 0
    threads: int = 0
    l0_override: int = -1
    warmup: int = 1000
    max_levels_above_l0: int = 30
    max_iterations: int = 200
    max_cost: float = 0.0  # extension: per-component model-unit budget (0 = off, the reference)

    def _c(self) -> L.OptionsC:
        return L.OptionsC(self.epsilon, self.seed, self.threads, self.l0_override, self.warmup,
                          self.max_levels_above_l0, self.max_iterations, self.max_cost)


@dataclass
class MlmcResult:
    """mlmc.hpp:33-43 (+ total_jumps / total_samples)."""

    estimate: float = 0.0
    statistical_error: float = 0.0
    bias_estimate: float = 0.0
    quadrature_bound: float = 0.0
    levels: list = field(default_factory=list)
    l0: int = 0
    L: int = 0
    total_cost: int = 0
    converged: bool = False
    total_jumps: int = 0
    total_samples: int = 0
    projected_cost: float = 0.0
    over_budget: bool = False


# --------------------------------------------------------------------------------- context
class Context:
    """Device-resident sampling tables of A plus the bound vector u on one GPU
    (decompose + LevelSampler tables + MlmcProblem::u)."""

    SAMPLERS = {"reference": L.SAMPLER_REFERENCE, "event": L.SAMPLER_EVENT}

    def __init__(self, a: SparseMatrix, u, device: int = 0, sampler: str = "reference", row_scale=None,
                 load=None):
        """row_scale: decompose_scaled (chain.cpp:80-85), the tables of diag(row_scale) A;
        load: the fem load vector (MlmcProblem::load)."""
        self._h = C.c_void_p()
        u = np.ascontiguousarray(u, np.float64)
        if u.shape != (a.n,):
            raise InvalidArgument("vector length does not match decomposition")
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        col = np.ascontiguousarray(a.col, np.int64)
        val = np.ascontiguousarray(a.val, np.float64)
        csr = L.Csr(a.n, int(rp[-1]) if len(rp) else 0, _ptr(rp), _ptr(col), _ptr(val))
        if row_scale is None:
            _check(L.lib.expmc_ctx_create(C.byref(csr), _ptr(u), device, C.byref(self._h)))
        else:
            sc = np.ascontiguousarray(row_scale, np.float64)
            if sc.shape != (a.n,):
                raise InvalidArgument("row scale length does not match matrix dimension")
            _check(L.lib.expmc_ctx_create_scaled(C.byref(csr), _ptr(sc), _ptr(u), device, C.byref(self._h)))
        info = L.CtxInfo()
        _check(L.lib.expmc_ctx_get_info(self._h, C.byref(info)))
        self.n = info.n
        self.n_edges = info.n_edges
        self.d_max = info.d_max
        self.d_bar = info.d_bar
        self.device = info.device
        self.num_sms = info.num_sms
        self.table_bytes = info.table_bytes
        self.set_sampler(sampler)
        if load is not None:
            self.set_load(load)

    def set_sampler(self, sampler: str):
        """'reference' (draw-for-draw the reference's sampler, exact parity) or 'event'
        (one exponential clock per jump; same law, O(jumps) per path)."""
        if sampler not in self.SAMPLERS:
            raise InvalidArgument(f"unknown sampler {sampler!r}")
        _check(L.lib.expmc_ctx_set_sampler(self._h, self.SAMPLERS[sampler]))
        self.sampler = sampler

    def set_full_hold(self, full: bool):
        """Event sampler only: evaluate every first holding interval in full (True) instead of
        the closed-form stay-at-entry decision (False, the default) -- same outcomes; A/B tests."""
        self._flags = (getattr(self, "_flags", 0) & ~1) | (1 if full else 0)
        _check(L.lib.expmc_ctx_set_sampler_flags(self._h, self._flags))

    def set_log_hold(self, log: bool):
        """Reference-order sampler: run every holding test in time space with a logarithm
        (True) instead of probability space (False, the default) -- same draws and outcomes up
        to ulp ties; A/B tests."""
        self._flags = (getattr(self, "_flags", 0) & ~2) | (2 if log else 0)
        _check(L.lib.expmc_ctx_set_sampler_flags(self._h, self._flags))

    def set_row_gather(self, separate: bool):
        """Event sampler: read the target's row record with a second gather (True) instead of
        the per-edge record carrying the target row's payload (False, the default) -- same draws
        and outcomes; A/B tests."""
        self._flags = (getattr(self, "_flags", 0) & ~8) | (8 if separate else 0)
        _check(L.lib.expmc_ctx_set_sampler_flags(self._h, self._flags))

    def set_screen_each(self, each: bool):
        """Event sampler, entry mode: test every sample's first draw for "never leaves the
        entry" (True) instead of locating the chunk's jumpers by geometric gaps (False, the
        default) -- same law; A/B tests."""
        self._flags = (getattr(self, "_flags", 0) & ~4) | (4 if each else 0)
        _check(L.lib.expmc_ctx_set_sampler_flags(self._h, self._flags))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib.expmc_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_vector(self, u):
        u = np.ascontiguousarray(u, np.float64)
        if u.shape != (self.n,):
            raise InvalidArgument("vector length does not match decomposition")
        _check(L.lib.expmc_ctx_set_vector(self._h, _ptr(u)))

    def set_load(self, load):
        """MlmcProblem::load for fem mode (length n)."""
        g = np.ascontiguousarray(load, np.float64)
        if g.shape != (self.n,):
            raise InvalidArgument("load length does not match decomposition")
        _check(L.lib.expmc_ctx_set_load(self._h, _ptr(g)))

    def sample_records(self, beta: float, entry, level, base_level, seed, sample_idx,
                       lane: int = L.LANE_ENTRY) -> np.ndarray:
        """Per-sample records of any lane (SAMPLE_RECORD_DT: eta_fine, eta_coarse, value,
        integ_fine, integ_coarse, cost, jumps, end_state)."""
        e, lv, b, sd, i = np.broadcast_arrays(np.asarray(entry, np.int64), np.asarray(level, np.int32),
                                              np.asarray(base_level, np.int32), np.asarray(seed, np.uint64),
                                              np.asarray(sample_idx, np.uint64))
        k = e.size
        req = np.zeros(k, _REQ_DT)
        req["entry"], req["seed"], req["first_index"] = e.ravel(), sd.ravel(), i.ravel()
        req["count"], req["level"], req["base_level"] = 1, lv.ravel(), b.ravel()
        out = np.zeros(k, SAMPLE_RECORD_DT)
        _check(L.lib.expmc_sample_debug_ex(self._h, beta, lane, k, _ptr(req), _ptr(out)))
        return out

    def decomposition(self) -> dict:
        n, m = self.n, self.n_edges
        d, rate = np.empty(n), np.empty(n)
        rp = np.empty(n + 1, np.int64)
        cdf, tgt, sign = np.empty(m), np.empty(m, np.int64), np.empty(m, np.uint8)
        _check(L.lib.expmc_ctx_export_tables(self._h, _ptr(d), _ptr(rate), _ptr(rp), _ptr(cdf), _ptr(tgt), _ptr(sign)))
        return dict(d=d, rate=rate, row_ptr=rp, jump_cdf=cdf, jump_target=tgt, sign=sign, d_max=self.d_max,
                    d_bar=self.d_bar)

    def alias_tables(self) -> dict | None:
        """The event sampler's alias records of the non-uniform rows (None when none were built:
        reference sampler, or every row uniform): per edge slot `prob`, and the target words
        `self` / `alias` (column, or -(column + 1) for a negative entry)."""
        rows = C.c_uint64()
        _check(L.lib.expmc_ctx_export_alias(self._h, None, None, None, C.byref(rows)))
        if rows.value == 0:
            return None
        m = self.n_edges
        prob, own, alias = np.empty(m), np.empty(m, np.int64), np.empty(m, np.int64)
        _check(L.lib.expmc_ctx_export_alias(self._h, _ptr(prob), _ptr(own), _ptr(alias), C.byref(rows)))
        return dict(prob=prob, self=own, alias=alias, rows=int(rows.value))

    def counters(self) -> dict:
        c = L.CountersC()
        _check(L.lib.expmc_ctx_get_counters(self._h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in L.CountersC._fields_}

    # ---- sample sharding over GPUs (one process per GPU)
    def shard_samples(self, nccl_id: bytes, rank: int, world: int):
        """Collective over the `world` ranks: every rank then samples the chunks g % world == rank
        of every batch and the chunk partials are summed exactly over NCCL (results are bit-for-bit
        one GPU's)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(L.lib.expmc_ctx_shard_samples(self._h, C.cast(buf, C.c_void_p), rank, world))

    def set_shard(self, rank: int, world: int):
        """The chunk filter alone (no exchange): single-GPU emulation of a rank."""
        _check(L.lib.expmc_ctx_set_shard(self._h, rank, world))

    def last_partials(self) -> dict:
        n = C.c_int64()
        _check(L.lib.expmc_ctx_last_partials(self._h, C.byref(n), None, None, None, None))
        k = n.value
        s, s2 = np.empty(k), np.empty(k)
        c, j = np.empty(k, np.uint64), np.empty(k, np.uint64)
        _check(L.lib.expmc_ctx_last_partials(self._h, C.byref(n), _ptr(s), _ptr(s2), _ptr(c), _ptr(j)))
        return dict(sum=s, sum_sq=s2, cost=c, jumps=j)

    @property
    def stream_ptr(self) -> int:
        """cudaStream_t the sampler kernels run on (for CUDA-event timing on that stream)."""
        p = C.c_void_p()
        _check(L.lib.expmc_ctx_get_stream(self._h, C.byref(p)))
        return p.value or 0

    def reset_counters(self):
        _check(L.lib.expmc_ctx_reset_counters(self._h))

    # ---- batched primitives
    def run_level_batch(self, beta: float, entry, level, base_level, first_index, count, seed,
                        lane: int = L.LANE_ENTRY) -> np.ndarray:
        """Vectorised run_level: every argument broadcasts to the request count.  Returns a
        structured array (sum, sum_sq, samples, cost, jumps).  lane=LANE_FORWARD: forward mode
        (entry ignored)."""
        e, lv, b, f, c, s = np.broadcast_arrays(np.asarray(entry, np.int64), np.asarray(level, np.int32),
                                                np.asarray(base_level, np.int32), np.asarray(first_index, np.uint64),
                                                np.asarray(count, np.uint64), np.asarray(seed, np.uint64))
        k = e.size
        req = np.zeros(k, _REQ_DT)
        req["entry"], req["seed"], req["first_index"] = e.ravel(), s.ravel(), f.ravel()
        req["count"], req["level"], req["base_level"] = c.ravel(), lv.ravel(), b.ravel()
        out = np.zeros(k, _STATS_DT)
        _check(L.lib.expmc_run_level_batch(self._h, beta, lane, k, _ptr(req), _ptr(out)))
        return out

    def sample_debug(self, beta: float, entry, level, base_level, seed, sample_idx, lane: int = L.LANE_ENTRY) -> dict:
        e, lv, b, s, i = np.broadcast_arrays(np.asarray(entry, np.int64), np.asarray(level, np.int32),
                                             np.asarray(base_level, np.int32), np.asarray(seed, np.uint64),
                                             np.asarray(sample_idx, np.uint64))
        k = e.size
        req = np.zeros(k, _REQ_DT)
        req["entry"], req["seed"], req["first_index"] = e.ravel(), s.ravel(), i.ravel()
        req["count"], req["level"], req["base_level"] = 1, lv.ravel(), b.ravel()
        fine, coarse = np.empty(k), np.empty(k)
        cost, jumps, end = np.empty(k, np.uint64), np.empty(k, np.uint64), np.empty(k, np.int64)
        _check(L.lib.expmc_sample_debug(self._h, beta, lane, k, _ptr(req), _ptr(fine), _ptr(coarse),
                                        _ptr(cost), _ptr(jumps), _ptr(end)))
        return dict(fine=fine, coarse=coarse, cost=cost, jumps=jumps, end_state=end)


_REQ_DT = np.dtype([("entry", np.int64), ("seed", np.uint64), ("first_index", np.uint64), ("count", np.uint64),
                    ("level", np.int32), ("base_level", np.int32)])
_STATS_DT = np.dtype([("sum", np.float64), ("sum_sq", np.float64), ("samples", np.uint64), ("cost", np.uint64),
                      ("jumps", np.uint64), ("integ_sum", np.float64)])
_RESULT_DT = np.dtype([("estimate", np.float64), ("statistical_error", np.float64), ("bias_estimate", np.float64),
                       ("l0", np.int32), ("L", np.int32), ("total_cost", np.uint64), ("converged", np.int32),
                       ("nlevels", np.int32), ("total_jumps", np.uint64), ("total_samples", np.uint64),
                       ("projected_cost", np.float64), ("over_budget", np.int32), ("pad", np.int32),
                       ("quadrature_bound", np.float64)])
SAMPLE_RECORD_DT = np.dtype([("eta_fine", np.float64), ("eta_coarse", np.float64), ("value", np.float64),
                             ("integ_fine", np.float64), ("integ_coarse", np.float64), ("cost", np.uint64),
                             ("jumps", np.uint64), ("end_state", np.int64)])
LEVEL_RECORD_DT = np.dtype([("level", np.int32), ("pad", np.int32), ("sum", np.float64), ("sum_sq", np.float64),
                            ("samples", np.uint64), ("cost", np.uint64)])
assert _REQ_DT.itemsize == C.sizeof(L.LevelReq)
assert _STATS_DT.itemsize == C.sizeof(L.LevelStatsC)
assert _RESULT_DT.itemsize == C.sizeof(L.ResultC)
assert LEVEL_RECORD_DT.itemsize == C.sizeof(L.LevelRecordC)
assert SAMPLE_RECORD_DT.itemsize == C.sizeof(L.SampleRecordC)


class SampleMode(enum.IntEnum):
    """mlmc.hpp:45."""

    entry = 0
    forward = 1
    fem = 2


@dataclass
class MlmcProblem:
    """mlmc.hpp:47-57: the context carries dec and u.  entry mode estimates (e^{beta A} u)_entry
    on Context(A, u); forward mode estimates sum(e^{beta A} u) on Context(A^T, u)."""

    ctx: Context
    entry: int = 0
    beta: float = 1.0
    mode: SampleMode = SampleMode.entry


def _mode(problem: MlmcProblem) -> SampleMode:
    return SampleMode(problem.mode)


def run_level(problem: MlmcProblem, level: int, base_level: bool, first_index: int, additional: int,
              seed: int, threads: int = 0) -> LevelStats:
    """mlmc.hpp:86-88."""
    out = L.LevelStatsC()
    mode = _mode(problem)
    if mode == SampleMode.forward:
        _check(L.lib.expmc_run_level_forward(problem.ctx.handle, problem.beta, level, int(bool(base_level)),
                                             first_index, additional, seed, C.byref(out)))
    elif mode == SampleMode.fem:
        _check(L.lib.expmc_run_level_fem(problem.ctx.handle, problem.entry, problem.beta, level,
                                         int(bool(base_level)), first_index, additional, seed, C.byref(out)))
    else:
        _check(L.lib.expmc_run_level(problem.ctx.handle, problem.entry, problem.beta, level, int(bool(base_level)),
                                     first_index, additional, seed, C.byref(out)))
    return LevelStats(level, out.sum, out.sum_sq, out.samples, out.cost, out.jumps)


def _result(r, levels) -> MlmcResult:
    lv = [LevelStats(int(x["level"]), float(x["sum"]), float(x["sum_sq"]), int(x["samples"]), int(x["cost"]))
          for x in levels]
    return MlmcResult(float(r["estimate"]), float(r["statistical_error"]), float(r["bias_estimate"]),
                      float(r["quadrature_bound"]), lv,
                      int(r["l0"]), int(r["L"]), int(r["total_cost"]), bool(r["converged"]), int(r["total_jumps"]),
                      int(r["total_samples"]), float(r["projected_cost"]), bool(r["over_budget"]))


def mlmc_driver(problem: MlmcProblem, options: MlmcOptions = MlmcOptions(), max_levels: int = 64) -> MlmcResult:
    """mlmc.hpp:94, mlmc.cpp:170-260."""
    res = np.zeros(1, _RESULT_DT)
    lv = np.zeros(max_levels, LEVEL_RECORD_DT)
    o = options._c()
    mode = _mode(problem)
    if mode == SampleMode.forward:
        _check(L.lib.expmc_mlmc_driver_forward(problem.ctx.handle, problem.beta, C.byref(o), 1, None, _ptr(res),
                                               _ptr(lv), max_levels))
    elif mode == SampleMode.fem:
        rows = np.array([problem.entry], np.int64)
        seeds = np.array([options.seed], np.uint64)
        _check(L.lib.expmc_mlmc_driver_fem(problem.ctx.handle, problem.beta, C.byref(o), 1, _ptr(rows), _ptr(seeds),
                                           _ptr(res), _ptr(lv), max_levels))
    else:
        _check(L.lib.expmc_mlmc_driver(problem.ctx.handle, problem.entry, problem.beta, C.byref(o),
                                       C.cast(_ptr(res), C.POINTER(L.ResultC)), _ptr(lv), max_levels))
    return _result(res[0], lv[: int(res[0]["nlevels"])])


def mlmc_driver_forward(ctx: Context, beta: float, seeds, options: MlmcOptions = MlmcOptions(),
                        max_levels: int = 64, want_levels: bool = True):
    """Forward-mode estimator of sum(e^{beta A} u) on Context(A^T, u): one reference
    mlmc_driver decision sequence per seed, all runs batched on the GPU.  Returns (results
    structured array, levels [nruns, max_levels] or None)."""
    seeds = np.ascontiguousarray(seeds, np.uint64).ravel()
    res = np.zeros(seeds.size, _RESULT_DT)
    lv = np.zeros((seeds.size, max_levels), LEVEL_RECORD_DT) if want_levels else None
    o = options._c()
    _check(L.lib.expmc_mlmc_driver_forward(ctx.handle, beta, C.byref(o), seeds.size, _ptr(seeds), _ptr(res),
                                           _ptr(lv), max_levels))
    return res, lv


def mlmc_driver_rows(ctx: Context, beta: float, rows, row_seeds, options: MlmcOptions = MlmcOptions(),
                     max_levels: int = 64, want_levels: bool = True):
    """All-components estimator: one reference mlmc_driver decision sequence per row, all rows
    batched on the GPU.  Returns (results structured array, levels [nrows, max_levels] or None)."""
    rows = np.ascontiguousarray(rows, np.int64)
    seeds = np.ascontiguousarray(row_seeds, np.uint64)
    if seeds.shape != rows.shape:
        raise InvalidArgument("one seed per row required")
    res = np.zeros(rows.size, _RESULT_DT)
    lv = np.zeros((rows.size, max_levels), LEVEL_RECORD_DT) if want_levels else None
    o = options._c()
    _check(L.lib.expmc_mlmc_driver_rows(ctx.handle, beta, C.byref(o), rows.size, _ptr(rows), _ptr(seeds), _ptr(res),
                                        _ptr(lv), max_levels))
    return res, lv


def mlmc_driver_fem(ctx: Context, beta: float, rows, row_seeds, options: MlmcOptions = MlmcOptions(),
                    max_levels: int = 64, want_levels: bool = True):
    """fem-mode driver for many entries (lane 2): one reference decision sequence per row,
    batched; results carry quadrature_bound."""
    rows = np.ascontiguousarray(rows, np.int64)
    seeds = np.ascontiguousarray(row_seeds, np.uint64)
    if seeds.shape != rows.shape:
        raise InvalidArgument("one seed per row required")
    res = np.zeros(rows.size, _RESULT_DT)
    lv = np.zeros((rows.size, max_levels), LEVEL_RECORD_DT) if want_levels else None
    o = options._c()
    _check(L.lib.expmc_mlmc_driver_fem(ctx.handle, beta, C.byref(o), rows.size, _ptr(rows), _ptr(seeds), _ptr(res),
                                       _ptr(lv), max_levels))
    return res, lv


@dataclass
class FemSystem:
    """fem.hpp FemSystem: lumped-mass system M u' = -K u + F, u(0) = u0."""

    mass_diag: np.ndarray
    stiffness: SparseMatrix
    load: np.ndarray
    u0: np.ndarray

    @property
    def n(self) -> int:
        return self.stiffness.n


def load_fem_system(mass_path, stiffness_path, load_path, u0_path) -> FemSystem:
    """fem.cpp:12-37: mass (Matrix Market, lumped: diagonal and positive), stiffness, load and
    initial vectors, with the reference's checks and messages."""
    mass = read_matrix_market(mass_path)
    stiffness = read_matrix_market(stiffness_path)
    load = read_vector(load_path)
    u0 = read_vector(u0_path)
    n = stiffness.n
    if mass.n != n or load.size != n or u0.size != n:
        raise InvalidArgument("FEM system dimensions disagree")
    md = np.zeros(n)
    for i in range(n):
        for k in range(int(mass.row_ptr[i]), int(mass.row_ptr[i + 1])):
            if mass.col[k] != i:
                raise InvalidArgument("mass matrix is not lumped (off-diagonal entry)")
            md[i] = mass.val[k]
        if not md[i] > 0.0:
            raise InvalidArgument("lumped mass must be positive on the diagonal")
    return FemSystem(md, stiffness, load, u0)


def fem_context(sys: FemSystem, device: int = 0) -> Context:
    """The chain of -M^{-1}K with u0 and the load M^{-1}F bound (fem.cpp:58-64)."""
    md = np.asarray(sys.mass_diag, np.float64)
    return Context(sys.stiffness, sys.u0, device, row_scale=-1.0 / md,
                   load=np.asarray(sys.load, np.float64) / md)


def solve_convdiff_point(sys: FemSystem, node: int, t: float, options: MlmcOptions = MlmcOptions(),
                         device: int = 0) -> MlmcResult:
    """fem.cpp:51-73: u(node, t) of the inhomogeneous system by fem-mode MLMC."""
    if not t > 0.0:
        raise InvalidArgument("time must be positive")
    if node < 0 or node >= sys.n:
        raise OutOfRange("node index outside system")
    with fem_context(sys, device) as ctx:
        return mlmc_driver(MlmcProblem(ctx, node, t, SampleMode.fem), options)


# --------------------------------------------------------------------------------- classical MC
@dataclass
class McResult:
    """mc.hpp McResult (+ jumps)."""

    estimate: float = 0.0
    std_error: float = 0.0
    samples: int = 0
    dt: float = 0.0
    steps: int = 0
    wall_cost: int = 0
    jumps: int = 0


def _mc(r) -> McResult:
    return McResult(r.estimate, r.std_error, r.samples, r.dt, r.steps, r.wall_cost, r.jumps)


def mc_single_entry(ctx: Context, entry: int, beta: float, dt: float, samples: int, seed: int,
                    threads: int = 0) -> McResult:
    """mc.cpp:42-58: plain MC of (e^{beta A} u)_entry at one step size, Welford statistics."""
    r = L.McResultC()
    _check(L.lib.expmc_mc_single_entry(ctx.handle, entry, beta, dt, samples, seed, C.byref(r)))
    return _mc(r)


def mc_forward_scalar(ctx_t: Context, beta: float, dt: float, samples: int, seed: int,
                      threads: int = 0) -> McResult:
    """mc.cpp:60-76: plain MC of sum(e^{beta A} u) on Context(A^T, u)."""
    r = L.McResultC()
    _check(L.lib.expmc_mc_forward_scalar(ctx_t.handle, beta, dt, samples, seed, C.byref(r)))
    return _mc(r)


def mc_auto(ctx: Context, entry: int, beta: float, epsilon: float, seed: int, threads: int = 0) -> McResult:
    """mc.cpp:78-113: pilot-sized plain MC to tolerance epsilon."""
    r = L.McResultC()
    _check(L.lib.expmc_mc_auto(ctx.handle, entry, beta, epsilon, seed, C.byref(r)))
    return _mc(r)


def mc_batch(ctx: Context, entries, seeds, samples, beta: float, dt: float, lane: int = L.LANE_ENTRY) -> list:
    """Many classical-MC runs (one per entry / seed) in one GPU pass."""
    e, sd, m = np.broadcast_arrays(np.asarray(entries, np.int64), np.asarray(seeds, np.uint64),
                                   np.asarray(samples, np.uint64))
    k = e.size
    req = (L.McReqC * k)()
    for i in range(k):
        req[i] = L.McReqC(int(e.ravel()[i]), int(sd.ravel()[i]), int(m.ravel()[i]), beta, dt)
    out = (L.McResultC * k)()
    _check(L.lib.expmc_mc_batch(ctx.handle, lane, k, C.cast(req, C.c_void_p), C.cast(out, C.c_void_p)))
    return [_mc(out[i]) for i in range(k)]


def spectral_scale(ctx: Context) -> float:
    """chain.cpp:98-102: 1 / d_max of the context's decomposition."""
    if not ctx.d_max > 0.0:
        raise DomainError("d_max <= 0: no spectral scale, supply beta explicitly")
    return 1.0 / ctx.d_max


def total_communicability(a: SparseMatrix, beta: float | None = None, options: MlmcOptions = MlmcOptions(),
                          device: int = 0, sampler: str = "reference") -> MlmcResult:
    """communicability.cpp:10-21: 1^T e^{beta A} 1 by forward-mode MLMC on A^T (one scalar
    MLMC problem); beta defaults to spectral_scale of A^T's decomposition."""
    with Context(a.transposed(), np.ones(a.n), device, sampler) as ctx:
        b = spectral_scale(ctx) if beta is None else beta
        return mlmc_driver(MlmcProblem(ctx, 0, b, SampleMode.forward), options)


def node_communicability(a: SparseMatrix, node: int, beta: float | None = None,
                         options: MlmcOptions = MlmcOptions(), device: int = 0,
                         sampler: str = "reference") -> MlmcResult:
    """communicability.cpp:23-35: (e^{beta A} 1)_node, entry mode."""
    with Context(a, np.ones(a.n), device, sampler) as ctx:
        b = spectral_scale(ctx) if beta is None else beta
        return mlmc_driver(MlmcProblem(ctx, node, b, SampleMode.entry), options)


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for Context.shard_samples (create on one rank, broadcast to the rest)."""
    buf = (C.c_uint8 * 128)()
    _check(L.lib.expmc_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def bench_gather(device: int, nbytes: int, loads_per_thread: int = 64, reps: int = 5) -> float:
    """Random 32-B sector gather throughput (GB/s) over an nbytes buffer: the roofline
    denominator of the sampler's table reads."""
    out = C.c_double()
    _check(L.lib.expmc_bench_gather(device, nbytes, loads_per_thread, reps, C.byref(out)))
    return out.value


def initial_level(beta: float, d_max: float) -> int:
    out = C.c_int32()
    _check(L.lib.expmc_initial_level(beta, d_max, C.byref(out)))
    return out.value


def optimal_allocation(variances, unit_costs, epsilon: float) -> np.ndarray:
    v = np.ascontiguousarray(variances, np.float64)
    c = np.ascontiguousarray(unit_costs, np.float64)
    if v.shape != c.shape:
        raise InvalidArgument("variance and cost arrays differ in length")
    out = np.empty(v.size, np.uint64)
    _check(L.lib.expmc_optimal_allocation(v.size, _ptr(v), _ptr(c), epsilon, _ptr(out)))
    return out


def bias_estimate(coupled_means) -> float:
    m = np.ascontiguousarray(coupled_means, np.float64)
    out = C.c_double()
    _check(L.lib.expmc_bias_estimate(m.size, _ptr(m), C.byref(out)))
    return out.value
