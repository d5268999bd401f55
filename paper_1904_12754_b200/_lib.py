"""ctypes binding of the C-ABI in ``include/expmc_b200.h`` (libexpmc_b200.so, in-tree).

There is no CPU fallback: if the library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EXPMC_LIB") or os.path.join(_HERE, "_lib", "libexpmc_b200.so")

_I32, _I64, _U32, _U64, _D = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double

EXPMC_OK, EXPMC_EINVAL, EXPMC_ERANGE, EXPMC_EDOMAIN, EXPMC_ECUDA, EXPMC_ENOTIMPL, EXPMC_EIO, EXPMC_EOVERFLOW = (
    0, 1, 2, 3, 4, 5, 6, 7)
EXPMC_EINTERNAL = 9
LANE_ENTRY, LANE_FORWARD, LANE_FEM = 0, 1, 2
SAMPLER_REFERENCE, SAMPLER_EVENT = 0, 1


class Csr(C.Structure):
    _fields_ = [("n", _I64), ("nnz", _I64), ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p)]


class CtxInfo(C.Structure):
    _fields_ = [("n", _I64), ("n_edges", _I64), ("d_max", _D), ("d_bar", _D), ("device", _I32), ("num_sms", _I32),
                ("table_bytes", _U64)]


class LevelReq(C.Structure):
    _fields_ = [("entry", _I64), ("seed", _U64), ("first_index", _U64), ("count", _U64), ("level", _I32),
                ("base_level", _I32)]


class LevelStatsC(C.Structure):
    _fields_ = [("sum", _D), ("sum_sq", _D), ("samples", _U64), ("cost", _U64), ("jumps", _U64), ("integ_sum", _D)]


class OptionsC(C.Structure):
    _fields_ = [("epsilon", _D), ("seed", _U64), ("threads", _I32), ("l0_override", _I32), ("warmup", _U64),
                ("max_levels_above_l0", _I32), ("max_iterations", _I32), ("max_cost", _D)]


class ResultC(C.Structure):
    _fields_ = [("estimate", _D), ("statistical_error", _D), ("bias_estimate", _D), ("l0", _I32), ("L", _I32),
                ("total_cost", _U64), ("converged", _I32), ("nlevels", _I32), ("total_jumps", _U64),
                ("total_samples", _U64), ("projected_cost", _D), ("over_budget", _I32), ("pad", _I32),
                ("quadrature_bound", _D)]


class SampleRecordC(C.Structure):
    _fields_ = [("eta_fine", _D), ("eta_coarse", _D), ("value", _D), ("integ_fine", _D), ("integ_coarse", _D),
                ("cost", _U64), ("jumps", _U64), ("end_state", _I64)]


class McResultC(C.Structure):
    _fields_ = [("estimate", _D), ("std_error", _D), ("samples", _U64), ("dt", _D), ("steps", _I64),
                ("wall_cost", _U64), ("jumps", _U64)]


class McReqC(C.Structure):
    _fields_ = [("entry", _I64), ("seed", _U64), ("samples", _U64), ("beta", _D), ("dt", _D)]


class LevelRecordC(C.Structure):
    _fields_ = [("level", _I32), ("pad", _I32), ("sum", _D), ("sum_sq", _D), ("samples", _U64), ("cost", _U64)]


class CountersC(C.Structure):
    _fields_ = [("kernel_launches", _U64), ("sampler_launches", _U64), ("sampler_ms", _D), ("h2d_bytes", _U64),
                ("d2h_bytes", _U64), ("samples", _U64), ("jumps", _U64), ("fine_steps", _U64), ("rounds", _U64),
                ("nccl_bytes", _U64)]


# (name, restype, argtypes) -- every symbol declared in include/expmc_b200.h
_P = C.c_void_p
SYMBOLS = [
    ("expmc_last_error", C.c_char_p, []),
    ("expmc_version", C.c_char_p, []),
    ("expmc_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("expmc_ctx_create", C.c_int, [C.POINTER(Csr), _P, C.c_int, C.POINTER(_P)]),
    ("expmc_ctx_destroy", None, [_P]),
    ("expmc_ctx_get_info", C.c_int, [_P, C.POINTER(CtxInfo)]),
    ("expmc_ctx_create_scaled", C.c_int, [C.POINTER(Csr), _P, _P, C.c_int, C.POINTER(_P)]),
    ("expmc_ctx_set_vector", C.c_int, [_P, _P]),
    ("expmc_ctx_set_load", C.c_int, [_P, _P]),
    ("expmc_ctx_export_tables", C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    ("expmc_ctx_export_alias", C.c_int, [_P, _P, _P, _P, C.POINTER(_U64)]),
    ("expmc_ctx_get_counters", C.c_int, [_P, C.POINTER(CountersC)]),
    ("expmc_ctx_reset_counters", C.c_int, [_P]),
    ("expmc_ctx_get_stream", C.c_int, [_P, C.POINTER(_P)]),
    ("expmc_ctx_set_sampler", C.c_int, [_P, _I32]),
    ("expmc_ctx_get_sampler", C.c_int, [_P, C.POINTER(_I32)]),
    ("expmc_ctx_set_sampler_flags", C.c_int, [_P, C.c_uint32]),
    ("expmc_bench_gather", C.c_int, [C.c_int, _U64, _I32, _I32, C.POINTER(_D)]),
    ("expmc_selftest_exp", C.c_int, [C.c_int, _I64, _P, _P]),
    ("expmc_nccl_unique_id", C.c_int, [_P]),
    ("expmc_ctx_shard_samples", C.c_int, [_P, _P, _I32, _I32]),
    ("expmc_ctx_set_shard", C.c_int, [_P, _I32, _I32]),
    ("expmc_ctx_last_partials", C.c_int, [_P, C.POINTER(_I64), _P, _P, _P, _P]),
    ("expmc_run_level", C.c_int, [_P, _I64, _D, _I32, _I32, _U64, _U64, _U64, C.POINTER(LevelStatsC)]),
    ("expmc_run_level_forward", C.c_int, [_P, _D, _I32, _I32, _U64, _U64, _U64, C.POINTER(LevelStatsC)]),
    ("expmc_run_level_batch", C.c_int, [_P, _D, _U32, _I64, _P, _P]),
    ("expmc_sample_debug", C.c_int, [_P, _D, _U32, _I64, _P, _P, _P, _P, _P, _P]),
    ("expmc_sample_debug_ex", C.c_int, [_P, _D, _U32, _I64, _P, _P]),
    ("expmc_run_level_fem", C.c_int, [_P, _I64, _D, _I32, _I32, _U64, _U64, _U64, C.POINTER(LevelStatsC)]),
    ("expmc_mlmc_driver_fem", C.c_int, [_P, _D, C.POINTER(OptionsC), _I64, _P, _P, _P, _P, _I32]),
    ("expmc_mlmc_driver", C.c_int, [_P, _I64, _D, C.POINTER(OptionsC), C.POINTER(ResultC), _P, _I32]),
    ("expmc_mlmc_driver_rows", C.c_int, [_P, _D, C.POINTER(OptionsC), _I64, _P, _P, _P, _P, _I32]),
    ("expmc_mlmc_driver_forward", C.c_int, [_P, _D, C.POINTER(OptionsC), _I64, _P, _P, _P, _I32]),
    ("expmc_gen_ba", C.c_int, [_I64, _I64, _U64, C.POINTER(_P)]),
    ("expmc_gen_rmat", C.c_int, [_I32, _I64, _D, _D, _D, _U64, C.POINTER(_P)]),
    ("expmc_gen_convdiff3d", C.c_int, [_I64, _D, _I32, C.POINTER(_P)]),
    ("expmc_mc_single_entry", C.c_int, [_P, _I64, _D, _D, _U64, _U64, C.POINTER(McResultC)]),
    ("expmc_mc_forward_scalar", C.c_int, [_P, _D, _D, _U64, _U64, C.POINTER(McResultC)]),
    ("expmc_mc_batch", C.c_int, [_P, _U32, _I64, _P, _P]),
    ("expmc_mc_auto", C.c_int, [_P, _I64, _D, _D, _U64, C.POINTER(McResultC)]),
    ("expmc_read_matrix_market", C.c_int, [C.c_char_p, C.POINTER(_P)]),
    ("expmc_read_vector", C.c_int, [C.c_char_p, _I64, _P, C.POINTER(_I64)]),
    ("expmc_csr_from_triplets", C.c_int, [_I64, _I64, _P, _P, _P, C.POINTER(_P)]),
    ("expmc_matrix_info", C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64)]),
    ("expmc_matrix_copy", C.c_int, [_P, _P, _P, _P]),
    ("expmc_matrix_destroy", None, [_P]),
    ("expmc_power_iteration", C.c_int, [C.POINTER(Csr), _I32, C.POINTER(_D)]),
    ("expmc_initial_level", C.c_int, [_D, _D, C.POINTER(_I32)]),
    ("expmc_optimal_allocation", C.c_int, [_I64, _P, _P, _D, _P]),
    ("expmc_bias_estimate", C.c_int, [_I64, _P, C.POINTER(_D)]),
]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: the CUDA library is the only implementation (no CPU fallback). "
            "Build it with `python -m paper_1904_12754_b200.build` or __graft_entry__.build().")
    lib = C.CDLL(path)
    for name, res, args in SYMBOLS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = load()
