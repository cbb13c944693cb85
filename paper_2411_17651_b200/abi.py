"""ctypes mirror of include/psg.h and loaders for the in-tree libpsg.so.

The engine library is loaded from the package directory only; when it is
missing the import fails loudly (there is no CPU fallback on the product
path).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libpsg.so")

PSG_OK, PSG_ERR_USAGE, PSG_ERR_INFEASIBLE, PSG_ERR_DATA, PSG_ERR_CUDA = 0, 2, 3, 4, 5
OP = {"attention": 0, "gemm": 1, "moe_gemm": 2}
COLL = {"allreduce": 0, "allgather": 1, "reduce_scatter": 2, "all_to_all": 3, "p2p": 4}
DTYPE = {"fp16": 0, "fp8": 1, "int4": 2}

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class PlanSetC(C.Structure):
    _fields_ = [("n_plans", C.c_int32)] + [
        (n, t) for n, t in [
            ("model_dp", _i32p), ("num_stages", _i32p), ("stage_devices", _i32p),
            ("stage_repetitions", _i32p), ("compute_dtype", _i32p), ("enc_rank", _i32p),
            ("kv_bytes_per_token", _f64p), ("kv_budget_per_replica", _f64p),
            ("p2p_payload_per_token", _f64p), ("shape_hidden", _f64p),
            ("shape_head_dim", _f64p), ("shape_kv_elems", _f64p),
            ("cell_begin", _i32p), ("cell_op", _i32p), ("cell_tasks", _f64p),
            ("cell_width", _f64p), ("cell_token_scale", _f64p),
            ("coll_begin", _i32p), ("coll_kind", _i32p), ("coll_devices", _i32p),
            ("coll_nodes", _i32p), ("coll_groups", _i32p), ("coll_ppt", _f64p),
            ("coll_share", _f64p), ("p2p_begin", _i32p), ("p2p_nodes", _i32p)]]


class ClusterC(C.Structure):
    _fields_ = [("total_devices", C.c_int32), ("peak_mem_bandwidth", C.c_double),
                ("peak_flops", C.c_double * 3), ("max_frequency_ghz", C.c_double)]


class StoreC(C.Structure):
    _fields_ = [("n_compute", C.c_int32), ("c_op", _i32p), ("c_dtype", _i32p),
                ("c_freq_micro", _i64p), ("c_n_ctx", _i32p), ("c_n_tasks", _i32p),
                ("c_n_width", _i32p), ("c_knot_begin", _i64p), ("c_value_begin", _i64p),
                ("c_knots", _f64p), ("c_seconds", _f64p), ("c_joules", _f64p),
                ("n_curves", C.c_int32), ("k_kind", _i32p), ("k_devices", _i32p),
                ("k_nodes", _i32p), ("k_n", _i32p), ("k_begin", _i64p),
                ("k_payload", _f64p), ("k_seconds", _f64p), ("k_joules", _f64p)]


class TraceC(C.Structure):
    _fields_ = [("n", C.c_int64), ("id", _i64p), ("context_len", _i64p),
                ("gen_len", _i64p), ("arrival", _f64p)]


class ConfigC(C.Structure):
    _fields_ = [("objective", C.c_int32), ("batch_mode", C.c_int32),
                ("chunk_size", C.c_int64), ("max_batch_size", C.c_int64),
                ("ttft_anchor", C.c_int32), ("n_freqs", C.c_int32),
                ("freqs", _f64p), ("detail", C.c_int32), ("rank", C.c_int32),
                ("n_entry_subset", C.c_int32), ("entry_subset", _i32p),
                ("entry_max_batch_size", _i64p), ("emit_iterations", C.c_int32),
                ("ttft_slo", C.c_double), ("slo_quantile", C.c_double)]


ENTRY_DTYPE = np.dtype([
    ("entry_index", "<i8"), ("plan_index", "<i8"), ("freq_ghz", "<f8"),
    ("e2e_latency", "<f8"), ("total_energy", "<f8"), ("p95_latency", "<f8"),
    ("mean_ttft", "<f8"), ("mean_tpot", "<f8"), ("mfu", "<f8"), ("mbu", "<f8"),
    ("num_completed", "<i8"), ("num_rejected", "<i8"), ("num_iterations", "<i8"),
    ("max_batch_observed", "<i8"), ("p50_ttft", "<f8"), ("p99_ttft", "<f8"),
    ("p50_tpot", "<f8"), ("p99_tpot", "<f8"), ("slo_ttft", "<f8"), ("slo_met", "<i8"),
    ("per_request_offset", "<i8"),
    ("rejected_offset", "<i8")])
METRICS_DTYPE = np.dtype([("id", "<i8"), ("ttft", "<f8"), ("tpot", "<f8"),
                          ("e2e", "<f8"), ("gen_len", "<i8")])
ITERATION_DTYPE = np.dtype([("clock_start", "<f8"), ("duration", "<f8"), ("energy", "<f8"),
                            ("batch_size", "<i8")])
RANK_KEY_DTYPE = np.dtype([("num_rejected", "<i8"), ("objective_metric", "<f8"),
                           ("other_metric", "<f8"), ("enc_rank", "<i4"), ("slo_miss", "<i4"),
                           ("freq_ghz", "<f8"), ("entry_index", "<i8")])


def empty_rank_keys():
    """A zero-length psg_rank_key array (an empty shard's contribution)."""
    return np.zeros(0, dtype=RANK_KEY_DTYPE)


class ResultC(C.Structure):
    _fields_ = [("n_entries", C.c_int64), ("entries", C.c_void_p),
                ("n_per_request", C.c_int64), ("per_request", C.c_void_p),
                ("n_rejected", C.c_int64), ("rejected_ids", C.c_void_p),
                ("n_compute", C.c_int32), ("compute_clamp", C.c_void_p),
                ("n_curves", C.c_int32), ("curve_clamp", C.c_void_p),
                ("gpu_launches", C.c_int64), ("total_iterations", C.c_int64),
                ("ms_total", C.c_double), ("ms_h2d", C.c_double), ("ms_sim", C.c_double),
                ("ms_reduce", C.c_double), ("ms_d2h", C.c_double), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("sum_batch", C.c_int64), ("admissions", C.c_int64),
                ("finishes", C.c_int64), ("n_iterations", C.c_int64),
                ("iterations", C.c_void_p), ("n_stages", C.c_int32),
                ("stage_seconds", C.c_void_p), ("stage_joules", C.c_void_p)]


EXPORTED_SYMBOLS = ("psg_version", "psg_context_create", "psg_context_destroy",
                    "psg_last_error", "psg_search", "psg_search_many", "psg_rank_keys",
                    "psg_result_free")

_lib = None


def load_library(path: str = None) -> C.CDLL:
    """Loads the in-tree engine library; raises if it has not been built.
    PSG_LIBRARY may name another in-tree build (dev: libpsg_prof.so)."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        path = os.path.join(PKG_DIR, os.environ.get("PSG_LIBRARY", "libpsg.so"))
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA engine with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    lib.psg_version.restype = C.c_char_p
    lib.psg_context_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.psg_context_destroy.argtypes = [C.c_void_p]
    lib.psg_last_error.restype = C.c_char_p
    lib.psg_last_error.argtypes = [C.c_void_p]
    lib.psg_search.argtypes = [C.c_void_p, C.POINTER(PlanSetC), C.POINTER(ClusterC),
                               C.POINTER(StoreC), C.POINTER(TraceC), C.POINTER(ConfigC),
                               C.POINTER(C.POINTER(ResultC))]
    lib.psg_rank_keys.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    lib.psg_result_free.argtypes = [C.POINTER(ResultC)]
    _lib = lib
    return lib


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))
