"""ctypes binding of include/liftcut_b200.h (libliftcut_b200.so).

The shared library is the product: it must be built (``python -m
paper_2509_18612_b200.build``) and it is loaded from the package directory, so a
missing build fails loudly instead of falling back to anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LCB_LIB_PATH") or os.path.join(HERE, "libliftcut_b200.so")

P = C.c_void_p
i64, u64, u32, i32, f64 = C.c_int64, C.c_uint64, C.c_uint32, C.c_int32, C.c_double

LCB_OK, LCB_VALIDATION, LCB_SHAPE, LCB_NUMERIC, LCB_CUDA, LCB_ERROR, LCB_PARSE = range(7)
LCB_FP64, LCB_FP32 = 0, 1


class Config(C.Structure):
    """lcb_config — SolverConfig + AscentParams + InitConfig + SearchConfig."""

    _fields_ = [
        ("algorithm", i32), ("lift_dim", i32), ("batch_size", i64), ("num_batches", i64),
        ("alpha", f64), ("iterations", i64), ("momentum", f64), ("early_exit", i32),
        ("has_lifted_ascent", i32), ("l_alpha", f64), ("l_iterations", i64),
        ("l_momentum", f64), ("l_early_exit", i32), ("init_method", i32), ("beta", f64),
        ("eta", f64), ("init_scale", f64), ("init_seed", u64), ("resample_idi", i32),
        ("scale_noise", i32), ("time_budget_s", f64), ("has_search", i32),
        ("population_size", i32), ("t_lower", i64), ("t_upper", i64), ("e_lower", f64),
        ("e_upper", f64), ("rounds", i32), ("search_refresh", i32),
        ("deco_alternations", i32), ("deco_carry", i32),
    ]


class BatchTrace(C.Structure):
    _fields_ = [("serial", i64), ("kind", i32), ("pad_", i32), ("alpha", f64),
                ("iterations", i64), ("batch_best", i64), ("best_so_far", i64)]


class PhaseTrace(C.Structure):
    _fields_ = [("phase", i32), ("kind", i32), ("best_after", i64)]


class SearchTrace(C.Structure):
    _fields_ = [("round", i32), ("pad_", i32), ("exponent", f64), ("iterations", i64),
                ("fitness", f64)]


class Outcome(C.Structure):
    _fields_ = [("cut_value", i64), ("batch_index", i64), ("member_index", i64),
                ("batches_run", i64), ("n_batch_trace", i64), ("n_phase_trace", i64),
                ("n_search_trace", i64), ("init_s", f64), ("ascent_s", f64),
                ("rounding_s", f64), ("search_s", f64), ("wall_s", f64)]


TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, i64, i64, f64)


class RunOpts(C.Structure):
    _fields_ = [("precision", i32), ("host_init", i32), ("batched_search", i32), ("pad_", i32),
                ("comm", P), ("step_ms", P), ("step_launches", P), ("node_updates", P),
                ("step_bytes", P), ("solve_ms", P), ("kernel_stats", P), ("trace_fn", TRACE_FN),
                ("trace_ctx", P)]


SIGNATURES = {
    "lcb_last_error": (C.c_char_p, []),
    "lcb_abi_version": (C.c_int, []),
    "lcb_device_count": (C.c_int, [P]),
    "lcb_set_option": (C.c_int, [C.c_char_p, i64]),
    "lcb_get_option": (C.c_int, [C.c_char_p, P]),
    "lcb_graph_create": (C.c_int, [u32, P, P, C.c_int, C.POINTER(P)]),
    "lcb_graph_destroy": (None, [P]),
    "lcb_graph_info": (C.c_int, [P, P, P, P]),
    "lcb_laplacian_apply": (C.c_int, [P, P, P, i64, i32]),
    "lcb_ascend": (C.c_int, [P, P, i64, i32, i64, f64, i64, f64, i32, i32, P, P, P]),
    "lcb_ascend_rows": (C.c_int, [P, u32, i64, i64, P, P, P, i32, i64, f64, i64, f64, i32, i32, C.c_int, P, P]),
    "lcb_cut_values": (C.c_int, [P, P, i64, P]),
    "lcb_round_cut_batch": (C.c_int, [P, P, i32, i64, i32, P, P, P, P]),
    "lcb_round": (C.c_int, [C.c_int, P, i64, i32, i64, i32, P]),
    "lcb_brute_force_maxcut": (C.c_int, [P, i32, P, P, P]),
    "lcb_graph_from_edges": (C.c_int, [u32, P, P, i64, C.c_int, C.POINTER(P)]),
    "lcb_graph_parse": (C.c_int, [C.c_char_p, i64, C.c_int, C.POINTER(P), C.POINTER(C.c_int)]),
    "lcb_graph_csr": (C.c_int, [P, P, P]),
    "lcb_dui_init": (C.c_int, [P, u64, P]),
    "lcb_idi_init": (C.c_int, [P, f64, u64, P]),
    "lcb_lifted_init_mean": (C.c_int, [P, i32, f64, i32, u64, P]),
    "lcb_gaussian_batch": (C.c_int, [C.c_int, P, i64, i32, f64, i64, u64, P]),
    "lcb_gaussian_batch_exact": (C.c_int, [P, i64, i32, f64, i64, u64, P]),
    "lcb_solve": (C.c_int, [P, P, u64, i32, P, P, P, P, i64, P, i64, P, i64]),
    "lcb_comm_unique_id": (C.c_int, [P]),
    "lcb_comm_create": (C.c_int, [P, i32, i32, C.c_int, C.POINTER(P)]),
    "lcb_comm_destroy": (None, [P]),
    "lcb_solve_runs": (C.c_int, [P, P, P, i64, i32, P, P, P, P, P]),
    "lcb_debug_resident_layout": (C.c_int, [P, P, P, P, P, P]),
    "lcb_loopback_create": (C.c_int, [i32, C.POINTER(P)]),
    "lcb_loopback_destroy": (None, [P]),
    "lcb_comm_create_loopback": (C.c_int, [P, i32, C.c_int, C.POINTER(P)]),
    "lcb_counters": (None, [P, P, P]),
    "lcb_release_workspaces": (None, []),
    "lcb_pack_key": (u64, [i64, i64]),
    "lcb_unpack_key": (None, [u64, P, P]),
}

_lib = None


def lib():
    """Load libliftcut_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2509_18612_b200.build`")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        if L.lcb_abi_version() != 3:
            raise RuntimeError("libliftcut_b200.so ABI mismatch")
        _lib = L
    return _lib


def last_error() -> str:
    return lib().lcb_last_error().decode(errors="replace")
