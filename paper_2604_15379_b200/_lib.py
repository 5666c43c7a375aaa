"""ctypes binding of libmk.so (the C ABI in include/mk.h).

This is the whole host->device boundary: plain structs, raw device pointers,
int status codes.  Importing never silently degrades: if the shared library
is missing the import of :mod:`.runtime` raises, and there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MK_LIB_PATH") or os.path.join(_HERE, "libmk.so")

MK_OK, MK_ERR_CONFIG, MK_ERR_DEADLOCK, MK_ERR_CUDA = 0, 2, 3, 4
LEVEL_WAVEFRONT, LEVEL_CU, LEVEL_CHIPLET = 0, 1, 2
(OP_NOP, OP_RMSNORM, OP_GEMM, OP_ATTN_PARTIAL, OP_ATTN_REDUCE, OP_SILU, OP_ARGMAX,
 OP_TP_ALLREDUCE, OP_TP_ARGMAX) = range(9)
EPI_NONE, EPI_RESIDUAL, EPI_SILU, EPI_LOGITS, EPI_PARTIAL = range(5)
BODY_GEMV, BODY_UMMA = 0, 1
TRAV_N_MAJOR, TRAV_M_MAJOR = 0, 1
DIST_M_TILE, DIST_M_SPLIT = 0, 1
SCHED_PER_DIE, SCHED_FLAT = 0, 1
MAX_SMS, MAX_DIES, MAX_TP = 256, 8, 8

P = C.c_void_p
I32 = C.c_int32
F32 = C.c_float


class Topology(C.Structure):
    _fields_ = [("num_sms", I32), ("num_dies", I32),
                ("sms_per_die", I32 * MAX_DIES), ("die_of_sm", I32 * MAX_SMS),
                ("separation", F32), ("near_cycles", F32), ("far_cycles", F32)]


class Task(C.Structure):
    _fields_ = [("op", I32), ("level", I32), ("die", I32), ("wait0", I32),
                ("wait1", I32), ("signal", I32), ("n_items", I32),
                ("n_units", I32), ("sub_ctr", I32), ("param_off", I32),
                ("layer", I32), ("graph_index", I32), ("pad", I32 * 4)]


class Unit(C.Structure):
    _fields_ = [("task", I32), ("item_begin", I32), ("item_end", I32), ("pad", I32)]


class GemmParams(C.Structure):
    _fields_ = [("w", P), ("x", P), ("y", P), ("res", P), ("amax_val", P),
                ("amax_idx", P), ("norm_gamma", P), ("M", I32), ("K", I32), ("N", I32),
                ("T_M", I32), ("T_N", I32), ("T_K", I32), ("ldx", I32),
                ("ldy", I32), ("ldres", I32), ("y_col0", I32),
                ("epilogue", I32), ("traversal", I32), ("distribution", I32),
                ("xcd", I32), ("tile_m", I32), ("tile_n", I32),
                ("amax_base", I32), ("amax_stride", I32), ("stage_x", I32),
                ("norm_eps", F32), ("body", I32), ("y_cols", I32),
                ("ksplit", I32), ("tile_ctr0", I32), ("piece_floats", I32),
                ("ss_nparts", I32), ("kpart", P), ("ss_out", P), ("ss_in", P)]


class NormParams(C.Structure):
    _fields_ = [("x", P), ("gamma", P), ("y", P), ("embed", P), ("tokens", P),
                ("x_store", P), ("M", I32), ("d", I32), ("eps", F32), ("fused", I32),
                ("ss_out", P)]


class AttnParams(C.Structure):
    _fields_ = [("qkv", P), ("q_gamma", P), ("k_gamma", P), ("k_cache", P),
                ("v_cache", P), ("rope_cos", P), ("rope_sin", P),
                ("positions", P), ("partial", P), ("out", P), ("M", I32),
                ("ldqkv", I32), ("q_heads", I32), ("kv_heads", I32),
                ("head_dim", I32), ("group", I32), ("kv_head", I32),
                ("split", I32), ("n_splits", I32), ("t_max", I32),
                ("eps", F32), ("scale", F32), ("sub_splits", I32), ("mma", I32),
                ("fuse_reduce", I32), ("red_ctr0", I32), ("page_table", P),
                ("max_pages", I32), ("prefill", I32)]


class SiluParams(C.Structure):
    _fields_ = [("gu", P), ("y", P), ("F", I32), ("row0", I32), ("rows", I32),
                ("col0", I32), ("cols", I32), ("pad", I32)]


class ArgmaxParams(C.Structure):
    _fields_ = [("amax_val", P), ("amax_idx", P), ("out_tokens", P),
                ("next_tokens", P), ("positions", P), ("M", I32), ("n_slots", I32)]


class TPParams(C.Structure):
    _fields_ = [("recv_off", C.c_int64), ("flag_off", C.c_int64), ("gather_off", C.c_int64),
                ("res", P), ("y", P), ("amax_val", P), ("amax_idx", P),
                ("out_tokens", P), ("next_tokens", P), ("positions", P),
                ("M", I32), ("d", I32), ("n_slots", I32), ("vocab0", I32)]


class GraphDesc(C.Structure):
    _fields_ = [("n_tasks", I32), ("n_events", I32), ("n_units", I32),
                ("n_sub_ctrs", I32), ("n_schedulers", I32), ("sched_mode", I32),
                ("workers_per_sched", I32), ("param_bytes", I32),
                ("tasks", P), ("event_required", P), ("units", P),
                ("sched_begin", P), ("params", P), ("positions", P), ("n_rows", I32),
                ("pad", I32), ("tokens", P), ("out_tokens", P)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "dispatches", "mailbox_writes", "global_atomics", "local_atomics",
        "fences", "fanout_atomics", "polls", "tiles", "executions", "steps",
        "wait_ring_empty", "wait_mma_full", "wait_mma_x", "wait_mma_tmem",
        "wait_epi_done", "mma_chunks")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class LogRec(C.Structure):
    _fields_ = [("kind", I32), ("task", I32), ("item_begin", I32),
                ("worker", I32), ("smid", I32), ("die", I32),
                ("t_start", C.c_uint64), ("t_end", C.c_uint64)]


EXPORTS = ("mk_probe", "mk_probe_raw", "mk_create", "mk_step", "mk_step_tokens", "mk_sync",
           "mk_counters_get",
           "mk_counters_reset", "mk_log_enable", "mk_log_read",
           "mk_tile_log_enable", "mk_tile_log_read", "mk_trace_enable", "mk_trace_read",
           "mk_set_watchdog", "mk_set_prefetch", "mk_set_debug",
           "mk_tp_init", "mk_tp_alloc", "mk_tp_free", "mk_ipc_export", "mk_ipc_import",
           "mk_ipc_close", "mk_set_grid",
           "mk_destroy", "mk_last_error", "mk_version")

_lib = None


def load() -> C.CDLL:
    """Load libmk.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` "
                          "(build) first; there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    lib.mk_probe.argtypes = [C.c_int, C.POINTER(Topology)]
    lib.mk_probe_raw.argtypes = [C.c_int, C.POINTER(C.c_uint32), C.POINTER(I32)]
    lib.mk_create.argtypes = [C.c_int, C.POINTER(GraphDesc), C.POINTER(Topology),
                              C.POINTER(C.c_void_p)]
    lib.mk_step.argtypes = [C.c_void_p, C.c_void_p]
    lib.mk_step_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.mk_set_prefetch.argtypes = [C.c_void_p, C.c_int]
    lib.mk_sync.argtypes = [C.c_void_p]
    lib.mk_counters_get.argtypes = [C.c_void_p, C.POINTER(Counters)]
    lib.mk_counters_reset.argtypes = [C.c_void_p]
    lib.mk_log_enable.argtypes = [C.c_void_p, C.c_int64]
    lib.mk_log_read.argtypes = [C.c_void_p, C.POINTER(LogRec), C.c_int64]
    lib.mk_log_read.restype = C.c_int64
    lib.mk_tile_log_enable.argtypes = [C.c_void_p, C.c_int64]
    lib.mk_tile_log_read.argtypes = [C.c_void_p, C.POINTER(I32), C.c_int64]
    lib.mk_tile_log_read.restype = C.c_int64
    lib.mk_trace_enable.argtypes = [C.c_void_p, C.c_int32]
    lib.mk_trace_read.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]
    lib.mk_trace_read.restype = C.c_int64
    lib.mk_set_watchdog.argtypes = [C.c_void_p, C.c_double]
    lib.mk_set_debug.argtypes = [C.c_void_p, C.c_int]
    lib.mk_tp_init.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.mk_tp_alloc.argtypes = [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]
    lib.mk_tp_free.argtypes = [C.c_void_p]
    lib.mk_ipc_export.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
    lib.mk_ipc_import.argtypes = [C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_void_p)]
    lib.mk_ipc_close.argtypes = [C.c_void_p]
    lib.mk_set_grid.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.mk_destroy.argtypes = [C.c_void_p]
    lib.mk_last_error.restype = C.c_char_p
    _lib = lib
    return lib


class MkError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[mk status {code}] {msg}")
        self.code = code


def check(rc: int):
    if rc != MK_OK:
        raise MkError(rc, load().mk_last_error().decode())
