"""ctypes binding of libdbk.so (include/dbk.h).  Argument marshalling only.

Every ``dbk_*`` function of the header is exposed under the same name; a
non-zero status raises ``DbkError`` carrying ``dbk_last_error()``.  There is
no fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DBK_LIB: an alternative build of the same library (e.g. libdbk_asan.so, the sanitizer build)
LIB_PATH = os.environ.get("DBK_LIB") or os.path.join(_HERE, "libdbk.so")

STATUS = {0: "DBK_OK", 1: "DBK_EINVAL", 2: "DBK_ECAP", 3: "DBK_ENOENT", 4: "DBK_EINFEASIBLE",
          5: "DBK_ECUDA", 6: "DBK_ENCCL", 7: "DBK_EFATAL"}
DBK_OK, DBK_EINVAL, DBK_ECAP, DBK_ENOENT, DBK_EINFEASIBLE, DBK_ECUDA, DBK_ENCCL, DBK_EFATAL = range(8)
POLICY_STATIC, POLICY_MEMORY, POLICY_SLA, POLICY_COMBINED = range(4)
R_STATIC, R_MEMORY, R_SLA, R_MIN, R_CARRY = range(5)
MODE_DP, MODE_TP = 0, 1


class DbkError(RuntimeError):
    def __init__(self, status, fn, msg):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class dbk_pool_config(C.Structure):
    _fields_ = [("layers", C.c_int32), ("q_heads", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("page_size", C.c_int32), ("kv_dtype", C.c_int32),
                ("cap_pages", C.c_int64), ("max_requests", C.c_int32),
                ("max_pages_per_req", C.c_int32), ("device", C.c_int32),
                ("kv_head_offset", C.c_int32)]


class dbk_pool_info(C.Structure):
    _fields_ = [("decode_path", C.c_int32), ("ctas_per_sm", C.c_int32), ("chunk_pages", C.c_int32),
                ("work_items", C.c_int32), ("launches", C.c_int64), ("last_decode_bytes", C.c_int64),
                ("tma_rank", C.c_int32), ("_reserved", C.c_int32)]


class dbk_batch(C.Structure):
    _fields_ = [("n", C.c_int32), ("layer", C.c_int32), ("fuse_stats", C.c_int32),
                ("chain", C.c_int32), ("req_ids", C.POINTER(C.c_int64))]


class dbk_prefill_batch(C.Structure):
    _fields_ = [("n", C.c_int32), ("layer", C.c_int32), ("req_ids", C.POINTER(C.c_int64)),
                ("q_start", C.POINTER(C.c_int32)), ("q_len", C.POINTER(C.c_int32))]


STATS_FIELDS = ("n_active", "sum_ctx", "sum_ctx_sq", "max_ctx", "sum_pages", "cap_pages",
                "free_pages", "over_cap", "table_mismatch", "n_finished", "fin_sum_lin",
                "fin_sum_lin_sq", "fin_sum_lout", "fin_sum_lout_sq", "step_ns", "n_waiting")


class dbk_stats(C.Structure):
    _fields_ = [(f, C.c_int64) for f in STATS_FIELDS]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f in STATS_FIELDS}


class dbk_sched_config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("b_static", C.c_int32), ("b_min", C.c_int32),
                ("b_max", C.c_int32), ("b0", C.c_int32), ("alpha", C.c_int32), ("delta", C.c_int32),
                ("w_len", C.c_int32), ("w_sla", C.c_int32), ("refresh_steps", C.c_int32),
                ("page_size", C.c_int32), ("_reserved", C.c_int32), ("eps_m", C.c_double),
                ("d_sla_ms", C.c_double), ("eps_d_ms", C.c_double), ("bytes_per_token", C.c_int64),
                ("prior_n", C.c_int64), ("prior_sum_lin", C.c_int64), ("prior_sum_lin_sq", C.c_int64),
                ("prior_sum_lout", C.c_int64), ("prior_sum_lout_sq", C.c_int64)]


class dbk_sched_state(C.Structure):
    _fields_ = [("t", C.c_int64), ("eta", C.c_int64), ("L0", C.c_int64), ("b_quad", C.c_int64),
                ("theta_q", C.c_int64), ("win_n", C.c_int64), ("win_S", C.c_int64),
                ("win_V2", C.c_int64), ("b", C.c_int32), ("b_mem", C.c_int32), ("b_sla", C.c_int32),
                ("b_low", C.c_int32), ("b_high", C.c_int32), ("sla_count", C.c_int32)]


class dbk_engine_config(C.Structure):
    _fields_ = [("n_requests", C.c_int32), ("q_scale_log2", C.c_int32),
                ("arrival_ns", C.POINTER(C.c_int64)), ("l_in", C.POINTER(C.c_int32)),
                ("l_out", C.POINTER(C.c_int32)), ("req_ids", C.POINTER(C.c_int64)),
                ("mem_cap_bytes", C.c_int64), ("sla_ms", C.c_double), ("synth_seed", C.c_uint64),
                ("out_dtype", C.c_int32), ("time_attention", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("pd_fusion", C.c_int32), ("preempt_mode", C.c_int32),
                ("pd_token_budget", C.c_int32), ("per_layer_launches", C.c_int32)]


class dbk_engine_buffers(C.Structure):
    _fields_ = [("q_dev", C.c_void_p), ("out_dev", C.c_void_p), ("kv_dev", C.c_void_p),
                ("host_q", C.c_void_p), ("host_k", C.c_void_p), ("host_v", C.c_void_p),
                ("host_out", C.c_void_p), ("host_tokens", C.c_void_p)]


class dbk_model_config(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("rms_eps", C.c_double), ("rope_theta", C.c_double), ("weight_seed", C.c_uint64),
                ("token_seed", C.c_uint64), ("tp_size", C.c_int32), ("tp_rank", C.c_int32)]


class dbk_step_record(C.Structure):
    _fields_ = [("t", C.c_int64), ("clock_ns", C.c_int64), ("step_ns", C.c_int64),
                ("sum_ctx", C.c_int64), ("used_pages", C.c_int64), ("table_hash", C.c_int64),
                ("b_t", C.c_int32), ("b_next", C.c_int32), ("n_admitted", C.c_int32),
                ("n_preempted", C.c_int32), ("n_decode", C.c_int32), ("n_finished", C.c_int32),
                ("rationale", C.c_int32), ("n_waiting", C.c_int32), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("launches", C.c_int32), ("n_prefill", C.c_int32),
                ("n_swap_out", C.c_int32), ("n_swap_in", C.c_int32), ("swap_bytes", C.c_int64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_ if f != "_reserved"}


P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
PI32, PI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)

# name -> argtypes (restype dbk_status unless listed in _RESTYPE)
SIGNATURES = {
    "dbk_last_error": [],
    "dbk_version": [],
    "dbk_kv_pool_bytes": [C.POINTER(dbk_pool_config)],
    "dbk_kv_pool_create": [C.POINTER(dbk_pool_config), P, C.c_size_t, C.POINTER(P)],
    "dbk_kv_pool_destroy": [P],
    "dbk_request_begin": [P, I64, I32, I32],
    "dbk_append_tokens": [P, I32, PI64, PI32, P, P, U64, P],
    "dbk_release": [P, I32, PI64],
    "dbk_reserve_tokens": [P, I32, PI64, PI32, P],
    "dbk_model_weight_bytes": [C.POINTER(dbk_pool_config), C.POINTER(dbk_model_config)],
    "dbk_model_create": [P, C.POINTER(dbk_model_config), P, C.c_size_t, C.POINTER(P)],
    "dbk_model_destroy": [P],
    "dbk_model_step": [P, I32, PI64, I32, P, P],
    "dbk_model_step_pd": [P, I32, PI64, C.POINTER(dbk_prefill_batch), I32, P, P, P, P],
    "dbk_model_timing": [P, C.POINTER(C.c_double), C.POINTER(C.c_double), PI64, I32],
    "dbk_engine_attach_model": [P, P],
    "dbk_tp_create": [I32, I32, I32, I64, I32, P, C.POINTER(P)],
    "dbk_tp_open": [P, P],
    "dbk_tp_barrier": [P, P],
    "dbk_tp_destroy": [P],
    "dbk_model_attach_tp": [P, P],
    "dbk_gemm_create": [I32, I32, C.POINTER(P)],
    "dbk_gemm_run": [P, I32, I32, I32, P, I64, P, P, I64, I32, P],
    "dbk_gemm_trace": [P, P, I32],
    "dbk_gemm_force_tile": [P, I32],
    "dbk_gemm_last_plan": [P, PI32, PI32, PI32, PI32, PI32],
    "dbk_gemm_destroy": [P],
    "dbk_model_buffers": [P, C.POINTER(C.c_void_p)],
    "dbk_swap_space_attach": [P, P, C.c_size_t, PI64],
    "dbk_swap_out": [P, I32, PI64, P],
    "dbk_swap_in": [P, I32, PI64, P],
    "dbk_swap_usage": [P, PI64, PI64, PI64],
    "dbk_request_info": [P, I64, PI32, PI32, PI32, PI32, I32],
    "dbk_pool_usage": [P, PI64, PI64],
    "dbk_block_table_d2h": [P, PI32, P],
    "dbk_pool_get_info": [P, C.POINTER(dbk_pool_info)],
    "dbk_decode_step": [P, C.POINTER(dbk_batch), P, P, I32, P],
    "dbk_batch_stats": [P, C.POINTER(dbk_stats), P],
    "dbk_prefill_step": [P, C.POINTER(dbk_prefill_batch), P, P, I32, P],
    "dbk_synth_fill": [U64, I32, I32, PI64, PI32, I32, I32, I32, I32, I32, P, P],
    "dbk_probe_read_bandwidth": [P, C.c_size_t, I32, P, C.POINTER(C.c_double)],
    "dbk_sched_create": [C.POINTER(dbk_sched_config), C.POINTER(P)],
    "dbk_sched_destroy": [P],
    "dbk_choose_batch_size": [P, C.POINTER(dbk_stats), I64, D, I32, PI32, PI32],
    "dbk_sched_get_state": [P, C.POINTER(dbk_sched_state)],
    "dbk_theta_q": [D, PI64],
    "dbk_b_quad": [I64, I64, I64, I64, I64, PI64],
    "dbk_engine_create": [P, P, C.POINTER(dbk_engine_config), C.POINTER(P)],
    "dbk_engine_destroy": [P],
    "dbk_engine_step": [P, C.POINTER(dbk_engine_buffers), P, C.POINTER(dbk_step_record)],
    "dbk_engine_step_launch": [P, C.POINTER(dbk_engine_buffers), P, C.POINTER(dbk_stats)],
    "dbk_engine_step_finish": [P, C.POINTER(dbk_stats), C.POINTER(dbk_step_record)],
    "dbk_engine_done": [P, PI32],
    "dbk_engine_last_batch": [P, PI32, PI64, PI32, I32],
    "dbk_engine_attn_timing": [P, C.POINTER(C.c_double), PI64, PI64, I32],
    "dbk_engine_request_times": [P, I32, PI64, PI64],
    "dbk_comm_unique_id": [P],
    "dbk_comm_create": [I32, I32, P, I32, C.POINTER(P)],
    "dbk_comm_destroy": [P],
    "dbk_stats_allgather": [P, C.POINTER(dbk_stats), C.POINTER(dbk_stats), C.POINTER(dbk_stats), I32, P],
    "dbk_stats_reduce": [C.POINTER(dbk_stats), I32, I32, C.POINTER(dbk_stats)],
    "dbk_engine_attach_comm": [P, P, I32],
    "dbk_comm_info": [P, PI32, PI32],
    "dbk_pool_trace_d2h": [P, P, I64, PI64, I32],
    "dbk_decode_step_layers": [P, C.POINTER(dbk_batch), I32, P, I64, P, I64, I32, P, PI32],
    "dbk_mbox_create": [I32, I32, I32, P, C.POINTER(P)],
    "dbk_mbox_open": [P, P],
    "dbk_mbox_destroy": [P],
    "dbk_mbox_exchange": [P, C.POINTER(dbk_stats), C.POINTER(dbk_stats), C.POINTER(dbk_stats), I32, P],
    "dbk_engine_attach_mbox": [P, P, I32],
    "dbk_engine_last_exchange": [P, C.POINTER(dbk_stats), I32, PI32, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), PI64, I32],
}
_RESTYPE = {"dbk_last_error": C.c_char_p, "dbk_version": C.c_char_p, "dbk_kv_pool_bytes": C.c_size_t,
            "dbk_model_weight_bytes": C.c_size_t}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def _check(name, status):
    if status != 0:
        raise DbkError(status, name, lib().dbk_last_error().decode(errors="replace"))


def _wrap(name):
    def call(*args):
        f = getattr(lib(), name)
        r = f(*args)
        if name in _RESTYPE:
            return r
        _check(name, r)
        return r
    call.__name__ = name
    call.__doc__ = f"{name}{tuple(a.__name__ for a in SIGNATURES[name])} -- see include/dbk.h"
    return call


for _n in SIGNATURES:
    globals()[_n] = _wrap(_n)
