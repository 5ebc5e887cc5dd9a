"""B200-native decode hot path of arXiv 2503.05248 (dynamic batching).

The product is ``libdbk.so`` (C-ABI, ``include/dbk.h``): paged decode attention
+ fused batch statistics (sm_100a CUDA), the page allocator, Algorithm 1 /
Algorithm 2 batch-size rules and the continuous-batching engine (host C++),
and the NCCL statistics exchange.  This package is a thin binding:

* ``paper_2503_05248_b200._lib`` -- every ``dbk_*`` entry point under the same name;
* ``KVPool``, ``Scheduler``, ``Engine`` -- argument marshalling for numpy / torch.

Importing the package fails loudly when the library has not been built.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (DbkError, dbk_batch, dbk_engine_buffers, dbk_engine_config,  # noqa: F401
                   dbk_model_config, dbk_pool_config, dbk_prefill_batch, dbk_sched_config, dbk_sched_state,
                   dbk_stats, dbk_step_record)

_lib.lib()  # load now: no silent fallback


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _ptr(t):
    """Device/host pointer of a torch tensor (or an int, or None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(s):
    if s is None:
        return None
    return s.cuda_stream if hasattr(s, "cuda_stream") else int(s)


class KVPool:
    """dbk_pool: paged KV cache over caller-owned device memory (a torch tensor)."""

    def __init__(self, layers, q_heads, kv_heads, head_dim, cap_pages, max_requests,
                 max_pages_per_req, kv_dtype="f16", page_size=16, device=0, kv_mem=None, kv_head_offset=0):
        import torch
        self.cfg = dbk_pool_config(layers, q_heads, kv_heads, head_dim, page_size,
                                   0 if kv_dtype == "f16" else 1, cap_pages, max_requests,
                                   max_pages_per_req, device, int(kv_head_offset))
        self.nbytes = _lib.dbk_kv_pool_bytes(C.byref(self.cfg))
        if self.nbytes == 0:
            raise DbkError(1, "dbk_kv_pool_bytes", "invalid pool config")
        self.kv = kv_mem if kv_mem is not None else torch.empty(
            self.nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        h = C.c_void_p()
        _lib.dbk_kv_pool_create(C.byref(self.cfg), self.kv.data_ptr(), self.kv.numel(), C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and _lib is not None:  # _lib is None during interpreter teardown
            _lib.dbk_kv_pool_destroy(self.h)
            self.h = None

    __del__ = close

    def request_begin(self, req_id, l_in, l_out):
        _lib.dbk_request_begin(self.h, int(req_id), int(l_in), int(l_out))

    def append_tokens(self, req_ids, n_tok, k=None, v=None, seed=0, stream=None):
        ids, pids = _i64(req_ids)
        nt, pnt = _i32(n_tok)
        _lib.dbk_append_tokens(self.h, len(ids), pids, pnt, _ptr(k), _ptr(v), int(seed), _stream(stream))

    def release(self, req_ids):
        ids, pids = _i64(req_ids)
        _lib.dbk_release(self.h, len(ids), pids)

    def reserve_tokens(self, req_ids, n_tok, stream=None):
        ids, pids = _i64(req_ids)
        nt, pnt = _i32(n_tok)
        _lib.dbk_reserve_tokens(self.h, len(ids), pids, pnt, _stream(stream))

    def swap_space_attach(self, host_mem):
        """host_mem: a pinned torch tensor (kept alive by the pool object); returns swap pages."""
        self._swap_mem = host_mem
        n = C.c_int64()
        nbytes = host_mem.numel() * host_mem.element_size() if host_mem is not None else 0
        _lib.dbk_swap_space_attach(self.h, _ptr(host_mem), nbytes, C.byref(n))
        return n.value

    def swap_out(self, req_ids, stream=None):
        ids, pids = _i64(req_ids)
        _lib.dbk_swap_out(self.h, len(ids), pids, _stream(stream))

    def swap_in(self, req_ids, stream=None):
        ids, pids = _i64(req_ids)
        _lib.dbk_swap_in(self.h, len(ids), pids, _stream(stream))

    def swap_usage(self):
        u, f, b = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.dbk_swap_usage(self.h, C.byref(u), C.byref(f), C.byref(b))
        return u.value, f.value, b.value

    def request_info(self, req_id):
        ctx, npg, slot = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.dbk_request_info(self.h, int(req_id), C.byref(ctx), C.byref(npg), C.byref(slot), None, 0)
        pages = np.zeros(max(npg.value, 1), np.int32)
        _lib.dbk_request_info(self.h, int(req_id), None, None, None,
                              pages.ctypes.data_as(C.POINTER(C.c_int32)), npg.value)
        return ctx.value, slot.value, pages[:npg.value].tolist()

    def usage(self):
        u, f = C.c_int64(), C.c_int64()
        _lib.dbk_pool_usage(self.h, C.byref(u), C.byref(f))
        return u.value, f.value

    def info(self):
        o = _lib.dbk_pool_info()
        _lib.dbk_pool_get_info(self.h, C.byref(o))
        return {f: getattr(o, f) for f, _ in o._fields_}

    def block_table(self, stream=None):
        out = np.zeros((self.cfg.max_requests, self.cfg.max_pages_per_req), np.int32)
        _lib.dbk_block_table_d2h(self.h, out.ctypes.data_as(C.POINTER(C.c_int32)), _stream(stream))
        return out

    def decode_step(self, req_ids, layer, q, out, out_dtype=2, fuse_stats=False, stream=None, chain=False):
        ids, pids = _i64(req_ids)
        b = dbk_batch(len(ids), int(layer), 1 if fuse_stats else 0, 1 if chain else 0, pids)
        _lib.dbk_decode_step(self.h, C.byref(b), _ptr(q), _ptr(out), int(out_dtype), _stream(stream))

    def decode_step_layers(self, req_ids, layer0, n_layers, q, q_layer_stride, out, out_layer_stride, out_dtype=2,
                           fuse_stats=False, stream=None, chain=False):
        """Layers [layer0, layer0 + n_layers) in multi-layer launches; returns the launch count."""
        ids, pids = _i64(req_ids)
        b = dbk_batch(len(ids), int(layer0), 1 if fuse_stats else 0, 1 if chain else 0, pids)
        nl = C.c_int32()
        _lib.dbk_decode_step_layers(self.h, C.byref(b), int(n_layers), _ptr(q), int(q_layer_stride), _ptr(out),
                                    int(out_layer_stride), int(out_dtype), _stream(stream), C.byref(nl))
        return nl.value

    def prefill_step(self, req_ids, q_start, q_len, layer, q, out, out_dtype=2, stream=None):
        ids, pids = _i64(req_ids)
        s0, ps0 = _i32(q_start)
        ln, pln = _i32(q_len)
        b = dbk_prefill_batch(len(ids), int(layer), pids, ps0, pln)
        _lib.dbk_prefill_step(self.h, C.byref(b), _ptr(q), _ptr(out), int(out_dtype), _stream(stream))

    def batch_stats(self, stream=None):
        st = dbk_stats()
        _lib.dbk_batch_stats(self.h, C.byref(st), _stream(stream))
        return st.as_dict()


class Gemm:
    """dbk_gemm: the model projections' tensor-core GEMM, y (=|+=) x w^T (torch fp16 operands)."""

    MODES = {"f16": 0, "f32": 1, "acc32": 2, "silu": 4}

    def __init__(self, device=0, cta_group=2):
        h = C.c_void_p()
        _lib.dbk_gemm_create(device, cta_group, C.byref(h))
        self.h = h
        self.cta_group = cta_group

    def __call__(self, x, w, y, mode="f16", stream=None):
        M, K = x.shape
        N = w.shape[0]
        _lib.dbk_gemm_run(self.h, M, N, K, _ptr(x), x.stride(0), _ptr(w), _ptr(y), y.stride(0),
                          self.MODES[mode], _stream(stream))
        return y

    def last_plan(self):
        """Tiling of the last launch: bn, bn_b, units_a, units, split (dbk_gemm_last_plan)."""
        v = [C.c_int32() for _ in range(5)]
        _lib.dbk_gemm_last_plan(self.h, *[C.byref(x) for x in v])
        return dict(zip(("bn", "bn_b", "units_a", "units", "split"), (x.value for x in v)))

    def close(self):
        if getattr(self, "h", None):
            _lib.dbk_gemm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


def synth_fill(seed, kind, req, pos, layer, n_heads, d, out, scale_log2=0, dtype=2, stream=None):
    r, pr = _i64(req)
    p, pp = _i32(pos)
    _lib.dbk_synth_fill(int(seed), int(kind), len(r), pr, pp, int(layer), int(n_heads), int(d),
                        int(scale_log2), int(dtype), _ptr(out), _stream(stream))


class Scheduler:
    """dbk_sched: Alg. 1 / Alg. 2 / min / static (host C++)."""

    def __init__(self, policy=1, b_static=256, b_min=1, b_max=512, b0=1, alpha=8, delta=2,
                 w_len=256, w_sla=20, refresh_steps=100, page_size=16, eps_m=0.02, d_sla_ms=50.0,
                 eps_d_ms=2.0, bytes_per_token=1, prior=(1, 1, 1, 1, 1)):
        self.cfg = dbk_sched_config(policy, b_static, b_min, b_max, b0, alpha, delta, w_len, w_sla,
                                    refresh_steps, page_size, 0, eps_m, d_sla_ms, eps_d_ms,
                                    bytes_per_token, *[int(x) for x in prior])
        h = C.c_void_p()
        _lib.dbk_sched_create(C.byref(self.cfg), C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and _lib is not None:  # _lib is None during interpreter teardown
            _lib.dbk_sched_destroy(self.h)
            self.h = None

    __del__ = close

    def choose(self, stats: dict, mem_cap_bytes, sla_ms=0.0, n_prefill_waiting=0):
        st = dbk_stats(*[int(stats.get(f, 0)) for f in _lib.STATS_FIELDS])
        b, why = C.c_int32(), C.c_int32()
        _lib.dbk_choose_batch_size(self.h, C.byref(st), int(mem_cap_bytes), float(sla_ms),
                                   int(n_prefill_waiting), C.byref(b), C.byref(why))
        return b.value, why.value

    def state(self):
        s = dbk_sched_state()
        _lib.dbk_sched_get_state(self.h, C.byref(s))
        return {f: getattr(s, f) for f, _ in s._fields_}


class Model:
    """dbk_model: full decode step with synthetic fp16 weights over a KVPool (NEXT row 3)."""

    def __init__(self, pool: KVPool, hidden, ffn, vocab, max_pos=4096, rms_eps=1e-5, rope_theta=10000.0,
                 weight_seed=0, token_seed=None, tp_size=1, tp_rank=0):
        import torch
        self.pool = pool
        self.cfg = dbk_model_config(int(hidden), int(ffn), int(vocab), int(max_pos), float(rms_eps),
                                    float(rope_theta), int(weight_seed),
                                    int(weight_seed if token_seed is None else token_seed), int(tp_size),
                                    int(tp_rank))
        nbytes = _lib.dbk_model_weight_bytes(C.byref(pool.cfg), C.byref(self.cfg))
        if nbytes == 0:
            raise DbkError(1, "dbk_model_weight_bytes", "invalid model config")
        self.weights = torch.empty(nbytes, dtype=torch.uint8, device=pool.kv.device)
        h = C.c_void_p()
        _lib.dbk_model_create(pool.h, C.byref(self.cfg), self.weights.data_ptr(), nbytes, C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and _lib is not None:  # _lib is None during interpreter teardown
            _lib.dbk_model_destroy(self.h)
            self.h = None

    __del__ = close

    def step(self, req_ids, logits=None, fuse_stats=True, stream=None):
        ids, pids = _i64(req_ids)
        _lib.dbk_model_step(self.h, len(ids), pids, 1 if fuse_stats else 0, _ptr(logits), _stream(stream))

    def step_pd(self, req_ids, chunk_ids, q_start, q_len, logits=None, fuse_stats=True, stream=None,
                tokens=None, sampled=None):
        ids, pids = _i64(req_ids)
        cid, pcid = _i64(chunk_ids)
        s0, ps0 = _i32(q_start)
        ln, pln = _i32(q_len)
        b = dbk_prefill_batch(len(cid), 0, pcid, ps0, pln)
        _lib.dbk_model_step_pd(self.h, len(ids), pids, C.byref(b), 1 if fuse_stats else 0, _ptr(logits),
                               _ptr(tokens), _ptr(sampled), _stream(stream))

    def attach_tp(self, tp):
        _lib.dbk_model_attach_tp(self.h, tp.h)
        self._tp = tp

    def timing(self, reset=False):
        a, t, n = C.c_double(), C.c_double(), C.c_int64()
        _lib.dbk_model_timing(self.h, C.byref(a), C.byref(t), C.byref(n), 1 if reset else 0)
        return a.value, t.value, n.value


class Engine:
    """dbk_engine over a KVPool and a Scheduler; trace arrays are copied."""

    def __init__(self, pool: KVPool, sched: Scheduler, arrival_ns, l_in, l_out, mem_cap_bytes,
                 sla_ms=0.0, seed=0, out_dtype=2, time_attention=False, rank=0, world=1,
                 q_scale_log2=0, req_ids=None, pd_fusion=False, preempt_mode=0, pd_token_budget=0,
                 per_layer_launches=False):
        self.pool, self.sched = pool, sched
        self._arr, pa = _i64(arrival_ns)
        self._li, pli = _i32(l_in)
        self._lo, plo = _i32(l_out)
        pids = None
        if req_ids is not None:
            self._ids, pids = _i64(req_ids)
        self.cfg = dbk_engine_config(len(self._arr), q_scale_log2, pa, pli, plo, pids,
                                     int(mem_cap_bytes), float(sla_ms), int(seed), int(out_dtype),
                                     1 if time_attention else 0, rank, world, 1 if pd_fusion else 0,
                                     int(preempt_mode), int(pd_token_budget), 1 if per_layer_launches else 0)
        h = C.c_void_p()
        _lib.dbk_engine_create(pool.h, sched.h, C.byref(self.cfg), C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and _lib is not None:  # _lib is None during interpreter teardown
            _lib.dbk_engine_destroy(self.h)
            self.h = None

    __del__ = close

    def attach_comm(self, comm, mode):
        """Exchange every step's record through a libdbk communicator (Comm); mode MODE_DP / MODE_TP."""
        self.comm = comm
        _lib.dbk_engine_attach_comm(self.h, comm.h if comm is not None else None, int(mode))

    def last_exchange(self, reset=False, cap=64):
        """The last step's exchange: per-rank records (rank order), host us of that exchange,
        total us and count since the last reset."""
        arr = (dbk_stats * cap)()
        n, us, tot, cnt = C.c_int32(), C.c_double(), C.c_double(), C.c_int64()
        _lib.dbk_engine_last_exchange(self.h, arr, cap, C.byref(n), C.byref(us), C.byref(tot), C.byref(cnt),
                                      1 if reset else 0)
        return dict(records=[arr[r].as_dict() for r in range(min(n.value, cap))], us=us.value,
                    us_total=tot.value, count=cnt.value)

    def attach_mbox(self, mbox, mode):
        """Exchange every step's record through a Mailbox (the step's last kernel); mode MODE_DP / MODE_TP."""
        self.mbox = mbox
        _lib.dbk_engine_attach_mbox(self.h, mbox.h if mbox is not None else None, int(mode))

    def attach_model(self, model):
        _lib.dbk_engine_attach_model(self.h, model.h if model is not None else None)
        self.model = model

    @staticmethod
    def buffers(q_dev, out_dev, kv_dev=None, host_q=None, host_k=None, host_v=None, host_out=None,
                host_tokens=None):
        return dbk_engine_buffers(_ptr(q_dev), _ptr(out_dev), _ptr(kv_dev), _ptr(host_q),
                                  _ptr(host_k), _ptr(host_v), _ptr(host_out), _ptr(host_tokens))

    def step(self, bufs, stream=None):
        rec = dbk_step_record()
        _lib.dbk_engine_step(self.h, C.byref(bufs), _stream(stream), C.byref(rec))
        return rec.as_dict()

    def step_launch(self, bufs, stream=None):
        st = dbk_stats()
        _lib.dbk_engine_step_launch(self.h, C.byref(bufs), _stream(stream), C.byref(st))
        return st.as_dict()

    def step_finish(self, global_stats: dict):
        st = dbk_stats(*[int(global_stats.get(f, 0)) for f in _lib.STATS_FIELDS])
        rec = dbk_step_record()
        _lib.dbk_engine_step_finish(self.h, C.byref(st), C.byref(rec))
        return rec.as_dict()

    def done(self):
        d = C.c_int32()
        _lib.dbk_engine_done(self.h, C.byref(d))
        return bool(d.value)

    def last_batch(self, cap=1 << 16):
        n = C.c_int32()
        ids = np.zeros(cap, np.int64)
        ctx = np.zeros(cap, np.int32)
        _lib.dbk_engine_last_batch(self.h, C.byref(n), ids.ctypes.data_as(C.POINTER(C.c_int64)),
                                   ctx.ctypes.data_as(C.POINTER(C.c_int32)), cap)
        return ids[:n.value].copy(), ctx[:n.value].copy()

    def attn_timing(self, reset=False):
        ms, la, by = C.c_double(), C.c_int64(), C.c_int64()
        _lib.dbk_engine_attn_timing(self.h, C.byref(ms), C.byref(la), C.byref(by), 1 if reset else 0)
        return ms.value, la.value, by.value

    def request_times(self):
        """(first_admit_ns, finish_ns) per trace index, -1 = not yet / another rank."""
        n = len(self._arr)
        a = np.full(n, -1, np.int64)
        f = np.full(n, -1, np.int64)
        _lib.dbk_engine_request_times(self.h, n, a.ctypes.data_as(C.POINTER(C.c_int64)),
                                      f.ctypes.data_as(C.POINTER(C.c_int64)))
        return a, f


class Comm:
    """dbk_comm: libdbk's NCCL communicator for the 128-B statistics exchange.  The
    ncclUniqueId comes from rank 0 (dbk_comm_unique_id) and is broadcast over the caller's
    torch.distributed process group (`dist`)."""

    def __init__(self, dist, world, rank, device):
        buf = (C.c_char * 128)()
        if rank == 0:
            _lib.dbk_comm_unique_id(buf)
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        idbuf = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _lib.dbk_comm_create(int(world), int(rank), idbuf, int(device), C.byref(h))
        self.h = h

    def info(self):
        """(nranks, rank) as NCCL reports them."""
        n, r = C.c_int32(), C.c_int32()
        _lib.dbk_comm_info(self.h, C.byref(n), C.byref(r))
        return n.value, r.value

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dbk_comm_destroy(self.h)
            self.h = None

    __del__ = close


class Mailbox:
    """dbk_mbox: the statistics exchange over peer memory (CUDA IPC mailboxes, one exchange
    kernel per step).  The 64-byte IPC handles are gathered over the caller's
    torch.distributed process group (`dist`)."""

    def __init__(self, dist, world, rank, device):
        h = C.c_void_p()
        buf = (C.c_char * 64)()
        _lib.dbk_mbox_create(int(world), int(rank), int(device), buf, C.byref(h))
        self.h = h
        handles = [None] * world
        dist.all_gather_object(handles, bytes(buf.raw))
        allb = (C.c_char * (64 * world)).from_buffer_copy(b"".join(handles))
        _lib.dbk_mbox_open(self.h, allb)
        self.world = world

    def exchange(self, local: dict, mode=0, stream=None):
        """(records of every rank, reduced global record) of one exchange."""
        st = dbk_stats(*[int(local.get(f, 0)) for f in _lib.STATS_FIELDS])
        arr = (dbk_stats * self.world)()
        g = dbk_stats()
        _lib.dbk_mbox_exchange(self.h, C.byref(st), arr, C.byref(g), int(mode), _stream(stream))
        return [arr[r].as_dict() for r in range(self.world)], g.as_dict()

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dbk_mbox_destroy(self.h)
            self.h = None

    __del__ = close


class Tp:
    """dbk_tp: the tensor-parallel residual stream (IPC-mapped buffers of every rank, barrier).
    The 64-byte IPC handles are gathered over the caller's torch.distributed group (`dist`)."""

    def __init__(self, dist, world, rank, device, rows, hidden):
        h = C.c_void_p()
        buf = (C.c_char * 64)()
        _lib.dbk_tp_create(int(world), int(rank), int(device), int(rows), int(hidden), buf, C.byref(h))
        self.h = h
        handles = [None] * world
        dist.all_gather_object(handles, bytes(buf.raw))
        allb = (C.c_char * (64 * world)).from_buffer_copy(b"".join(handles))
        _lib.dbk_tp_open(self.h, allb)

    def barrier(self, stream=None):
        _lib.dbk_tp_barrier(self.h, _stream(stream))

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dbk_tp_destroy(self.h)
            self.h = None

    __del__ = close


def stats_reduce(records, mode=0):
    arr = (dbk_stats * len(records))(*[dbk_stats(*[int(r.get(f, 0)) for f in _lib.STATS_FIELDS])
                                       for r in records])
    out = dbk_stats()
    _lib.dbk_stats_reduce(arr, len(records), int(mode), C.byref(out))
    return out.as_dict()


def theta_q(eps_m):
    x = C.c_int64()
    _lib.dbk_theta_q(float(eps_m), C.byref(x))
    return x.value


def b_quad(n, S, V2, eta, tq):
    x = C.c_int64()
    _lib.dbk_b_quad(int(n), int(S), int(V2), int(eta), int(tq), C.byref(x))
    return x.value
