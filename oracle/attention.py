"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

ctypes front-end for ``oracle/attention.c`` (O1, paged decode attention in
fp64) plus a helper that lays out synthetic K/V in the oracle's own paged
layout.  The C file is compiled with plain gcc (``build()``); nothing here
touches CUDA.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from synth import hashgen

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attention.c")
_LIB = os.path.join(_HERE, "_oracle_attention.so")
_lib = None

DTYPES = {"f16": 0, "bf16": 1}


def build(force=False) -> str:
    """Compile attention.c with gcc -O2 -fopenmp (no -ffast-math: IEEE semantics).  With
    DBK_ORACLE_SANITIZE=1: a separate ASan + UBSan build (the sanitizer run of SURVEY.md §5)."""
    global _LIB
    san = os.environ.get("DBK_ORACLE_SANITIZE") == "1"
    if san:
        _LIB = os.path.join(_HERE, "_oracle_attention_asan.so")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB, _SRC, "-lm"]
        if san:
            cmd[1:1] = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=undefined"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_half_to_double.argtypes = [ctypes.c_uint16]
        L.oracle_half_to_double.restype = ctypes.c_double
        L.oracle_bf16_to_double.argtypes = [ctypes.c_uint16]
        L.oracle_bf16_to_double.restype = ctypes.c_double
        P = ctypes.c_void_p
        L.oracle_paged_decode_attention.argtypes = [ctypes.c_int] * 5 + [P, P, ctypes.c_int, P, P, P,
                                                                         ctypes.c_int, P, ctypes.c_int]
        L.oracle_paged_decode_attention.restype = ctypes.c_int
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def paged_decode_attention(ctx, block_table, pool_k, pool_v, q, dtype="f16", nthreads=1):
    """O1.  ctx int32 [n]; block_table int32 [n][W]; pool_k/pool_v uint16
    [pages][Hkv][P][d]; q uint16 [n][Hq][d].  Returns float64 [n][Hq][d]."""
    ctx = np.ascontiguousarray(ctx, dtype=np.int32)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    pk = np.ascontiguousarray(pool_k, dtype=np.uint16)
    pv = np.ascontiguousarray(pool_v, dtype=np.uint16)
    qq = np.ascontiguousarray(q, dtype=np.uint16)
    n, Hq, d = qq.shape
    _, Hkv, P, d2 = pk.shape
    if d2 != d or pv.shape != pk.shape or bt.shape[0] != n or ctx.shape[0] != n:
        raise ValueError("shape mismatch")
    out = np.zeros((n, Hq, d), np.float64)
    rc = lib().oracle_paged_decode_attention(n, Hq, Hkv, d, P, _ptr(ctx), _ptr(bt), bt.shape[1],
                                             _ptr(pk), _ptr(pv), _ptr(qq), DTYPES[dtype], _ptr(out),
                                             int(nthreads))
    if rc != 0:
        raise ValueError("oracle_paged_decode_attention: invalid arguments")
    return out


def paged_prefill_attention(q_start, q_len, block_table, pool_k, pool_v, q, dtype="f16", nthreads=1):
    """O1 applied to a prefill chunk (PD fusion; R24): chunk i holds
    query tokens at positions q_start[i] + j, j < q_len[i]; each attends causally to keys
    0..q_start[i]+j of its request -- exactly the decode formula with ctx = position + 1.
    q uint16 [sum q_len][Hq][d] (chunks concatenated); block_table int32 [n][W] (one row per
    chunk).  Returns float64 [sum q_len][Hq][d]."""
    q_start = np.asarray(q_start, np.int64)
    q_len = np.asarray(q_len, np.int64)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    rows_ctx = np.concatenate([s + np.arange(n) + 1 for s, n in zip(q_start, q_len)]).astype(np.int32)
    rows_bt = np.repeat(bt, q_len, axis=0)
    return paged_decode_attention(rows_ctx, rows_bt, pool_k, pool_v, q, dtype, nthreads)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def synth_paged_batch(seed, req_ids, ctx, pages, layer, Hq, Hkv, d, P, dtype,
                      q_scale_log2=0, n_phys=None):
    """Build the oracle-side inputs of one decode launch from the synthetic generator.

    req_ids[i], ctx[i]: the request and its KV length (incl. this step's token);
    pages[i]: list of physical page ids (logical page p -> pages[i][p]), e.g.
    from oracle.allocator.  K/V of token (req, pos) in layer `layer`, head g
    are synth values (kind K / V); q of request i is the synth q at
    pos = ctx_i - 1.  Returns (block_table, pool_k, pool_v, q) as uint16 bits.
    """
    n = len(req_ids)
    width = max([len(p) for p in pages] + [1])
    if n_phys is None:
        n_phys = max([max(p) for p in pages if len(p)] + [-1]) + 1
    bt = np.full((n, width), -1, np.int32)
    pool_k = np.zeros((max(n_phys, 1), Hkv, P, d), np.uint16)
    pool_v = np.zeros_like(pool_k)
    q = np.zeros((n, Hq, d), np.uint16)
    heads = np.arange(Hkv)
    for i, (r, c, pg) in enumerate(zip(req_ids, ctx, pages)):
        if len(pg) < -(-c // P):
            raise ValueError("not enough pages for ctx")
        bt[i, :len(pg)] = pg
        pos = np.arange(c)
        kv = {}
        for kind in (hashgen.KIND_K, hashgen.KIND_V):
            vals = hashgen.gen_values(seed, kind, r, pos[:, None], layer, heads[None, :], d)
            kv[kind] = hashgen.to_bits(vals, dtype)  # [c][Hkv][d]
        for j in range(c):
            pool_k[pg[j // P], :, j % P, :] = kv[hashgen.KIND_K][j]
            pool_v[pg[j // P], :, j % P, :] = kv[hashgen.KIND_V][j]
        qv = hashgen.gen_values(seed, hashgen.KIND_Q, r, c - 1, layer, np.arange(Hq), d, q_scale_log2)
        q[i] = hashgen.to_bits(qv, dtype)
    return bt, pool_k, pool_v, q
