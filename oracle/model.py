"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O8: one full decode step of a Llama-2-shaped decoder in float64,
step by step, no fusion.  The paper does not define the model: its decode latency is the
whole model's ("the enlarged matrix dimensions in the matrix multiplication operations
required for larger batches"), measured on LLaMA-2/3 models (Table I).
Readings R32-R35 of DESIGN.md fix the architecture (Llama-2: pre-norm RMSNorm, RoPE with the
rotate-half pairing (j, j + d/2), causal attention = O1 over the paged history, SwiGLU MLP,
no biases, untied LM head) and the synthetic inputs (synth/hashgen.py weights and tokens).

For request i with ctx_i tokens (the decode token at position p = ctx_i - 1, token id
t_i = gen_token(req_i, p)):
    x = E[t_i]
    for each layer l:
        h = RMSNorm(x) * g1_l
        [q | k | v] = h W_qkv,l^T                (q: Hq x d, k, v: Hkv x d)
        q, k = RoPE(q, p), RoPE(k, p)
        K/V history of (req_i, layer l): positions < p from the pool's synthetic fill
            (kinds K/V of the generator), position p = (k, v) just computed
        a = attention(q, K, V) per q head (O1: softmax(q K^T / sqrt(d)) V, head group g(h))
        x = x + a W_o,l^T
        h = RMSNorm(x) * g2_l
        [gate | up] = h W_gu,l^T
        x = x + (silu(gate) * up) W_down,l^T
    logits = (RMSNorm(x) * g_f) W_lm^T
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from synth import hashgen


@dataclass(frozen=True)
class ModelShape:
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    hidden: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0


def weights(seed, s: ModelShape, layer):
    """float64 weights of one layer (the values the fp16 device weights hold exactly)."""
    H, d = s.hidden, s.head_dim
    nqkv = (s.q_heads + 2 * s.kv_heads) * d
    return dict(
        g1=hashgen.gen_norm_weight(seed, hashgen.KIND_LN1, layer, H),
        w_qkv=hashgen.gen_matrix(seed, hashgen.KIND_WQKV, layer, nqkv, H, hashgen.weight_scale_log2(H)),
        w_o=hashgen.gen_matrix(seed, hashgen.KIND_WO, layer, H, s.q_heads * d,
                               hashgen.weight_scale_log2(s.q_heads * d)),
        g2=hashgen.gen_norm_weight(seed, hashgen.KIND_LN2, layer, H),
        w_gu=hashgen.gen_matrix(seed, hashgen.KIND_WGU, layer, 2 * s.ffn, H, hashgen.weight_scale_log2(H)),
        w_down=hashgen.gen_matrix(seed, hashgen.KIND_WDOWN, layer, H, s.ffn, hashgen.weight_scale_log2(s.ffn)),
    )


def embed_rows(seed, s: ModelShape, tokens):
    return hashgen.gen_matrix(seed, hashgen.KIND_EMBED, 0, np.asarray(tokens), s.hidden, 0)


def head_weights(seed, s: ModelShape):
    sl = hashgen.weight_scale_log2(s.hidden)
    rows = [hashgen.gen_matrix(seed, hashgen.KIND_LM, 0, min(4096, s.vocab - r0), s.hidden, sl, row0=r0)
            for r0 in range(0, s.vocab, 4096)]
    return dict(g_f=hashgen.gen_norm_weight(seed, hashgen.KIND_LNF, 0, s.hidden), w_lm=np.concatenate(rows))


def linear(x, w):
    """y = x W^T in float64 (x: [M][K], W: [N][K] as stored: one output feature per row) -- the
    projections whose size grows with the batch ("the enlarged matrix dimensions in the matrix
    multiplication operations required for larger batches")."""
    return np.asarray(x, np.float64) @ np.asarray(w, np.float64).T


def rmsnorm(x, g, eps):
    """x / sqrt(mean(x^2) + eps) * g over the last axis."""
    x = np.asarray(x, np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x, pos, theta):
    """Rotate-half RoPE: pairs (j, j + d/2), angle pos * theta^(-2j/d)."""
    x = np.asarray(x, np.float64)
    d = x.shape[-1]
    j = np.arange(d // 2)
    ang = float(pos) * theta ** (-2.0 * j / d)
    c, sn = np.cos(ang), np.sin(ang)
    a, b = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([a * c - b * sn, b * c + a * sn], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


def greedy_ok(logits_row, token, tol):
    """Greedy sampling (argmax) has several right answers when logits tie within the rounding
    of a lower-precision path: token is valid iff its logit is within tol * max|logit| of the
    row's maximum."""
    row = np.asarray(logits_row, np.float64)
    return 0 <= token < len(row) and row[token] >= row.max() - tol * np.abs(row).max()


def attention(q, K, V):
    """q [Hq][d], K, V [ctx][Hkv][d]: O1 for one request (full softmax, scale 1/sqrt(d))."""
    Hq, d = q.shape
    grp = Hq // K.shape[1]
    out = np.empty((Hq, d))
    for h in range(Hq):
        g = h // grp
        s = K[:, g, :] @ q[h] / np.sqrt(d)
        p = np.exp(s - s.max())
        out[h] = (p / p.sum()) @ V[:, g, :]
    return out


def forward_rows(s: ModelShape, weight_seed, kv_seed, rows, token_seed=None, layer_weights=None, head=None,
                 kv_written=None, tokens=None):
    """One model step over activation rows [(req, pos)] -- decode tokens (pos = ctx - 1) and
    prefill-chunk tokens (PD fusion, R24: a chunk token at position p attends causally to
    positions 0..p of its request).  Layer by layer: every row's (k, v) is computed first,
    then each row attends over its request's positions 0..p, taking a position's K/V from
    (in order) this step's rows, kv_written {(req, pos, layer): (k, v)} of earlier steps, or
    the pool's synthetic fill (generator kinds K/V).  tokens: optional input token ids of the
    first len(tokens) rows (instead of gen_token).  Returns (logits [R][V],
    written {(req, pos, layer): (k, v)} of this step, x_final [R][H])."""
    R = len(rows)
    d, Hkv = s.head_dim, s.kv_heads
    token_seed = weight_seed if token_seed is None else token_seed
    toks = [int(hashgen.gen_token(token_seed, int(r), int(p), s.vocab)) for r, p in rows]
    for i, t in enumerate(tokens or []):
        toks[i] = int(t)
    x = embed_rows(weight_seed, s, toks)
    written = {}
    for lay in range(s.layers):
        W = layer_weights[lay] if layer_weights is not None else weights(weight_seed, s, lay)
        h = rmsnorm(x, W["g1"], s.rms_eps)
        qkv = h @ W["w_qkv"].T
        qs = []
        for i, (r, p) in enumerate(rows):
            q = qkv[i, : s.q_heads * d].reshape(s.q_heads, d)
            k = qkv[i, s.q_heads * d:(s.q_heads + Hkv) * d].reshape(Hkv, d)
            v = qkv[i, (s.q_heads + Hkv) * d:].reshape(Hkv, d)
            qs.append(rope(q, p, s.rope_theta))
            written[(int(r), int(p), lay)] = (rope(k, p, s.rope_theta), v)
        a = np.zeros((R, s.q_heads * d))
        for i, (r, p) in enumerate(rows):
            pos = np.arange(p + 1)[:, None]
            K = hashgen.gen_values(kv_seed, hashgen.KIND_K, int(r), pos, lay, np.arange(Hkv)[None, :], d)
            V = hashgen.gen_values(kv_seed, hashgen.KIND_V, int(r), pos, lay, np.arange(Hkv)[None, :], d)
            for j in range(p + 1):
                src = written.get((int(r), j, lay))
                if src is None and kv_written is not None:
                    src = kv_written.get((int(r), j, lay))
                if src is not None:
                    K[j], V[j] = src
            a[i] = attention(qs[i], K, V).reshape(-1)
        x = x + a @ W["w_o"].T
        h = rmsnorm(x, W["g2"], s.rms_eps)
        gu = h @ W["w_gu"].T
        x = x + (silu(gu[:, : s.ffn]) * gu[:, s.ffn:]) @ W["w_down"].T
    hw = head if head is not None else head_weights(weight_seed, s)
    logits = rmsnorm(x, hw["g_f"], s.rms_eps) @ hw["w_lm"].T
    return logits, written, x


def decode_step(s: ModelShape, weight_seed, kv_seed, req_ids, ctx, token_seed=None, layer_weights=None,
                head=None, kv_written=None, tokens=None):
    """The decode step of every request (module docstring): forward_rows over the rows
    (req_i, ctx_i - 1).  Returns (logits [n][V], new_k [L][n][Hkv][d], new_v, x_final [n][H])."""
    rows = [(int(r), int(c) - 1) for r, c in zip(req_ids, ctx)]
    logits, written, x = forward_rows(s, weight_seed, kv_seed, rows, token_seed, layer_weights, head, kv_written,
                                      tokens)
    n = len(rows)
    new_k = np.zeros((s.layers, n, s.kv_heads, s.head_dim))
    new_v = np.zeros_like(new_k)
    for lay in range(s.layers):
        for i, (r, p) in enumerate(rows):
            new_k[lay, i], new_v[lay, i] = written[(r, p, lay)]
    return logits, new_k, new_v, x
