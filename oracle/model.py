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


def decode_step(s: ModelShape, weight_seed, kv_seed, req_ids, ctx, token_seed=None, layer_weights=None,
                head=None, kv_written=None):
    """The decode step of every request (module docstring).  Returns (logits [n][V],
    new_k [L][n][Hkv][d], new_v, x_final [n][H]).  layer_weights / head: optional cached
    results of weights() / head_weights().  kv_written: {(req, pos, layer): (k [Hkv][d], v)}
    -- history positions written by earlier model steps (instead of the synthetic fill)."""
    n = len(req_ids)
    d, Hkv = s.head_dim, s.kv_heads
    token_seed = weight_seed if token_seed is None else token_seed
    pos = [int(c) - 1 for c in ctx]
    toks = [int(hashgen.gen_token(token_seed, int(r), p, s.vocab)) for r, p in zip(req_ids, pos)]
    x = embed_rows(weight_seed, s, toks)
    new_k = np.zeros((s.layers, n, Hkv, d))
    new_v = np.zeros_like(new_k)
    for lay in range(s.layers):
        W = layer_weights[lay] if layer_weights is not None else weights(weight_seed, s, lay)
        h = rmsnorm(x, W["g1"], s.rms_eps)
        qkv = h @ W["w_qkv"].T
        a = np.zeros((n, s.q_heads * d))
        for i, (r, p) in enumerate(zip(req_ids, pos)):
            q = qkv[i, : s.q_heads * d].reshape(s.q_heads, d)
            k = qkv[i, s.q_heads * d:(s.q_heads + Hkv) * d].reshape(Hkv, d)
            v = qkv[i, (s.q_heads + Hkv) * d:].reshape(Hkv, d)
            q, k = rope(q, p, s.rope_theta), rope(k, p, s.rope_theta)
            new_k[lay, i], new_v[lay, i] = k, v
            hist = np.arange(p)[:, None]
            K = np.concatenate([hashgen.gen_values(kv_seed, hashgen.KIND_K, int(r), hist, lay,
                                                   np.arange(Hkv)[None, :], d), k[None]], axis=0)
            V = np.concatenate([hashgen.gen_values(kv_seed, hashgen.KIND_V, int(r), hist, lay,
                                                   np.arange(Hkv)[None, :], d), v[None]], axis=0)
            for (wr, wp, wl), (kk, vv) in (kv_written or {}).items():
                if wr == int(r) and wl == lay and wp < p:
                    K[wp], V[wp] = kk, vv
            a[i] = attention(q, K, V).reshape(-1)
        x = x + a @ W["w_o"].T
        h = rmsnorm(x, W["g2"], s.rms_eps)
        gu = h @ W["w_gu"].T
        x = x + (silu(gu[:, : s.ffn]) * gu[:, s.ffn:]) @ W["w_down"].T
    hw = head if head is not None else head_weights(weight_seed, s)
    logits = rmsnorm(x, hw["g_f"], s.rms_eps) @ hw["w_lm"].T
    return logits, new_k, new_v, x
