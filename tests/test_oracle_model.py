"""Pins for oracle O8 (full decode step, oracle/model.py; R32-R35) -- CPU only.

The oracle is checked against formulations it does not share: RoPE as complex
multiplication, the whole decoder against torch.nn.functional (rms_norm, complex RoPE via
torch.polar, scaled_dot_product_attention with GQA, silu, linear) in float64, and closed
forms (RMSNorm of a constant vector, RoPE at position 0, relative-position invariance,
attention over one token, the residual path with zeroed output projections)."""
import numpy as np
import pytest

from oracle import model as om
from synth import hashgen

torch = pytest.importorskip("torch")


def test_rmsnorm_closed_form():
    g = np.array([0.5, 2.0, 1.0, 1.5])
    x = np.full(4, -3.0)
    assert np.allclose(om.rmsnorm(x, g, 1e-5), g * (-3.0 / np.sqrt(9.0 + 1e-5)), rtol=0, atol=1e-15)
    y = np.array([3.0, 4.0, 0.0, 0.0])             # mean square 25/4
    assert np.allclose(om.rmsnorm(y, 1.0, 0.0), y / 2.5, rtol=0, atol=1e-15)


def test_rope_matches_complex_rotation_and_is_relative():
    rng = np.random.default_rng(0)
    d, theta = 128, 10000.0
    q, k = rng.standard_normal(d), rng.standard_normal(d)
    for p in (0, 1, 17, 4095):
        z = (q[: d // 2] + 1j * q[d // 2:]) * np.exp(1j * p * theta ** (-np.arange(d // 2) * 2.0 / d))
        assert np.allclose(om.rope(q, p, theta), np.concatenate([z.real, z.imag]), rtol=0, atol=1e-12)
    assert np.array_equal(om.rope(q, 0, theta), q)
    assert np.isclose(np.linalg.norm(om.rope(q, 999, theta)), np.linalg.norm(q), rtol=1e-13)
    # q(m).k(n) depends on m - n only
    a = om.rope(q, 40, theta) @ om.rope(k, 33, theta)
    b = om.rope(q, 1040, theta) @ om.rope(k, 1033, theta)
    assert np.isclose(a, b, rtol=1e-10)


def test_attention_over_one_token_is_v():
    rng = np.random.default_rng(1)
    q = rng.standard_normal((8, 64))
    K, V = rng.standard_normal((1, 2, 64)), rng.standard_normal((1, 2, 64))
    out = om.attention(q, K, V)
    assert np.allclose(out, np.repeat(V[0], 4, axis=0), rtol=0, atol=1e-15)


def _torch_decode_step(s, wseed, kvseed, req_ids, ctx):
    """Independent float64 formulation with torch.nn.functional."""
    import torch.nn.functional as F
    T = lambda a: torch.from_numpy(np.asarray(a, np.float64))  # noqa: E731
    d, n = s.head_dim, len(req_ids)
    pos = [c - 1 for c in ctx]
    toks = [int(hashgen.gen_token(wseed, r, p, s.vocab)) for r, p in zip(req_ids, pos)]
    x = T(hashgen.gen_matrix(wseed, hashgen.KIND_EMBED, 0, np.array(toks), s.hidden, 0))
    inv = torch.tensor([s.rope_theta ** (-2.0 * j / d) for j in range(d // 2)], dtype=torch.float64)

    def rot(t, p):  # [..., d] as complex pairs (j, j + d/2)
        z = torch.complex(t[..., : d // 2], t[..., d // 2:]) * torch.polar(torch.ones_like(inv), p * inv)
        return torch.cat([z.real, z.imag], dim=-1)
    for lay in range(s.layers):
        W = {k: T(v) for k, v in om.weights(wseed, s, lay).items()}
        h = F.rms_norm(x, (s.hidden,), W["g1"], s.rms_eps)
        qkv = F.linear(h, W["w_qkv"])
        outs = []
        for i in range(n):
            q = qkv[i, : s.q_heads * d].view(s.q_heads, d)
            k = qkv[i, s.q_heads * d:(s.q_heads + s.kv_heads) * d].view(s.kv_heads, d)
            v = qkv[i, (s.q_heads + s.kv_heads) * d:].view(s.kv_heads, d)
            q, k = rot(q, pos[i]), rot(k, pos[i])
            hist = np.arange(pos[i])[:, None]
            K = torch.cat([T(hashgen.gen_values(kvseed, 1, req_ids[i], hist, lay, np.arange(s.kv_heads)[None], d)),
                           k[None]])
            V = torch.cat([T(hashgen.gen_values(kvseed, 2, req_ids[i], hist, lay, np.arange(s.kv_heads)[None], d)),
                           v[None]])
            o = F.scaled_dot_product_attention(q[:, None, :], K.transpose(0, 1), V.transpose(0, 1),
                                               enable_gqa=True)
            outs.append(o[:, 0, :].reshape(-1))
        x = x + F.linear(torch.stack(outs), W["w_o"])
        h = F.rms_norm(x, (s.hidden,), W["g2"], s.rms_eps)
        gate, up = F.linear(h, W["w_gu"]).split(s.ffn, dim=-1)
        x = x + F.linear(F.silu(gate) * up, W["w_down"])
        hw = {k: T(v) for k, v in om.head_weights(wseed, s).items()}
    return F.linear(F.rms_norm(x, (s.hidden,), hw["g_f"], s.rms_eps), hw["w_lm"]).numpy(), x.numpy()


@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (8, 2)])
def test_decode_step_matches_torch_functional(Hq, Hkv):
    s = om.ModelShape(layers=2, q_heads=Hq, kv_heads=Hkv, head_dim=64, hidden=256, ffn=384, vocab=300)
    req, ctx = [3, 10, 77], [1, 17, 40]
    logits, nk, nv, x = om.decode_step(s, 5, 9, req, ctx)
    tl, tx = _torch_decode_step(s, 5, 9, req, ctx)
    assert np.allclose(x, tx, rtol=1e-12, atol=1e-12)
    assert np.allclose(logits, tl, rtol=1e-12, atol=1e-12)
    assert nk.shape == (2, 3, Hkv, 64)


def test_zero_output_projections_leave_the_embedding():
    s = om.ModelShape(layers=2, q_heads=4, kv_heads=4, head_dim=64, hidden=256, ffn=256, vocab=50)
    lw = [om.weights(1, s, lay) for lay in range(2)]
    for W in lw:
        W["w_o"][:] = 0.0
        W["w_down"][:] = 0.0
    _, _, _, x = om.decode_step(s, 1, 2, [5, 6], [3, 9], layer_weights=lw)
    toks = [int(hashgen.gen_token(1, r, c - 1, 50)) for r, c in ((5, 3), (6, 9))]
    assert np.array_equal(x, om.embed_rows(1, s, toks))


def test_synthetic_weights_are_exact_in_fp16():
    s = om.ModelShape(layers=1, q_heads=4, kv_heads=2, head_dim=128, hidden=512, ffn=1024, vocab=64)
    for v in list(om.weights(3, s, 0).values()) + list(om.head_weights(3, s).values()):
        hashgen.to_bits(v, "f16")  # raises if any value is not exact


def test_chunked_prefill_equals_token_by_token_decode():
    """R24 causal semantics: a whole prompt in one step (rows (r, 0..P-1)), the same prompt in
    two chunks, and P single-token steps (each attending over the K/V the earlier steps
    wrote) give the same logits and K/V."""
    s = om.ModelShape(layers=2, q_heads=8, kv_heads=2, head_dim=64, hidden=256, ffn=256, vocab=120)
    r, P = 42, 9
    full, wf, _ = om.forward_rows(s, 1, 2, [(r, p) for p in range(P)])
    a, wa, _ = om.forward_rows(s, 1, 2, [(r, p) for p in range(4)])
    b, wb, _ = om.forward_rows(s, 1, 2, [(r, p) for p in range(4, P)], kv_written=wa)
    assert np.allclose(np.concatenate([a, b]), full, rtol=1e-12, atol=1e-12)
    seq, kv = [], {}
    for p in range(P):
        lg, w, _ = om.forward_rows(s, 1, 2, [(r, p)], kv_written=kv)
        kv.update(w)
        seq.append(lg[0])
    assert np.allclose(np.stack(seq), full, rtol=1e-12, atol=1e-12)
    for key, (k, v) in wf.items():
        assert np.allclose(kv[key][0], k, rtol=1e-12, atol=1e-12) and np.allclose(kv[key][1], v, rtol=1e-12, atol=1e-12)


def test_prefill_matches_torch_causal_attention():
    """A whole prompt through one layer vs torch (F.scaled_dot_product_attention is_causal)."""
    import torch.nn.functional as F
    s = om.ModelShape(layers=1, q_heads=4, kv_heads=4, head_dim=64, hidden=256, ffn=256, vocab=50)
    r, P, d = 7, 6, 64
    _, written, x = om.forward_rows(s, 3, 4, [(r, p) for p in range(P)])
    W = om.weights(3, s, 0)
    toks = [int(hashgen.gen_token(3, r, p, s.vocab)) for p in range(P)]
    T = lambda a: torch.from_numpy(np.asarray(a, np.float64))  # noqa: E731
    x0 = T(om.embed_rows(3, s, toks))
    h = F.rms_norm(x0, (s.hidden,), T(W["g1"]), s.rms_eps)
    qkv = F.linear(h, T(W["w_qkv"]))
    q = torch.stack([T(om.rope(qkv[p, :256].view(4, d).numpy(), p, s.rope_theta)) for p in range(P)])
    k = torch.stack([T(written[(r, p, 0)][0]) for p in range(P)])
    v = qkv[:, 512:].view(P, 4, d)
    o = F.scaled_dot_product_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1), is_causal=True)
    x1 = x0 + F.linear(o.transpose(0, 1).reshape(P, -1), T(W["w_o"]))
    h2 = F.rms_norm(x1, (s.hidden,), T(W["g2"]), s.rms_eps)
    g, u = F.linear(h2, T(W["w_gu"])).split(s.ffn, dim=-1)
    x2 = x1 + F.linear(F.silu(g) * u, T(W["w_down"]))
    assert np.allclose(x, x2.numpy(), rtol=1e-12, atol=1e-12)


def test_greedy_ok_rule():
    row = np.array([0.5, 2.0, 1.999, -3.0])
    assert om.greedy_ok(row, 1, 2e-3)                 # the argmax
    assert om.greedy_ok(row, 2, 2e-3)                 # within 2e-3 * max|logit| = 6e-3 of it
    assert not om.greedy_ok(row, 0, 2e-3)
    assert not om.greedy_ok(row, 4, 2e-3) and not om.greedy_ok(row, -1, 2e-3)


def test_linear_is_the_brute_force_sum():
    """O8 linear (y = x W^T) pinned by the triple loop on a tiny case, W stored one output
    feature per row (so a transposed operand fails)."""
    rng = np.random.default_rng(5)
    x = rng.integers(-4, 5, (3, 5)).astype(np.float64)
    w = rng.integers(-4, 5, (4, 5)).astype(np.float64)
    want = np.zeros((3, 4))
    for m in range(3):
        for n in range(4):
            for k in range(5):
                want[m, n] += x[m, k] * w[n, k]
    assert np.array_equal(om.linear(x, w), want)
