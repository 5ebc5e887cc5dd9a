"""Pins for oracle O1 (paged decode attention) -- CPU only.

The oracle is checked against things other than itself: the IEEE formats
(every fp16/bf16 bit pattern), dense brute force computed from the LOGICAL
token values without any paging (numpy and torch SDPA in float64), closed
forms, and invariants (SURVEY.md §8(c) O1 pins i-iv)."""
import numpy as np
import pytest
import torch

from oracle import attention as oatt
from synth import hashgen


def test_half_to_double_all_bit_patterns():
    L = oatt.lib()
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([L.oracle_half_to_double(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def test_bf16_to_double_all_bit_patterns():
    L = oatt.lib()
    bits = np.arange(65536, dtype=np.uint32)
    with np.errstate(invalid="ignore"):  # the NaN patterns widen to NaN, as intended
        ref = (bits << 16).astype(np.uint32).view(np.float32).astype(np.float64)
    got = np.array([L.oracle_bf16_to_double(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def _dense_reference(q, K, V):
    """softmax(q K^T / sqrt(d)) V for one head, float64, written without paging."""
    s = K @ q / np.sqrt(q.shape[0])
    p = np.exp(s - s.max())
    return (p / p.sum()) @ V


def _random_case(rng, n, Hq, Hkv, d, P, dtype, seed, max_ctx=70, q_scale_log2=0):
    ctx = rng.integers(1, max_ctx + 1, n)
    npg = [-(-int(c) // P) for c in ctx]
    perm = rng.permutation(sum(npg) + 5)  # scattered physical ids, some unused
    pages, k = [], 0
    for m in npg:
        pages.append([int(x) for x in perm[k:k + m]])
        k += m
    req_ids = [int(x) for x in rng.integers(0, 1 << 40, n)]
    bt, pk, pv, q = oatt.synth_paged_batch(seed, req_ids, ctx, pages, 3, Hq, Hkv, d, P, dtype,
                                           q_scale_log2=q_scale_log2)
    return req_ids, ctx, pages, bt, pk, pv, q


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("Hq,Hkv,d", [(4, 4, 64), (8, 2, 64), (4, 1, 128)])
@pytest.mark.parametrize("q_scale_log2", [0, 4])
def test_paged_matches_dense_bruteforce(dtype, Hq, Hkv, d, q_scale_log2):
    rng = np.random.default_rng(7)
    P, seed, layer = 16, 11, 3
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 5, Hq, Hkv, d, P, dtype, seed,
                                                       q_scale_log2=q_scale_log2)
    out = oatt.paged_decode_attention(ctx, bt, pk, pv, q, dtype)
    for i, (r, c) in enumerate(zip(req_ids, ctx)):
        for h in range(Hq):
            g = h // (Hq // Hkv)
            K = hashgen.gen_values(seed, hashgen.KIND_K, r, np.arange(c), layer, g, d)
            V = hashgen.gen_values(seed, hashgen.KIND_V, r, np.arange(c), layer, g, d)
            qv = hashgen.gen_values(seed, hashgen.KIND_Q, r, c - 1, layer, h, d, q_scale_log2)
            ref = _dense_reference(qv, K, V)
            np.testing.assert_allclose(out[i, h], ref, rtol=1e-12, atol=1e-14)
            t = torch.nn.functional.scaled_dot_product_attention(
                torch.from_numpy(qv)[None, None, None, :], torch.from_numpy(K)[None, None],
                torch.from_numpy(V)[None, None])[0, 0, 0].numpy()
            np.testing.assert_allclose(out[i, h], t, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_prefill_oracle_matches_dense_causal_attention(dtype):
    """Pin of the chunked-prefill reading (R24): every chunk row equals dense causal
    attention over the request's whole prefix (torch SDPA with an explicit bottom-right
    causal mask, no paging)."""
    rng = np.random.default_rng(3)
    P, seed, layer, Hq, Hkv, d = 16, 5, 1, 4, 2, 64
    ctx = np.array([40, 17, 70])
    q_start = np.array([0, 9, 33])
    q_len = ctx - q_start
    npg = [-(-int(c) // P) for c in ctx]
    perm = rng.permutation(sum(npg) + 3)
    pages, k = [], 0
    for m in npg:
        pages.append([int(x) for x in perm[k:k + m]])
        k += m
    req_ids = [101, 7, 1 << 33]
    bt, pk, pv, _ = oatt.synth_paged_batch(seed, req_ids, ctx, pages, layer, Hq, Hkv, d, P, dtype)
    qrows = [hashgen.to_bits(hashgen.gen_values(seed, hashgen.KIND_Q, r, np.arange(s, c)[:, None], layer,
                                                np.arange(Hq)[None, :], d), dtype)
             for r, s, c in zip(req_ids, q_start, ctx)]
    out = oatt.paged_prefill_attention(q_start, q_len, bt, pk, pv, np.concatenate(qrows), dtype)
    conv = oatt.lib().oracle_half_to_double if dtype == "f16" else oatt.lib().oracle_bf16_to_double
    row = 0
    for i, (r, s, c) in enumerate(zip(req_ids, q_start, ctx)):
        K = hashgen.gen_values(seed, hashgen.KIND_K, r, np.arange(c)[:, None], layer, np.arange(Hkv)[None, :], d)
        V = hashgen.gen_values(seed, hashgen.KIND_V, r, np.arange(c)[:, None], layer, np.arange(Hkv)[None, :], d)
        # round K/V/q through the storage dtype exactly as the pool holds them
        rnd = np.vectorize(lambda b: conv(int(b)))
        K = rnd(hashgen.to_bits(K, dtype))
        V = rnd(hashgen.to_bits(V, dtype))
        Q = rnd(qrows[i])  # [c-s][Hq][d]
        mask = np.arange(c)[None, :] <= np.arange(s, c)[:, None]
        for h in range(Hq):
            g = h // (Hq // Hkv)
            t = torch.nn.functional.scaled_dot_product_attention(
                torch.from_numpy(Q[:, h])[None, None], torch.from_numpy(K[:, g])[None, None],
                torch.from_numpy(V[:, g])[None, None], attn_mask=torch.from_numpy(mask)[None, None])[0, 0].numpy()
            np.testing.assert_allclose(out[row:row + c - s, h], t, rtol=1e-12, atol=1e-14)
        row += c - s


def test_ctx_one_returns_v0_exactly():
    rng = np.random.default_rng(1)
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 6, 4, 4, 64, 16, "f16", 5, max_ctx=1)
    out = oatt.paged_decode_attention(ctx, bt, pk, pv, q, "f16")
    for i in range(6):
        v0 = pv[pages[i][0], :, 0, :].view(np.float16).astype(np.float64)
        assert np.array_equal(out[i], v0)


def test_identical_keys_or_zero_query_give_mean_of_v():
    rng = np.random.default_rng(2)
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 4, 2, 2, 64, 16, "bf16", 9, max_ctx=50)
    # identical keys: overwrite every K row with one row
    pk2 = pk.copy()
    pk2[:] = pk[0, 0, 0, :]
    out = oatt.paged_decode_attention(ctx, bt, pk2, pv, q, "bf16")
    q0 = np.zeros_like(q)
    out0 = oatt.paged_decode_attention(ctx, bt, pk, pv, q0, "bf16")
    for i, c in enumerate(ctx):
        V = np.stack([pv[pages[i][j // 16], :, j % 16, :] for j in range(c)])
        Vd = (V.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        np.testing.assert_allclose(out[i], Vd.mean(0), rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(out0[i], Vd.mean(0), rtol=1e-12, atol=1e-15)


def test_dominant_score_selects_its_value_row():
    d, P = 64, 16
    ctx = np.array([40], np.int32)
    bt = np.array([[2, 0, 1]], np.int32)
    pk = np.zeros((3, 1, P, d), np.float16)
    pv = np.random.default_rng(3).integers(-128, 128, (3, 1, P, d)).astype(np.float16) / 128
    pk[0, 0, 5, :] = 8.0  # logical token 16 + 5 = 21 lives on physical page 0, slot 5
    q = np.full((1, 1, d), 8.0, np.float16)
    out = oatt.paged_decode_attention(ctx, bt, pk.view(np.uint16), pv.view(np.uint16),
                                      q.view(np.uint16), "f16")
    np.testing.assert_allclose(out[0, 0], pv[0, 0, 5].astype(np.float64), rtol=0, atol=1e-12)


def test_paging_invariance_bit_identical():
    rng = np.random.default_rng(4)
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 5, 4, 2, 64, 16, "f16", 13)
    out = oatt.paged_decode_attention(ctx, bt, pk, pv, q, "f16")
    perm = rng.permutation(pk.shape[0])
    inv = np.argsort(perm)  # new id of old page p is inv[p]
    pk2, pv2 = pk[perm], pv[perm]
    bt2 = np.where(bt >= 0, inv[np.maximum(bt, 0)], -1).astype(np.int32)
    out2 = oatt.paged_decode_attention(ctx, bt2, pk2, pv2, q, "f16")
    assert np.array_equal(out, out2)


def test_gqa_reduces_to_mha_and_equal_queries_agree():
    rng = np.random.default_rng(5)
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 3, 8, 2, 64, 16, "f16", 17)
    q2 = q.copy()
    q2[:, 1] = q2[:, 0]  # heads 0 and 1 share KV head 0
    out = oatt.paged_decode_attention(ctx, bt, pk, pv, q2, "f16")
    assert np.array_equal(out[:, 0], out[:, 1])
    # Hq = Hkv: expand KV heads so each q head has its own copy -> same result as GQA
    pk_m = np.repeat(pk, 4, axis=1)
    pv_m = np.repeat(pv, 4, axis=1)
    out_m = oatt.paged_decode_attention(ctx, bt, pk_m, pv_m, q2, "f16")
    assert np.array_equal(out, out_m)


def test_threads_do_not_change_result():
    rng = np.random.default_rng(6)
    req_ids, ctx, pages, bt, pk, pv, q = _random_case(rng, 7, 4, 4, 64, 16, "bf16", 19)
    a = oatt.paged_decode_attention(ctx, bt, pk, pv, q, "bf16", nthreads=1)
    b = oatt.paged_decode_attention(ctx, bt, pk, pv, q, "bf16", nthreads=4)
    assert np.array_equal(a, b)


def test_invalid_arguments_rejected():
    bt = np.array([[0]], np.int32)
    pk = np.zeros((1, 1, 16, 64), np.uint16)
    q = np.zeros((1, 1, 64), np.uint16)
    with pytest.raises(ValueError):
        oatt.paged_decode_attention(np.array([0], np.int32), bt, pk, pk, q)
    with pytest.raises(ValueError):
        oatt.paged_decode_attention(np.array([20], np.int32), bt, pk, pk, q)  # page 1 missing (-1)
