"""GPU parity of the full decode step (NEXT row 3; dbk_model_*, R32-R35) against the
fp64 oracle O8 (oracle/model.py).

Bar (R35, element-wise like R23): fp16 weights and fp16 activations at every GEMM boundary with
fp32 accumulation and an fp32 residual stream vs the fp64 oracle on the same (exactly
representable) weights: for every row, max_j |got_j - want_j| <= MODEL_TOL * max_j |want_j| --
the logits row (one wrong logit among V fails it, which a row L2 norm would dilute by ~1/sqrt(V)),
and every K / V row [Hkv][d] the model writes into the pool.  Block tables / ctx after
dbk_reserve_tokens are bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import model as om  # noqa: E402
from oracle import policy as opol  # noqa: E402
from oracle import engine as oeng  # noqa: E402
from oracle.allocator import PagedKV  # noqa: E402
from synth import configs, trace  # noqa: E402
from test_gpu_parity import dbk  # noqa: E402,F401

MODEL_TOL = 2e-3  # R35 = R23 applied to the model step (observed maxima: profiles/r02_model_err.json)
P = 16


OBSERVED = {}  # largest error seen per quantity (written to gpurun_out/model_err.json if that exists)


def row_err(got, want, what=None):
    """max over rows of ||got - want||_inf / ||want||_inf, a row = the last axis (a request's
    logits; one head's K or V vector of d elements)."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    got, want = got.reshape(-1, got.shape[-1]), want.reshape(-1, want.shape[-1])
    e = float((np.abs(got - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)).max())
    if what:
        OBSERVED[what] = max(OBSERVED.get(what, 0.0), e)
    return e


@pytest.fixture(scope="module", autouse=True)
def _record_errors():
    yield
    import json
    import os
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if OBSERVED and os.path.isdir(out):
        with open(os.path.join(out, "model_err.json"), "w") as f:
            json.dump({"bar": MODEL_TOL, "observed_max_row_inf_rel": OBSERVED}, f, indent=1)


def _read_kv(pool, s, req, pos, layer):
    """The K and V rows [Hkv][d] of (req, pos, layer) straight from the pool's memory."""
    _, _, pages = pool.request_info(req)
    cap = pool.cfg.cap_pages
    t = pool.kv.view(torch.float16).view(s.layers, cap, s.kv_heads, 2, P, s.head_dim)
    tile = t[layer, pages[pos // P], :, :, pos % P, :].float().cpu().numpy()
    return tile[:, 0, :], tile[:, 1, :]


def _setup(dbk, s, ctx, kv_seed, wseed, cap=None, max_req=None):
    n = len(ctx)
    maxp = max(-(-(c + 4) // P) for c in ctx) + 1
    cap = cap or sum(-(-(c + 1) // P) for c in ctx) + 4
    pool = dbk.KVPool(s.layers, s.q_heads, s.kv_heads, s.head_dim, cap, max_req or n + 2, maxp, "f16")
    model = dbk.Model(pool, s.hidden, s.ffn, s.vocab, max_pos=maxp * P, weight_seed=wseed)
    ids = [int(i) * 131 + 7 for i in range(n)]
    ref = PagedKV(cap, P)
    for r, c in zip(ids, ctx):
        pool.request_begin(r, max(1, c - 1), 4)
        ref.begin(r)
    pool.append_tokens(ids, [c - 1 for c in ctx], seed=kv_seed)   # the synthetic history
    ref.append(ids, [c - 1 for c in ctx])
    return pool, model, ids, ref


@pytest.mark.parametrize("shape", [
    om.ModelShape(layers=2, q_heads=4, kv_heads=4, head_dim=64, hidden=256, ffn=384, vocab=300),
    om.ModelShape(layers=3, q_heads=8, kv_heads=2, head_dim=128, hidden=512, ffn=640, vocab=1000),
    om.ModelShape(layers=1, q_heads=16, kv_heads=2, head_dim=128, hidden=2048, ffn=1408, vocab=512),
])
def test_model_step_parity(dbk, shape):
    s = shape
    kv_seed, wseed = 5, 11
    ctx = [1, 2, 16, 17, 33, 100, 257]
    pool, model, ids, ref = _setup(dbk, s, ctx, kv_seed, wseed)
    pool.reserve_tokens(ids, [1] * len(ids))
    ref.append(ids, [1] * len(ids))
    for r in ids:
        c, _, pages = pool.request_info(r)
        assert c == ref.ctx[r] and pages == ref.pages[r]
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step(ids, logits)
    st = pool.batch_stats()
    assert st["n_active"] == len(ids) and st["sum_ctx"] == sum(ctx) and st["table_mismatch"] == 0
    want, nk, nv, _ = om.decode_step(s, wseed, kv_seed, ids, ctx)
    assert row_err(logits.cpu().numpy(), want, "logits") <= MODEL_TOL
    for lay in range(s.layers):
        for i, (r, c) in enumerate(zip(ids, ctx)):
            k, v = _read_kv(pool, s, r, c - 1, lay)
            assert row_err(k, nk[lay, i], "k") <= MODEL_TOL and row_err(v, nv[lay, i], "v") <= MODEL_TOL
    model.close()
    pool.close()


def test_model_two_steps_attend_to_model_written_kv(dbk):
    """Step 2 attends over the K/V step 1 wrote (oracle: kv_written from its own step 1)."""
    s = om.ModelShape(layers=2, q_heads=8, kv_heads=4, head_dim=64, hidden=512, ffn=512, vocab=400)
    kv_seed, wseed = 3, 4
    ctx = [5, 16, 31, 64]
    pool, model, ids, ref = _setup(dbk, s, ctx, kv_seed, wseed)
    pool.reserve_tokens(ids, [1] * len(ids))
    model.step(ids)
    _, k1, v1, _ = om.decode_step(s, wseed, kv_seed, ids, ctx)
    written = {(r, c - 1, lay): (k1[lay, i], v1[lay, i]) for i, (r, c) in enumerate(zip(ids, ctx))
               for lay in range(s.layers)}
    pool.reserve_tokens(ids, [1] * len(ids))
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step(ids, logits)
    want, _, _, _ = om.decode_step(s, wseed, kv_seed, ids, [c + 1 for c in ctx], kv_written=written)
    assert row_err(logits.cpu().numpy(), want, "logits_step2") <= MODEL_TOL
    model.close()
    pool.close()


def test_model_llama2_7b_layer_full_size(dbk):
    """One Llama-2-7B-shaped layer (H 4096, 32 x 128 heads, F 11008, V 32000), 4 requests."""
    s = om.ModelShape(layers=1, q_heads=32, kv_heads=32, head_dim=128, hidden=4096, ffn=11008, vocab=32000)
    kv_seed, wseed = 21, 22
    ctx = [3, 190, 573, 1100]
    pool, model, ids, ref = _setup(dbk, s, ctx, kv_seed, wseed)
    pool.reserve_tokens(ids, [1] * len(ids))
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step(ids, logits)
    want, nk, nv, _ = om.decode_step(s, wseed, kv_seed, ids, ctx)
    assert row_err(logits.cpu().numpy(), want, "logits_7b") <= MODEL_TOL
    for i, (r, c) in enumerate(zip(ids, ctx)):
        k, v = _read_kv(pool, s, r, c - 1, 0)
        assert row_err(k, nk[0, i], "k_7b") <= MODEL_TOL and row_err(v, nv[0, i], "v_7b") <= MODEL_TOL
    model.close()
    pool.close()


def test_engine_full_model_mode_replays(dbk):
    """The engine with the model attached: every decision bit-exact against the oracle's
    replay of the logged step times; the K/V the model writes is what later steps read
    (checked per step above); here the batch bookkeeping and telemetry."""
    c = configs.CONFIGS["toy-tight"]
    tr = trace.make_trace(30, 128, 128, 256, seed=1, dist="uniform")
    L, Hq, Hkv, d = 2, 8, 8, 64
    cap_pages = c["cap_tokens"] // P
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(c)
    kw = dict(policy=opol.MEMORY, b_static=c["b_max"], b_min=c["b_min"], b_max=c["b_max"], b0=c["b_min"],
              eps_m=c["eps_m"], bytes_per_token=beta, page_size=P, refresh_steps=5, w_len=16, w_sla=4,
              alpha=4, delta=1, d_sla_ms=50.0, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    max_req = c["b_max"] + 2
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, max_req, 16, "f16")
    model = dbk.Model(pool, 512, 768, 500, max_pos=256, weight_seed=9)
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=31, out_dtype=2)
    eng.attach_model(model)
    qd = torch.empty(L, max_req, Hq, d, dtype=torch.float16, device="cuda")
    od = torch.empty(L, max_req, Hq, d, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P)],
                     opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    n = 0
    while not eng.done():
        g = eng.step(bufs)
        o = rp.step(g["step_ns"])
        for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx", "used_pages",
                  "rationale"):
            assert g[k] == o[k], (k, g[k], o[k])
        assert (g["table_hash"] & ((1 << 64) - 1)) == o["table_hash"]
        n += 1
    assert rp.done() and n > 10
    a_ms, t_ms, steps = model.timing()
    assert steps > 0 and 0 < a_ms < t_ms
    eng.close()
    model.close()
    pool.close()


def test_model_step_pd_chunks_and_decode_rows(dbk):
    """PD fusion through the model (dbk_model_step_pd): decode rows of two requests with a
    synthetic history + a 40-token prompt prefilled in two chunks (24 + 16 tokens) over two
    steps; step 2's chunk attends over step 1's model-written K/V.  Oracle: forward_rows with
    the K/V of its own step 1 (R24)."""
    s = om.ModelShape(layers=2, q_heads=8, kv_heads=2, head_dim=128, hidden=512, ffn=640, vocab=700)
    kv_seed, wseed = 8, 9
    pool, model, ids, ref = _setup(dbk, s, [20, 45], kv_seed, wseed, cap=40, max_req=32)
    C = 999
    pool.request_begin(C, 40, 4)
    written = {}
    ctx = {ids[0]: 19, ids[1]: 44}
    for s0, k in ((0, 24), (24, 16)):
        pool.reserve_tokens(ids, [1, 1])
        pool.reserve_tokens([C], [k])
        for r in ids:
            ctx[r] += 1
        R = 2 + k
        logits = torch.empty(R, s.vocab, dtype=torch.float32, device="cuda")
        model.step_pd(ids, [C], [s0], [k], logits)
        st = pool.batch_stats()
        assert st["n_active"] == 2 and st["sum_ctx"] == ctx[ids[0]] + ctx[ids[1]]
        rows = [(r, ctx[r] - 1) for r in ids] + [(C, s0 + j) for j in range(k)]
        want, w, _ = om.forward_rows(s, wseed, kv_seed, rows, kv_written=written)
        written.update(w)
        assert row_err(logits.cpu().numpy(), want, "logits_pd") <= MODEL_TOL
        for lay in range(s.layers):
            for (r, p) in rows:
                kk, vv = _read_kv(pool, s, r, p, lay)
                assert row_err(kk, w[(r, p, lay)][0], "k_pd") <= MODEL_TOL
                assert row_err(vv, w[(r, p, lay)][1], "v_pd") <= MODEL_TOL
    with pytest.raises(dbk.DbkError):  # a chunk beyond the reserved tokens
        model.step_pd(ids, [C], [38], [4])
    model.close()
    pool.close()


def test_engine_pd_fusion_with_model_replays(dbk):
    """PD fusion + the full model in the engine: prompts are prefilled THROUGH the model in
    chunks of c_t = max(0, b_t - N^d) tokens (R25-R27, R34 no longer applies); every record
    incl. the chunk size and every decision bit-exact against the oracle's PD replay."""
    tr = trace.make_trace(30, 200, 80, 512, seed=6, dist="uniform")
    L, Hq, Hkv, d, P = 2, 8, 2, 128, 16
    cap_pages = 60
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(dict(prior=dict(n=8, mean_in=100.0, mean_out=40.0), trace=dict(dist="uniform")))
    b_max = 64
    # static b = 64 over-commits the 60-page cap: LIFO preemption and recompute through the model
    kw = dict(policy=opol.STATIC, b_static=b_max, b_min=1, b_max=b_max, b0=8, eps_m=0.02, bytes_per_token=beta,
              page_size=P, refresh_steps=5, w_len=16, w_sla=4, alpha=4, delta=1, d_sla_ms=50.0, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    max_req = b_max + 2
    maxp = -(-int((tr.l_in + tr.l_out).max()) // P) + 1
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, max_req, maxp, "f16")
    model = dbk.Model(pool, 512, 512, 300, max_pos=maxp * P, weight_seed=5)
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=17, out_dtype=2, pd_fusion=True)
    eng.attach_model(model)
    qd = torch.empty(L, max_req, Hq, d, dtype=torch.float16, device="cuda")
    od = torch.empty(L, max_req, Hq, d, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P, pd=True,
                                      max_rows=max_req)], opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    recs = []
    while not eng.done():
        g = eng.step(bufs)
        recs.append(g)
        o = rp.step(g["step_ns"])
        for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx", "used_pages",
                  "rationale", "n_prefill"):
            assert g[k] == o[k], (k, g[k], o[k])
        assert (g["table_hash"] & ((1 << 64) - 1)) == o["table_hash"]
    assert rp.done()
    assert sum(r["n_prefill"] for r in recs) >= int(tr.l_in.sum())
    assert sum(r["n_preempted"] for r in recs) > 0      # the 60-page cap forces recompute through the model
    eng.close()
    model.close()
    pool.close()


def test_model_explicit_tokens_and_greedy_sampling(dbk):
    """Caller-provided input tokens for the decode rows (dbk_model_step_pd tokens) and greedy
    sampling (sampled): logits vs O8 with the same token ids; every sample is a valid argmax
    of the oracle's logits (ties within the fp16 path's rounding, R35) and, bit for bit, the
    lowest-index argmax of the returned logits."""
    s = om.ModelShape(layers=2, q_heads=8, kv_heads=4, head_dim=64, hidden=512, ffn=512, vocab=32000)
    kv_seed, wseed = 12, 13
    ctx = [3, 40, 111]
    pool, model, ids, ref = _setup(dbk, s, ctx, kv_seed, wseed)
    pool.reserve_tokens(ids, [1] * len(ids))
    toks = [31999, 0, 12345]
    tk = torch.tensor(toks, dtype=torch.int32, device="cuda")
    smp = torch.full((len(ids),), -1, dtype=torch.int32, device="cuda")
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step_pd(ids, [], [], [], logits, tokens=tk, sampled=smp)
    want, _, _, _ = om.decode_step(s, wseed, kv_seed, ids, ctx, tokens=toks)
    got = logits.cpu().numpy()
    assert row_err(got, want, "logits_tokens") <= MODEL_TOL
    sm = smp.cpu().numpy()
    for i in range(len(ids)):
        assert sm[i] == int(np.argmax(got[i]))
        assert om.greedy_ok(want[i], int(sm[i]), MODEL_TOL)
    model.close()
    pool.close()


def test_engine_model_end_to_end_tokens(dbk):
    """The engine in full-model mode with host_tokens: each step reads the decode rows' token
    ids from the caller's pinned array and writes their greedy samples back (4 B per row each
    way).  The first decode step (synthetic history only) is checked against O8 with the
    caller's initial tokens; every decision replays bit-exactly."""
    c = configs.CONFIGS["toy"]
    tr = trace.make_trace(8, 40, 20, 128, seed=2, dist="uniform")
    L, Hq, Hkv, d, V = 2, 8, 8, 64, 700
    s = om.ModelShape(layers=L, q_heads=Hq, kv_heads=Hkv, head_dim=d, hidden=512, ffn=512, vocab=V)
    cap_pages = 256
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(c)
    kw = dict(policy=opol.STATIC, b_static=8, b_min=1, b_max=8, b0=8, eps_m=0.02, bytes_per_token=beta,
              page_size=P, refresh_steps=5, w_len=16, w_sla=4, alpha=4, delta=1, d_sla_ms=50.0, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, 10, 16, "f16")
    model = dbk.Model(pool, 512, 512, V, max_pos=256, weight_seed=9)
    seed = 31
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=seed, out_dtype=2)
    eng.attach_model(model)
    qd = torch.empty(L, 10, Hq, d, dtype=torch.float16, device="cuda")
    od = torch.empty(L, 10, Hq, d, dtype=torch.float32, device="cuda")
    host_tok = torch.tensor([(7 * i + 3) % V for i in range(len(tr))], dtype=torch.int32).pin_memory()
    init = host_tok.clone().numpy()
    bufs = eng.buffers(qd, od, host_tokens=host_tok)
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P)],
                     opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    first = True
    while not eng.done():
        g = eng.step(bufs)
        o = rp.step(g["step_ns"])
        for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx", "used_pages"):
            assert g[k] == o[k], (k, g[k], o[k])
        assert g["h2d_bytes"] == 4 * g["n_decode"] and g["d2h_bytes"] == 4 * g["n_decode"]
        if first and g["n_decode"]:
            bid, bctx = eng.last_batch()
            # the step's logits are in the model's internal buffer; recompute the samples' validity
            want, _, _, _ = om.decode_step(s, 9, seed, [int(r) for r in bid], [int(x) for x in bctx],
                                           tokens=[int(init[int(r)]) for r in bid])
            samples = host_tok.numpy()[[int(r) for r in bid]]
            for i in range(len(bid)):
                assert om.greedy_ok(want[i], int(samples[i]), MODEL_TOL)
            first = False
    assert rp.done() and not first
    assert np.all((host_tok.numpy() >= 0) & (host_tok.numpy() < V))
    eng.close()
    model.close()
    pool.close()


def test_model_edge_cases(dbk):
    """Empty step, too many rows, positions past the RoPE table, unsupported configs."""
    s = om.ModelShape(layers=1, q_heads=4, kv_heads=4, head_dim=64, hidden=256, ffn=256, vocab=100)
    pool, model, ids, ref = _setup(dbk, s, [5, 9], 1, 2)
    model.step([])                                     # n = 0: no-op
    pool.reserve_tokens(ids, [1, 1])
    with pytest.raises(dbk.DbkError):                  # a chunk of 3 rows + 2 decode rows > 4 slots
        pool.request_begin(77, 3, 1)
        pool.reserve_tokens([77], [3])
        model.step_pd(ids, [77], [0], [3])
    model.close()
    pool.close()
    pool = dbk.KVPool(1, 4, 4, 64, 16, 4, 8, "f16")
    small = dbk.Model(pool, 256, 256, 100, max_pos=8, weight_seed=1)
    pool.request_begin(1, 8, 8)
    pool.append_tokens([1], [8], seed=1)
    pool.reserve_tokens([1], [1])                      # position 8 >= max_pos
    with pytest.raises(dbk.DbkError):
        small.step([1])
    small.close()
    pool.close()
    bpool = dbk.KVPool(1, 4, 4, 64, 16, 4, 8, "bf16")
    with pytest.raises(dbk.DbkError):                  # the model path is fp16
        dbk.Model(bpool, 256, 256, 100)
    bpool.close()
    fpool = dbk.KVPool(1, 4, 4, 64, 16, 4, 8, "f16")
    with pytest.raises(dbk.DbkError):                  # hidden must be a multiple of 128
        dbk.Model(fpool, 200, 256, 100)
    fpool.close()


def test_model_step_split_k_epilogues(dbk):
    """A model whose projections have few weight tiles for their depth (QKV 5120 rows, gate|up
    2048, LM head 1000, at K = 4096): the GEMM splits K for the RoPE / KV-write, SwiGLU and fp32
    epilogues (partials reduce-added into the runner's fp32 workspace, the tile's segments read
    back and finish a share of its chunks each); two steps, the second attending to the K/V the
    first wrote through the split RoPE epilogue."""
    s = om.ModelShape(layers=2, q_heads=32, kv_heads=4, head_dim=128, hidden=4096, ffn=1024, vocab=1000)
    kv_seed, wseed = 9, 10
    ctx = [3, 40, 129, 300, 17]
    pool, model, ids, ref = _setup(dbk, s, ctx, kv_seed, wseed)
    pool.reserve_tokens(ids, [1] * len(ids))
    logits = torch.empty(len(ids), s.vocab, dtype=torch.float32, device="cuda")
    model.step(ids, logits)
    want, nk, nv, _ = om.decode_step(s, wseed, kv_seed, ids, ctx)
    assert row_err(logits.cpu().numpy(), want, "logits_split") <= MODEL_TOL
    for lay in range(s.layers):
        for i, (r, c) in enumerate(zip(ids, ctx)):
            k, v = _read_kv(pool, s, r, c - 1, lay)
            assert row_err(k, nk[lay, i], "k_split") <= MODEL_TOL and row_err(v, nv[lay, i], "v_split") <= MODEL_TOL
    written = {(r, c - 1, lay): (nk[lay, i], nv[lay, i]) for i, (r, c) in enumerate(zip(ids, ctx))
               for lay in range(s.layers)}
    pool.reserve_tokens(ids, [1] * len(ids))
    model.step(ids, logits)
    want2, _, _, _ = om.decode_step(s, wseed, kv_seed, ids, [c + 1 for c in ctx], kv_written=written)
    assert row_err(logits.cpu().numpy(), want2, "logits_split_step2") <= MODEL_TOL
    model.close()
    pool.close()


def test_engine_rejects_a_foreign_model_and_duplicate_trace_ids(dbk):
    """dbk_engine_attach_model: the model's QKV epilogue writes K/V into its OWN pool's pages, so
    a model created on another pool is EINVAL; dbk_engine_create: request ids name pool entries,
    so a trace naming one twice is EINVAL up front (it used to collide mid-run)."""
    pool_a = dbk.KVPool(1, 4, 4, 64, 64, 8, 8, "f16")
    pool_b = dbk.KVPool(1, 4, 4, 64, 64, 8, 8, "f16")
    sched = dbk.Scheduler(policy=1, b_max=8, bytes_per_token=2 * 4 * 64 * 2, page_size=16)
    arr, lin, lout = [0, 0, 0], [4, 5, 6], [3, 3, 3]
    eng = dbk.Engine(pool_a, sched, arr, lin, lout, 64 * 16 * 2 * 4 * 64 * 2)
    model_b = dbk.Model(pool_b, 256, 512, 128, max_pos=64)
    with pytest.raises(dbk.DbkError) as e:
        eng.attach_model(model_b)
    assert e.value.status == dbk._lib.DBK_EINVAL
    with pytest.raises(dbk.DbkError) as e:
        dbk.Engine(pool_a, sched, arr, lin, lout, 64 * 16 * 2 * 4 * 64 * 2, req_ids=[5, 9, 5])
    assert e.value.status == dbk._lib.DBK_EINVAL
    for o in (model_b, eng, pool_a, pool_b):
        if hasattr(o, "close"):
            o.close()
