"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element.

Bars (R23): block tables, KV-token counts, statistics and
every scheduling decision bit-exact; attention rows within 2e-3 relative (fp32
out).  The oracle's inputs come only from synth/ and oracle/ -- never from the GPU."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import attention as oatt  # noqa: E402
from oracle import engine as oeng  # noqa: E402
from oracle import policy as opol  # noqa: E402
from oracle import stats as ostats  # noqa: E402
from oracle.allocator import PagedKV  # noqa: E402
from synth import configs, hashgen, trace  # noqa: E402

TOL = 2e-3


@pytest.fixture(scope="module")
def dbk():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import paper_2503_05248_b200 as m
    return m


def row_err(got, want):
    return (np.abs(got - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)).max()


def dt_name(kv_dtype):
    return "f16" if kv_dtype == 0 else "bf16"


def torch_from_bits(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda()


def run_decode_case(dbk, L, Hq, Hkv, d, dtype, ctx_list, seed=7, explicit_kv=False, cap=None,
                    layer=None, q_scale_log2=0, chunk_pages=None, out_dtype=2, monkeypatch=None, multi_layer=False):
    P = 16
    n = len(ctx_list)
    ctx = np.asarray(ctx_list, np.int32)
    l_in = np.maximum(1, ctx - 3)
    l_out = np.maximum(1, ctx - l_in + np.arange(n) % 2)   # odd entries are not finishing
    max_pages = int(max(-(-(ctx + 1) // P))) + 1
    cap = cap or int(sum(-(-ctx // P))) + 7
    pool = dbk.KVPool(L, Hq, Hkv, d, cap, n + 3, max_pages, dtype)
    ref = PagedKV(cap, P)
    ids = np.arange(n, dtype=np.int64) * 7919 + 11
    for r, a, b in zip(ids, l_in, l_out):
        pool.request_begin(r, a, b)
        ref.begin(int(r))
    # append in two rounds (prefill-like then decode-like) to exercise page growth
    first = np.maximum(1, ctx // 2)
    for part in (first, ctx - first):
        if explicit_kv:
            rows_k, rows_v = [], []
            for r, c0, k in zip(ids, [ref.ctx[int(r)] for r in ids], part):
                pos = np.arange(c0, c0 + k)[:, None, None]
                lay = np.arange(L)[None, :, None]
                hd = np.arange(Hkv)[None, None, :]
                rows_k.append(hashgen.to_bits(hashgen.gen_values(seed, 1, int(r), pos, lay, hd, d), dtype))
                rows_v.append(hashgen.to_bits(hashgen.gen_values(seed, 2, int(r), pos, lay, hd, d), dtype))
            kt = torch_from_bits(np.concatenate(rows_k)) if sum(part) else None
            vt = torch_from_bits(np.concatenate(rows_v)) if sum(part) else None
            if kt is None:
                pool.append_tokens(ids, part, seed=seed)
            else:
                pool.append_tokens(ids, part, kt, vt)
        else:
            pool.append_tokens(ids, part, seed=seed)
        ref.append([int(r) for r in ids], [int(x) for x in part])
    # block tables and counts: bit-exact
    bt_dev = pool.block_table()
    for r in ids:
        c, slot, pages = pool.request_info(r)
        assert c == ref.ctx[int(r)] and pages == ref.pages[int(r)]
        row = bt_dev[slot]
        assert list(row[:len(pages)]) == pages and np.all(row[len(pages):] == -1)
    layers = [layer] if layer is not None else list(range(L))
    results = []
    if multi_layer:  # every layer through dbk_decode_step_layers (q / out [L][n][Hq][d])
        odt = {2: torch.float32, 0: torch.float16, 1: torch.bfloat16}[out_dtype]
        qb_all = np.stack([hashgen.to_bits(np.stack([hashgen.gen_values(seed, 0, int(r), int(c) - 1, lay,
                                                                        np.arange(Hq), d, q_scale_log2)
                                                     for r, c in zip(ids, ctx)]), dtype) for lay in range(L)])
        q_all = torch_from_bits(qb_all)
        out_all = torch.full((L, n, Hq, d), float("nan"), dtype=odt, device="cuda")
        launches = pool.decode_step_layers(ids, 0, L, q_all, n * Hq * d, out_all, n * Hq * d, out_dtype=out_dtype,
                                           fuse_stats=True)
        st = pool.batch_stats()
        assert st == ostats.batch_stats(ctx, l_in, l_out, [ref.pages[int(r)] for r in ids], P, cap)
        for lay in range(L):
            bt, pk, pv, qq = oatt.synth_paged_batch(seed, [int(r) for r in ids], ctx,
                                                    [ref.pages[int(r)] for r in ids], lay, Hq, Hkv, d, P,
                                                    dtype, q_scale_log2=q_scale_log2, n_phys=cap)
            want = oatt.paged_decode_attention(ctx, bt, pk, pv, qq, dtype, nthreads=8)
            results.append((out_all[lay].float().cpu().numpy().astype(np.float64), want))
        LAST_INFO.clear()
        LAST_INFO.update(pool.info(), launches=launches)
        pool.close()
        return results
    for lay in layers:
        qv = np.stack([hashgen.gen_values(seed, 0, int(r), int(c) - 1, lay, np.arange(Hq), d, q_scale_log2)
                       for r, c in zip(ids, ctx)])
        qb = hashgen.to_bits(qv, dtype)
        q = torch_from_bits(qb)
        out = torch.empty(n, Hq, d, dtype={2: torch.float32, 0: torch.float16, 1: torch.bfloat16}[out_dtype],
                          device="cuda")
        pool.decode_step(ids, lay, q, out, out_dtype=out_dtype, fuse_stats=(lay == layers[0]))
        st = pool.batch_stats()
        exp = ostats.batch_stats(ctx, l_in, l_out, [ref.pages[int(r)] for r in ids], P, cap)
        assert st == exp
        bt, pk, pv, qq = oatt.synth_paged_batch(seed, [int(r) for r in ids], ctx,
                                                [ref.pages[int(r)] for r in ids], lay, Hq, Hkv, d, P,
                                                dtype, q_scale_log2=q_scale_log2, n_phys=cap)
        assert np.array_equal(qq, qb)
        want = oatt.paged_decode_attention(ctx, bt, pk, pv, qq, dtype, nthreads=8)
        got = out.float().cpu().numpy().astype(np.float64)
        results.append((got, want))
    LAST_INFO.clear()
    LAST_INFO.update(pool.info())
    pool.close()
    return results


LAST_INFO = {}


def test_device_generator_matches_host_generator(dbk):
    seed = 99
    req = np.array([0, 5, 1 << 40, 12345678901], np.int64)
    pos = np.array([0, 17, 4095, 2 ** 31 - 1], np.int32)
    for kind in (0, 1, 2):
        for scale in (0, 4):
            out = torch.empty(4, 6, 128, dtype=torch.float32, device="cuda")
            dbk.synth_fill(seed, kind, req, pos, 3, 6, 128, out, scale_log2=scale, dtype=2)
            want = hashgen.gen_values(seed, kind, req[:, None], pos[:, None], 3, np.arange(6)[None, :], 128, scale)
            assert np.array_equal(out.cpu().numpy().astype(np.float64), want)
    for dt, name in ((0, "f16"), (1, "bf16")):
        out = torch.empty(4, 6, 64, dtype=torch.int16, device="cuda")
        dbk.synth_fill(seed, 1, req, pos, 0, 6, 64, out, dtype=dt)
        want = hashgen.to_bits(hashgen.gen_values(seed, 1, req[:, None], pos[:, None], 0, np.arange(6)[None, :], 64), name)
        assert np.array_equal(out.cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("Hq,Hkv,d", [(8, 8, 64), (4, 4, 128), (8, 2, 64), (16, 2, 128), (8, 4, 128)])
def test_decode_parity_shapes(dbk, dtype, Hq, Hkv, d):
    rng = np.random.default_rng(Hq * 100 + d)
    ctx = [1, 2, 15, 16, 17, 31, 32, 33] + list(rng.integers(1, 700, 6)) + [1500, 4100]
    for got, want in run_decode_case(dbk, 2, Hq, Hkv, d, dtype, ctx):
        assert row_err(got, want) <= TOL


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_decode_parity_explicit_kv_and_peaked_q(dbk, dtype):
    ctx = [3, 40, 129, 600, 1025]
    for got, want in run_decode_case(dbk, 3, 8, 8, 64, dtype, ctx, explicit_kv=True, q_scale_log2=4):
        assert row_err(got, want) <= TOL


def test_decode_parity_toy_config(dbk):
    c = configs.CONFIGS["toy"]
    tr = trace.make_trace(c["n_requests"], **c["trace"])
    ctx = list(tr.l_in + tr.l_out)
    for got, want in run_decode_case(dbk, 1, 8, 8, 64, "f16", ctx, cap=256):
        assert row_err(got, want) <= TOL


def test_decode_output_dtypes(dbk):
    ctx = [5, 77, 300]
    for od in (0, 1):
        for got, want in run_decode_case(dbk, 1, 8, 8, 128, "f16", ctx, out_dtype=od):
            # output rounding adds at most half an ulp of the output format
            ulp = 2.0 ** -11 if od == 0 else 2.0 ** -8
            assert row_err(got, want) <= TOL + ulp


def test_decode_chunking_is_invariant(dbk, monkeypatch):
    outs = []
    for cp in (4, 16, 64):
        monkeypatch.setenv("DBK_CHUNK_PAGES", str(cp))
        (got, want), = run_decode_case(dbk, 1, 8, 2, 128, "bf16", [2000, 700, 16, 4096], layer=0)
        assert row_err(got, want) <= TOL
        outs.append(got)
    assert max(row_err(o, outs[0]) for o in outs) < 1e-5


@pytest.mark.parametrize("dtype,Hq,Hkv,d,per_launch", [("f16", 8, 8, 64, None), ("bf16", 16, 2, 128, None),
                                                        ("f16", 8, 1, 128, 2), ("bf16", 8, 4, 64, 1)])
def test_decode_step_layers_matches_per_layer(dbk, monkeypatch, dtype, Hq, Hkv, d, per_launch):
    """dbk_decode_step_layers (tasks spanning the layers, one launch -- or several PDL-chained
    ones when the layers per launch are capped) vs O1 and vs one dbk_decode_step per layer (the
    chunk size, hence the split-K order, may differ: equal to 1e-5); the statistics record is
    exact."""
    L = 5
    ctx = [1, 16, 17, 300, 700, 2100, 4100, 33, 2, 1000]
    if per_launch:
        monkeypatch.setenv("DBK_LAYERS_PER_LAUNCH", str(per_launch))
    multi = run_decode_case(dbk, L, Hq, Hkv, d, dtype, ctx, multi_layer=True, q_scale_log2=2)
    launches = LAST_INFO["launches"]
    assert launches == (1 if not per_launch else -(-L // per_launch))
    monkeypatch.delenv("DBK_LAYERS_PER_LAUNCH", raising=False)
    single = run_decode_case(dbk, L, Hq, Hkv, d, dtype, ctx, q_scale_log2=2)
    for (gm, want), (gs, _) in zip(multi, single):
        assert row_err(gm, want) <= TOL
        assert row_err(gm, gs) < 1e-5


def test_append_cap_is_all_or_nothing(dbk):
    pool = dbk.KVPool(1, 8, 8, 64, 4, 4, 8, "f16")
    pool.request_begin(1, 10, 10)
    pool.request_begin(2, 10, 10)
    pool.append_tokens([1, 2], [17, 16])
    with pytest.raises(dbk.DbkError) as e:
        pool.append_tokens([1, 2], [16, 17])
    assert e.value.status == dbk._lib.DBK_ECAP
    assert pool.usage() == (3, 1)
    assert pool.request_info(1)[0] == 17 and pool.request_info(2)[0] == 16
    pool.release([1])
    assert pool.usage() == (1, 3)
    bt = pool.block_table()
    assert np.all(bt[0] == -1)
    with pytest.raises(dbk.DbkError):
        pool.request_begin(3, 40, 40)    # ceil(80/16) = 5 pages > cap 4: fatal
    pool.close()


# ------------------------------------------------------------------ engine replay
def _engine_vs_replay(dbk, cfgname, n_req=None, policy=None, sla_ms=None, tr=None, cap_pages=None,
                      layers=None, check_attention_every=0, dtype="f16", swap_pages=0):
    c = dict(configs.CONFIGS[cfgname])
    if tr is None:
        t = c["trace"]
        tr = trace.make_trace(n_req or c["n_requests"], t["mean_in"], t["mean_out"], t["L_max"], t["seed"],
                              dist=t["dist"])
    L = layers or c["layers"]
    Hq, Hkv, d, P = c["q_heads"], c["kv_heads"], c["head_dim"], c["page_size"]
    cap_pages = cap_pages or c["cap_tokens"] // P
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(c)
    kw = dict(policy=policy if policy is not None else opol.MEMORY, b_static=c["b_max"], b_min=c["b_min"],
              b_max=c["b_max"], b0=c["b_min"], eps_m=c["eps_m"], bytes_per_token=beta, page_size=P,
              refresh_steps=5, w_len=16, w_sla=4, alpha=4, delta=1, d_sla_ms=sla_ms or 50.0, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    max_req = c["b_max"] + 2
    maxp = -(-c["trace"]["L_max"] // P)
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, max_req, maxp, dtype)
    seed = 31
    if swap_pages:  # swap preemption (R29-R31): pinned host swap space of swap_pages pages
        assert pool.swap_space_attach(torch.empty(swap_pages * L * Hkv * 2 * P * d * 2, dtype=torch.uint8,
                                                  pin_memory=True)) == swap_pages
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=seed, out_dtype=2,
                     preempt_mode=1 if swap_pages else 0)
    et = torch.float16 if dtype == "f16" else torch.bfloat16
    qd = torch.empty(L, max_req, Hq, d, dtype=et, device="cuda")
    od = torch.empty(L, max_req, Hq, d, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    recs = []
    ids = list(range(len(tr)))
    rp = oeng.Replay([oeng.RankEngine(ids, tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P,
                                      swap_cap_pages=swap_pages)],
                     opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    checked = 0
    while not eng.done():
        g = eng.step(bufs)
        recs.append(g)
        o = rp.step(g["step_ns"])
        for k in ("t", "clock_ns", "b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished",
                  "sum_ctx", "used_pages", "rationale", "n_swap_out", "n_swap_in"):
            assert g[k] == o[k], (k, g, {kk: o[kk] for kk in g if kk in o})
        assert (g["table_hash"] & ((1 << 64) - 1)) == o["table_hash"]
        assert g["n_waiting"] == o["stats"]["n_waiting"]
        if check_attention_every and g["t"] % check_attention_every == 0 and g["n_decode"]:
            rs, ctx, li, lo, pages = o["batches"][0]
            bid, bctx = eng.last_batch()
            assert list(bid) == rs and list(bctx) == ctx
            n = len(rs)
            remap = {p: i for i, p in enumerate(sorted({x for pg in pages for x in pg}))}
            cp = [[remap[x] for x in pg] for pg in pages]
            lay = g["t"] % L
            bt, pk, pv, qq = oatt.synth_paged_batch(seed, rs, ctx, cp, lay, Hq, Hkv, d, P, dtype)
            want = oatt.paged_decode_attention(ctx, bt, pk, pv, qq, dtype, nthreads=8)
            got = od[lay, :n].cpu().numpy().astype(np.float64)
            assert row_err(got, want) <= TOL
            checked += 1
    assert rp.done()
    assert sum(r["n_finished"] for r in recs) == len(tr)
    if swap_pages:
        assert pool.swap_usage()[0] == 0
    pool.close()
    return recs, checked


def test_engine_toy_memory_policy_replays_bit_exact(dbk):
    recs, checked = _engine_vs_replay(dbk, "toy", check_attention_every=3)
    assert checked > 0
    assert max(r["b_t"] for r in recs) == 8        # b_quad = 27 clamps to B_max (non-binding)


def test_engine_toy_tight_preempts_and_replays(dbk):
    c = configs.CONFIGS["toy-tight"]
    tr = trace.make_trace(40, 128, 128, 256, seed=1, dist="uniform")
    # static b = 8 over-commits the 64-page cap: exercises LIFO preemption + recompute
    recs, _ = _engine_vs_replay(dbk, "toy-tight", tr=tr, policy=opol.STATIC, check_attention_every=7)
    assert sum(r["n_preempted"] for r in recs) > 0
    recs, _ = _engine_vs_replay(dbk, "toy-tight", tr=tr, policy=opol.MEMORY)
    assert all(r["used_pages"] <= c["cap_tokens"] // 16 for r in recs)


def test_engine_combined_sla_poisson_replays(dbk):
    tr = trace.make_trace(60, 100, 100, 256, seed=5, dist="uniform", arrival="poisson", rate_qps=400.0)
    recs, checked = _engine_vs_replay(dbk, "toy", tr=tr, policy=opol.COMBINED, sla_ms=0.05,
                                      check_attention_every=5, dtype="bf16")
    assert checked > 0
    assert any(r["rationale"] == opol.R_SLA for r in recs) or any(r["rationale"] == opol.R_MEMORY for r in recs)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("Hq,Hkv,d", [(8, 2, 64), (16, 2, 128), (8, 4, 128), (16, 8, 64)])
@pytest.mark.parametrize("path", ["tensor", "tensor_tma2d", "cuda_core"])
def test_gqa_paths_parity(dbk, monkeypatch, dtype, Hq, Hkv, d, path):
    """K2 (TMA tensor tiles + mma.sync; one 5-D box per tile, or 2-D boxes) and K1 (CUDA
    cores) on the same GQA inputs."""
    monkeypatch.delenv("DBK_GQA_CUDA_CORE", raising=False)
    monkeypatch.delenv("DBK_GQA_TMA2", raising=False)
    if path == "cuda_core":
        monkeypatch.setenv("DBK_GQA_CUDA_CORE", "1")
    elif path == "tensor_tma2d":
        monkeypatch.setenv("DBK_GQA_TMA2", "1")
    ctx = [1, 5, 16, 17, 100, 255, 256, 257, 1024, 3000]
    for got, want in run_decode_case(dbk, 2, Hq, Hkv, d, dtype, ctx, q_scale_log2=(4 if Hq == 16 else 0)):
        assert row_err(got, want) <= TOL
    assert LAST_INFO["decode_path"] == (1 if path == "cuda_core" else 2)
    if path != "cuda_core":
        assert LAST_INFO["tma_rank"] == (2 if path == "tensor_tma2d" else 5)


def test_nccl_single_rank_allgather(dbk):
    """The native NCCL exchange path (dbk_comm_*) with one rank on cuda:0."""
    import ctypes
    buf = (ctypes.c_char * 128)()
    dbk._lib.dbk_comm_unique_id(buf)
    comm = ctypes.c_void_p()
    dbk._lib.dbk_comm_create(1, 0, buf, 0, ctypes.byref(comm))
    rec = dict.fromkeys(dbk._lib.STATS_FIELDS, 0)
    rec.update(n_active=7, sum_ctx=99, step_ns=1234, n_finished=2)
    local = dbk.dbk_stats(*[rec[f] for f in dbk._lib.STATS_FIELDS])
    allr = (dbk.dbk_stats * 1)()
    glob = dbk.dbk_stats()
    stream = torch.cuda.current_stream().cuda_stream
    dbk._lib.dbk_stats_allgather(comm, ctypes.byref(local), allr, ctypes.byref(glob), 0, stream)
    assert allr[0].as_dict() == rec and glob.as_dict()["sum_ctx"] == 99 and glob.as_dict()["step_ns"] == 1234
    dbk._lib.dbk_comm_destroy(comm)


def test_bench_config_sampled_parity(dbk):
    """The bench's own launch configuration (Llama-2-7B shape, pool sized from free HBM,
    memory policy): run engine steps, then compare sampled (request, q-head, layer)
    outputs of the last step with the oracle computed from logical coordinates."""
    import gc

    import bench
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(device=0, time_attention=True, out_dtype=2, n_req=1200)
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    recs = [eng.step(bufs, stream) for _ in range(40)]
    rec = recs[-1]
    torch.cuda.synchronize()
    _replay_full_size(S, recs)
    c = S["c"]
    L, Hq, Hkv, d, P = c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["page_size"]
    ids, ctx = eng.last_batch()
    assert rec["n_decode"] == len(ids) and rec["sum_ctx"] == int(ctx.sum())
    rng = np.random.default_rng(5)
    sel = rng.choice(len(ids), size=12, replace=False)
    for lay in (0, L // 2, L - 1):
        pages, nxt = [], 0
        for cx in ctx[sel]:
            m = -(-int(cx) // P)
            pages.append(list(range(nxt, nxt + m)))
            nxt += m
        bt, pk, pv, qq = oatt.synth_paged_batch(S["seed"], [int(x) for x in ids[sel]], ctx[sel], pages, lay,
                                                Hq, Hkv, d, P, "f16")
        want = oatt.paged_decode_attention(ctx[sel], bt, pk, pv, qq, "f16", nthreads=8)
        got = S["od"][lay, torch.as_tensor(sel, device="cuda")].cpu().numpy().astype(np.float64)
        assert row_err(got, want) <= TOL
    _free(S)


def _free(S):
    """Release a full-size pool (~160 GB) before the next full-size test."""
    import gc
    S["eng"].close()
    S["pool"].close()
    S.clear()
    gc.collect()
    torch.cuda.empty_cache()


def _replay_full_size(S, recs):
    """Oracle replay (O7) of a full-size GPU engine run from its logged step times: every
    scheduling decision, admission/preemption count, token count, page count and block-table
    checksum must agree bit for bit."""
    import bench
    c, tr, P = S["c"], S["tr"], S["c"]["page_size"]
    kw = bench.sched_kwargs(c, S["beta"], S.get("policy"), 256, S.get("sla_ms"))
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, S["cap_pages"], P)],
                     opol.SchedConfig(**kw), S["mem_cap_total"])
    for g in recs:
        o = rp.step(g["step_ns"])
        for k in ("t", "clock_ns", "b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished",
                  "sum_ctx", "used_pages", "rationale"):
            assert g[k] == o[k], (k, g[k], o[k], g["t"])
        assert (g["table_hash"] & ((1 << 64) - 1)) == o["table_hash"]


def test_sla_binding_full_size_replay(dbk):
    """13B shape, combined policy with a binding SLA (D below the memory-bound step time):
    the device-timed step latencies drive Alg. 2 and the oracle replays the decisions."""
    import gc

    import bench
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(device=0, cfg_name="llama2-13b-sla", time_attention=False, out_dtype=0,
                           n_req=800, sla_ms=6.0)
    S["policy"], S["sla_ms"] = None, 6.0
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    recs = [eng.step(bufs, stream) for _ in range(120)]
    _replay_full_size(S, recs)
    assert any(r["rationale"] == opol.R_SLA for r in recs)       # the SLA search bound the batch
    # (running requests are never evicted by the SLA rule -- Alg. 2 line 16 clamps b >= N^d --
    # so the step time only falls as they finish; the replay above checks every decision)
    _free(S)


@pytest.mark.parametrize("tp", [1, 8])
def test_gqa_bench_config_sampled_parity(dbk, tp):
    """The 70B GQA bench launch configuration (K2 on tensor cores, 120 GB per-GPU cap, batch
    up to 1024; tp = 8: rank 0's KV-head shard, 8 q-heads of 1 kv head): decisions replayed
    bit-exactly, then sampled (request, layer) outputs of the last step vs the oracle from
    logical coordinates."""
    import gc

    import bench
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(device=0, cfg_name="llama3-70b-gqa", time_attention=True, out_dtype=2, n_req=2000,
                           tp=tp)
    assert S["pool"].info()["decode_path"] == 2
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    recs = [eng.step(bufs, stream) for _ in range(30)]
    torch.cuda.synchronize()
    _replay_full_size(S, recs)
    L, Hq, Hkv, d, P = S["L"], S["Hq"], S["Hkv"], S["d"], 16
    ids, ctx = eng.last_batch()
    assert recs[-1]["n_decode"] == len(ids) and len(ids) > 500
    rng = np.random.default_rng(7)
    sel = rng.choice(len(ids), size=8, replace=False)
    for lay in (0, L - 1):
        pages, nxt = [], 0
        for cx in ctx[sel]:
            m = -(-int(cx) // P)
            pages.append(list(range(nxt, nxt + m)))
            nxt += m
        bt, pk, pv, qq = oatt.synth_paged_batch(S["seed"], [int(x) for x in ids[sel]], ctx[sel], pages, lay,
                                                Hq, Hkv, d, P, "f16")
        want = oatt.paged_decode_attention(ctx[sel], bt, pk, pv, qq, "f16", nthreads=8)
        got = S["od"][lay, torch.as_tensor(sel, device="cuda")].cpu().numpy().astype(np.float64)
        assert row_err(got, want) <= TOL
    _free(S)


def test_bench_config_whole_trace_replay(dbk):
    """The bench's 7B launch configuration run to completion (3 000 requests all at once,
    memory-aware rule, pool sized from free HBM): every one of its ~2 000 steps replayed by the
    oracle from the logged step times, bit for bit (admissions, preemptions, tokens, pages,
    block-table checksums, b_t), and every request finished."""
    import gc

    import bench
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(device=0, time_attention=False, out_dtype=0)
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    recs = []
    while not eng.done():
        recs.append(eng.step(bufs, stream))
    assert sum(r["n_finished"] for r in recs) == len(S["tr"])
    assert sum(r["n_decode"] for r in recs) == int(S["tr"].l_out.sum())
    _replay_full_size(S, recs)
    _free(S)


def test_empty_batch_is_a_noop_with_the_empty_record(dbk):
    """Degenerate case n = 0 ('n = 0 is a no-op returning DBK_OK'): no
    launch, no output written, and a stats-fused empty step reports the oracle's empty record
    (cap_pages = free_pages = cap, R28) even while requests hold pages."""
    P, cap = 16, 64
    pool = dbk.KVPool(2, 8, 8, 64, cap, 4, 8, "f16")
    ref = PagedKV(cap, P)
    pool.request_begin(5, 20, 10)
    ref.begin(5)
    pool.append_tokens([5], [21], seed=3)
    ref.append([5], [21])
    q = torch.zeros(1, 8, 64, dtype=torch.float16, device="cuda")
    out = torch.full((1, 8, 64), float("nan"), dtype=torch.float32, device="cuda")
    pool.decode_step([], 0, q, out, fuse_stats=True)
    assert pool.batch_stats() == ostats.batch_stats([], [], [], [], P, cap)
    qa = torch.zeros(2, 1, 8, 64, dtype=torch.float16, device="cuda")
    oa = torch.full((2, 1, 8, 64), float("nan"), dtype=torch.float32, device="cuda")
    assert pool.decode_step_layers([], 0, 2, qa, 8 * 64, oa, 8 * 64, fuse_stats=True) == 0
    torch.cuda.synchronize()
    assert torch.isnan(out).all() and torch.isnan(oa).all()
    assert pool.batch_stats() == ostats.batch_stats([], [], [], [], P, cap)
    # the request is untouched: a non-empty step right after matches the oracle again
    c, slot, pages = pool.request_info(5)
    assert c == 21 and pages == ref.pages[5]
    pool.decode_step([5], 1, q, out, fuse_stats=True)
    assert pool.batch_stats() == ostats.batch_stats([21], [20], [10], [ref.pages[5]], P, cap)
    pool.close()


def test_malformed_batches_are_rejected_before_any_launch(dbk):
    """A request named twice (K4 would count it twice), an unknown request, a request holding no
    tokens: DBK_EINVAL / DBK_ENOENT, nothing written; the pool stays usable."""
    pool = dbk.KVPool(1, 8, 8, 64, 32, 4, 8, "f16")
    pool.request_begin(1, 10, 10)
    pool.request_begin(2, 10, 10)
    pool.append_tokens([1], [11], seed=2)
    q = torch.zeros(2, 8, 64, dtype=torch.float16, device="cuda")
    out = torch.full((2, 8, 64), float("nan"), dtype=torch.float32, device="cuda")
    for ids, status in (([1, 1], dbk._lib.DBK_EINVAL), ([1, 9], dbk._lib.DBK_ENOENT), ([1, 2], dbk._lib.DBK_EINVAL)):
        with pytest.raises(dbk.DbkError) as e:
            pool.decode_step(ids, 0, q, out, fuse_stats=True)
        assert e.value.status == status, (ids, e.value)
    torch.cuda.synchronize()
    assert torch.isnan(out).all()
    pool.decode_step([1], 0, q[:1], out[:1], fuse_stats=True)
    assert pool.batch_stats()["n_active"] == 1
    pool.close()


def test_release_is_all_or_nothing(dbk):
    """dbk_release like append_tokens (R8): an unknown id or an id named twice releases nothing."""
    pool = dbk.KVPool(1, 8, 8, 64, 16, 4, 8, "f16")
    for r in (1, 2):
        pool.request_begin(r, 10, 10)
    pool.append_tokens([1, 2], [20, 5], seed=1)
    before = pool.usage()
    for ids, status in (([1, 7], dbk._lib.DBK_ENOENT), ([2, 2], dbk._lib.DBK_EINVAL)):
        with pytest.raises(dbk.DbkError) as e:
            pool.release(ids)
        assert e.value.status == status
        assert pool.usage() == before and pool.request_info(1)[0] == 20 and pool.request_info(2)[0] == 5
    pool.release([2, 1])
    assert pool.usage() == (0, 16)
    pool.close()


def test_decode_and_prefill_argument_checks(dbk):
    """The C-ABI's argument contract (include/dbk.h): a layer out of range, an unknown output
    dtype, misaligned q / out, a chunk outside the tokens a request holds, a request begun twice
    -- DBK_EINVAL / DBK_ENOENT, nothing launched, nothing written; the pool keeps working."""
    E = dbk._lib
    pool = dbk.KVPool(2, 8, 8, 64, 32, 4, 8, "f16")
    pool.request_begin(1, 10, 10)
    with pytest.raises(dbk.DbkError) as e:
        pool.request_begin(1, 10, 10)
    assert e.value.status == E.DBK_EINVAL
    pool.append_tokens([1], [11], seed=4)
    q = torch.zeros(1, 8, 64, dtype=torch.float16, device="cuda")
    out = torch.full((1, 8, 64), float("nan"), dtype=torch.float32, device="cuda")
    raw = torch.zeros(8 * 64 * 4 + 8, dtype=torch.uint8, device="cuda")
    q_mis = raw[2:2 + 8 * 64 * 2].view(torch.float16)   # 2-byte aligned, not 16
    bad = [lambda: pool.decode_step([1], 2, q, out),              # layer out of range
           lambda: pool.decode_step([1], -1, q, out),
           lambda: pool.decode_step([1], 0, q, out, out_dtype=3),  # no such output dtype
           lambda: pool.decode_step([1], 0, q_mis, out),           # q not 16-byte aligned
           lambda: pool.prefill_step([1], [5], [7], 0, q, out),    # chunk [5, 12) beyond the 11 tokens
           lambda: pool.prefill_step([1], [0], [0], 0, q, out),    # empty chunk
           lambda: pool.prefill_step([1], [0], [4], 2, q, out)]    # layer out of range
    for f in bad:
        with pytest.raises(dbk.DbkError) as e:
            f()
        assert e.value.status == E.DBK_EINVAL, e.value
    with pytest.raises(dbk.DbkError) as e:
        pool.prefill_step([9], [0], [1], 0, q, out)
    assert e.value.status == E.DBK_ENOENT
    torch.cuda.synchronize()
    assert torch.isnan(out).all()
    pool.decode_step([1], 1, q, out)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    pool.close()
