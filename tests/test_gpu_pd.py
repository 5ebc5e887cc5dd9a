"""GPU parity of the PD-fusion engine mode (R25-R28).

The C-ABI engine with pd_fusion = 1 is replayed step by step by oracle O7 in PD mode, driven
by the GPU's own step latencies: admissions, preemptions, decode batch, chunk sizes, block-table
hash, waiting count and every scheduling decision must agree bit-exactly; on sampled steps the
chunk's prefill attention (K7, tcgen05) is compared with O1 per query position (2e-3, R23)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import attention as oatt  # noqa: E402
from oracle import engine as oeng  # noqa: E402
from oracle import policy as opol  # noqa: E402
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


def _pd_vs_replay(dbk, tr, L, Hq, Hkv, d, cap_pages, policy, b_max, dtype="bf16", check_every=5, sla_ms=50.0,
                  pd_token_budget=0):
    P = 16
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(dict(prior=dict(n=8, mean_in=float(tr.l_in.mean()), mean_out=float(tr.l_out.mean())),
                                   trace=dict(dist="uniform")))
    kw = dict(policy=policy, b_static=b_max, b_min=1, b_max=b_max, b0=min(8, b_max), eps_m=0.02,
              bytes_per_token=beta, page_size=P, refresh_steps=5, w_len=16, w_sla=4, alpha=4, delta=1,
              d_sla_ms=sla_ms, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    max_req = b_max + 2
    maxp = -(-int((tr.l_in + tr.l_out).max()) // P) + 1
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, max_req, maxp, dtype)
    seed = 17
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=seed, out_dtype=2, pd_fusion=True,
                     pd_token_budget=pd_token_budget)
    et = torch.float16 if dtype == "f16" else torch.bfloat16
    qd = torch.empty(L, max_req, Hq, d, dtype=et, device="cuda")
    od = torch.empty(L, max_req, Hq, d, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    ids = list(range(len(tr)))
    rp = oeng.Replay([oeng.RankEngine(ids, tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P, pd=True,
                                      max_rows=max_req, pd_token_budget=pd_token_budget)],
                     opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    recs, checked = [], 0
    while not eng.done():
        g = eng.step(bufs)
        recs.append(g)
        o = rp.step(g["step_ns"])
        for k in ("t", "clock_ns", "b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished",
                  "sum_ctx", "used_pages", "rationale", "n_prefill"):
            assert g[k] == o[k], (k, g, {kk: o[kk] for kk in g if kk in o})
        assert (g["table_hash"] & ((1 << 64) - 1)) == o["table_hash"]
        assert g["n_waiting"] == o["stats"]["n_waiting"]
        if check_every and g["t"] % check_every == 0 and g["n_prefill"]:
            e = rp.ranks[0]
            ch = o["chunks"][0]
            rs = [r for r, _, _ in ch]
            ctx = [e.kv.ctx[r] for r in rs]
            pages = [list(e.kv.pages[r]) for r in rs]
            remap = {p: i for i, p in enumerate(sorted({x for pg in pages for x in pg}))}
            cp = [[remap[x] for x in pg] for pg in pages]
            lay = g["t"] % L
            bt, pk, pv, _ = oatt.synth_paged_batch(seed, rs, ctx, cp, lay, Hq, Hkv, d, P, dtype)
            qb = np.concatenate([hashgen.to_bits(hashgen.gen_values(seed, hashgen.KIND_Q, r,
                                                                    np.arange(s0, s0 + k)[:, None], lay,
                                                                    np.arange(Hq)[None, :], d), dtype)
                                 for r, s0, k in ch])
            want = oatt.paged_prefill_attention([s0 for _, s0, _ in ch], [k for _, _, k in ch], bt, pk, pv, qb,
                                                dtype, nthreads=8)
            n = g["n_decode"]
            got = od[lay, n:n + g["n_prefill"]].cpu().numpy().astype(np.float64)
            assert row_err(got, want) <= TOL
            checked += 1
    assert rp.done()
    assert sum(r["n_finished"] for r in recs) == len(tr)
    assert sum(r["n_decode"] for r in recs) == int(tr.l_out.sum())
    # per-request timeline: admitted after arrival, FCFS first admissions, finished afterwards
    adm, fin = eng.request_times()
    assert (adm >= tr.arrival_ns).all() and (fin > adm).all()
    assert (np.diff(adm) >= 0).all()
    assert fin.max() == recs[-1]["clock_ns"] + recs[-1]["step_ns"]
    pool.close()
    return recs, checked


def test_pd_engine_mha_static_replays_bit_exact(dbk):
    tr = trace.make_trace(24, 150, 40, 400, seed=4, dist="uniform", arrival="poisson", rate_qps=400.0)
    recs, checked = _pd_vs_replay(dbk, tr, 2, 8, 8, 64, 400, opol.STATIC, 96)
    assert checked > 0 and sum(r["n_prefill"] for r in recs) >= int(tr.l_in.sum())
    # the chunk rule binds: some steps fill exactly the budget b_t - N^d (prompts split across steps)
    assert any(r["n_prefill"] and r["n_prefill"] == r["b_t"] - r["n_decode"] for r in recs)


def test_pd_engine_gqa_memory_policy_with_preemption(dbk):
    tr = trace.make_trace(30, 200, 80, 512, seed=6, dist="uniform")
    recs, checked = _pd_vs_replay(dbk, tr, 1, 16, 2, 128, 60, opol.STATIC, 64, check_every=3)
    assert checked > 0
    assert sum(r["n_preempted"] for r in recs) > 0
    recs, _ = _pd_vs_replay(dbk, tr, 1, 16, 2, 128, 60, opol.MEMORY, 64, check_every=0)
    assert all(r["used_pages"] <= 60 for r in recs)


def test_pd_engine_sla_policy(dbk):
    tr = trace.make_trace(40, 100, 60, 300, seed=8, dist="uniform", arrival="poisson", rate_qps=800.0)
    recs, _ = _pd_vs_replay(dbk, tr, 2, 8, 8, 128, 600, opol.COMBINED, 64, dtype="f16", check_every=7,
                            sla_ms=0.05)
    assert len({r["b_t"] for r in recs}) > 1


def test_pd_fixed_token_budget_replays(dbk):
    """R36: a fixed iteration token budget (here 48 tokens) under the combined policy; every
    record incl. the chunk size replayed bit-exactly, chunk attention checked."""
    tr = trace.make_trace(40, 100, 60, 300, seed=8, dist="uniform", arrival="poisson", rate_qps=800.0)
    recs, checked = _pd_vs_replay(dbk, tr, 2, 8, 8, 128, 600, opol.COMBINED, 64, dtype="f16", check_every=4,
                                  sla_ms=0.3, pd_token_budget=48)
    assert checked > 0
    assert max(r["n_prefill"] + r["n_decode"] for r in recs) <= 66
