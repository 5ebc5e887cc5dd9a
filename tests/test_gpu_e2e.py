"""GPU parity of the engine's end-to-end mode (bench.py `e2e`): q and the step's new K/V rows
come from pinned host memory layer by layer (layer-major rows, one copy per layer on a copy stream, per-layer
KV append), and every layer's output goes back to pinned host memory.

The oracle side: K/V of prefilled positions from the synthetic generator, K/V of decode
positions = the host rows the test handed to the engine at that step, q = the host q rows;
O1 (`oracle.attention.paged_decode_attention`) on logical pages (paging invariance).
Decisions are replayed bit-exactly by `oracle.engine.Replay` from the logged step times."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import attention as oatt  # noqa: E402
from oracle import engine as oeng  # noqa: E402
from oracle import policy as opol  # noqa: E402
from synth import configs, hashgen, trace  # noqa: E402

TOL = 2e-3
HOST_SEED = 0x5EED


@pytest.fixture(scope="module")
def dbk():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import paper_2503_05248_b200 as m
    return m


def _rows(kind, t, n_rows, d, dtype):
    """n_rows host rows of d elements for step t (values exact in fp16 / bf16)."""
    v = hashgen.gen_values(HOST_SEED, kind, t, np.arange(n_rows), 0, 0, d)
    return hashgen.to_bits(v, dtype)


@pytest.mark.parametrize("L,Hq,Hkv,d,dtype", [(3, 8, 8, 64, "f16"), (2, 16, 2, 128, "bf16")])
def test_engine_end_to_end_mode_parity(dbk, L, Hq, Hkv, d, dtype):
    c = configs.CONFIGS["toy"]
    P = 16
    t_ = c["trace"]
    tr = trace.make_trace(8, t_["mean_in"], t_["mean_out"], t_["L_max"], t_["seed"], dist=t_["dist"])
    cap_pages = c["cap_tokens"] // P
    beta = 2 * L * Hkv * d * 2
    mem_cap = cap_pages * P * beta
    pr = configs.prior_record(c)
    kw = dict(policy=opol.MEMORY, b_static=c["b_max"], b_min=c["b_min"], b_max=c["b_max"], b0=c["b_min"],
              eps_m=c["eps_m"], bytes_per_token=beta, page_size=P, refresh_steps=5, w_len=16, w_sla=4,
              alpha=4, delta=1, d_sla_ms=50.0, eps_d_ms=0.01)
    sched = dbk.Scheduler(prior=tuple(pr.values()), **kw)
    mr = c["b_max"] + 2
    maxp = -(-t_["L_max"] // P)
    pool = dbk.KVPool(L, Hq, Hkv, d, cap_pages, mr, maxp, dtype)
    seed = 31
    eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=seed, out_dtype=2)
    et = torch.float16 if dtype == "f16" else torch.bfloat16
    qd = torch.empty(L, mr, Hq, d, dtype=et, device="cuda")
    od = torch.empty(L, mr, Hq, d, dtype=torch.float32, device="cuda")
    kvd = torch.empty(2 * mr * L * Hkv * d, dtype=et, device="cuda")
    hq = torch.empty(L * mr * Hq * d, dtype=torch.int16, pin_memory=True)
    hk = torch.empty(mr * L * Hkv * d, dtype=torch.int16, pin_memory=True)
    hv = torch.empty(mr * L * Hkv * d, dtype=torch.int16, pin_memory=True)
    ho = torch.empty(L * mr * Hq * d, dtype=torch.float32, pin_memory=True)
    bufs = eng.buffers(qd, od, kvd, hq, hk, hv, ho)
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P)],
                     opol.SchedConfig(prior=tuple(pr.values()), **kw), mem_cap)
    over = {}  # (req, pos) -> (K rows [L][Hkv][d], V rows) handed over at that decode step
    checked = 0
    t = 0
    while not eng.done():
        qb = _rows(hashgen.KIND_Q, t, L * mr * Hq, d, dtype)
        kb = _rows(hashgen.KIND_K, t, mr * L * Hkv, d, dtype)
        vb = _rows(hashgen.KIND_V, t, mr * L * Hkv, d, dtype)
        hq.copy_(torch.from_numpy(qb.view(np.int16).reshape(-1)))
        hk.copy_(torch.from_numpy(kb.view(np.int16).reshape(-1)))
        hv.copy_(torch.from_numpy(vb.view(np.int16).reshape(-1)))
        g = eng.step(bufs)
        o = rp.step(g["step_ns"])
        for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx",
                  "used_pages"):
            assert g[k] == o[k], (k, g[k], o[k])
        assert g["n_preempted"] == 0
        ids, ctx = eng.last_batch()
        n = len(ids)
        assert g["h2d_bytes"] == n * (L * Hq * d * 2 + 2 * L * Hkv * d * 2)
        assert g["d2h_bytes"] == n * L * Hq * d * 4
        kv_k = kb[:L * n * Hkv].reshape(L, n, Hkv, d)   # layer-major host rows
        kv_v = vb[:L * n * Hkv].reshape(L, n, Hkv, d)
        for x in range(n):
            over[(int(ids[x]), int(ctx[x]) - 1)] = (kv_k[:, x], kv_v[:, x])
        if n and t % 2 == 0:
            pages = [[x * maxp + p for p in range(-(-int(cx) // P))] for x, cx in enumerate(ctx)]
            got_all = ho.numpy()[:L * n * Hq * d].reshape(L, n, Hq, d).astype(np.float64)
            for lay in range(L):
                bt, pk, pv, _ = oatt.synth_paged_batch(seed, [int(r) for r in ids], [int(cx) for cx in ctx],
                                                       pages, lay, Hq, Hkv, d, P, dtype)
                for x, (r, cx) in enumerate(zip(ids, ctx)):
                    for pos in range(int(cx)):
                        if (int(r), pos) in over:
                            krow, vrow = over[(int(r), pos)]
                            pk[pages[x][pos // P], :, pos % P, :] = krow[lay]
                            pv[pages[x][pos // P], :, pos % P, :] = vrow[lay]
                qq = qb[:L * n * Hq].reshape(L, n, Hq, d)[lay]
                want = oatt.paged_decode_attention([int(cx) for cx in ctx], bt, pk, pv, qq, dtype, nthreads=8)
                err = (np.abs(got_all[lay] - want).max(axis=-1) /
                       np.maximum(np.abs(want).max(axis=-1), 1e-30)).max()
                assert err <= TOL, (t, lay, err)
            checked += 1
        t += 1
    assert rp.done()
    assert checked > 3
    pool.close()
