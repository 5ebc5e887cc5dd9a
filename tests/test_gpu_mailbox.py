"""The mailbox statistics exchange (SURVEY.md §8(e) "B200-native v2"; csrc/mailbox.cu) at 2 and 4
ranks: processes on one B200, each mapping the others' mailboxes through CUDA IPC -- the same
code path as peer memory over NVLink on a multi-GPU box (P2P stores, release / acquire, the
gathered records written into mapped host memory by the exchange kernel).

* standalone: random records through dbk_mbox_exchange, every rank's gathered vector equals the
  records gathered independently over gloo, the reduction equals dbk_stats_reduce;
* DP engine: dbk_engine_step exchanging through the mailbox (no caller-side exchange): every
  rank takes the same b_{t+1} and the whole run replays bit for bit in the oracle's G-rank
  Replay from the logged (device-timed, MAX over ranks) step latencies;
* TP engine (real KV-head shards): records agree across ranks every step."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _standalone(dbk, dist, rank, world):
    fields = dbk._lib.STATS_FIELDS
    mb = dbk.Mailbox(dist, world, rank, 0)
    rng = np.random.default_rng(100 + rank)
    for it in range(40):
        local = {f: int(rng.integers(0, 1 << 40)) for f in fields}
        local["over_cap"] = int(rng.integers(0, 2))
        recs, glob = mb.exchange(local, dbk._lib.MODE_DP)
        t = torch.tensor([local[f] for f in fields], dtype=torch.int64)
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t)
        want = [dict(zip(fields, x.tolist())) for x in g]
        assert recs == want, it
        assert glob == dbk.stats_reduce(want, dbk._lib.MODE_DP)
    mb.close()
    return 40


def _dp_engine(dbk, dist, rank, world):
    from oracle import engine as oeng
    from oracle import policy as opol
    from synth import trace
    tr = trace.make_trace(100, 60, 80, 256, seed=17, arrival="poisson", rate_qps=3000.0)
    L, H, d, P, cap = 2, 8, 64, 16, 40
    beta = 2 * L * H * d * 2
    kw = dict(policy=opol.COMBINED, b_min=1, b_max=40, b0=1, bytes_per_token=beta, page_size=P,
              refresh_steps=9, w_len=24, w_sla=6, alpha=4, delta=1, d_sla_ms=0.5, eps_d_ms=0.05,
              prior=(16, 16 * 60, 16 * 4800, 16 * 80, 16 * 8000))
    mem_cap = world * cap * P * beta
    pool = dbk.KVPool(L, H, H, d, cap, 48, 16, "f16")
    eng = dbk.Engine(pool, dbk.Scheduler(**kw), tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=5, out_dtype=2,
                     rank=rank, world=world)
    mb = dbk.Mailbox(dist, world, rank, 0)
    eng.attach_mbox(mb, dbk._lib.MODE_DP)
    qd = torch.empty(L, 48, H, d, dtype=torch.float16, device="cuda")
    od = torch.empty(L, 48, H, d, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    recs = []
    while not eng.done():
        recs.append(eng.step(bufs))
        x = eng.last_exchange()
        assert len(x["records"]) == world
        assert recs[-1]["step_ns"] == max(r["step_ns"] for r in x["records"]) > 0
    ids = list(range(len(tr)))
    ref = oeng.Replay([oeng.RankEngine(ids[r::world], tr.arrival_ns[ids[r::world]], tr.l_in[ids[r::world]],
                                       tr.l_out[ids[r::world]], cap, P, r, world) for r in range(world)],
                      opol.SchedConfig(**kw), mem_cap)
    for g in recs:
        w = ref.step(g["step_ns"])
        for k in ("clock_ns", "b_t", "b_next", "n_decode", "n_finished", "sum_ctx", "used_pages", "rationale"):
            assert g[k] == w[k], (rank, g["t"], k, g[k], w[k])
    assert ref.done()
    dec = torch.tensor([r["b_next"] for r in recs], dtype=torch.int64)
    allg = [torch.zeros_like(dec) for _ in range(world)]
    dist.all_gather(allg, dec)
    assert all(torch.equal(a, allg[0]) for a in allg)
    mb.close()
    pool.close()
    return len(recs)


def _tp_engine(dbk, dist, rank, world):
    from oracle import policy as opol
    from synth import trace
    tr = trace.make_trace(40, 150, 60, 1024, seed=21)
    L, HQ, HKV, D, P, cap = 2, 64 // world, 8 // world, 128, 16, 800
    beta = 2 * L * HKV * D * 2
    kw = dict(policy=opol.MEMORY, b_min=1, b_max=40, b0=1, bytes_per_token=beta, page_size=P, refresh_steps=9,
              w_len=24, prior=(16, 16 * 150, 16 * 45000, 16 * 60, 16 * 7200))
    pool = dbk.KVPool(L, HQ, HKV, D, cap, 48, 64, "f16", kv_head_offset=rank * HKV)
    eng = dbk.Engine(pool, dbk.Scheduler(**kw), tr.arrival_ns, tr.l_in, tr.l_out, cap * P * beta, seed=3,
                     out_dtype=2)
    mb = dbk.Mailbox(dist, world, rank, 0)
    eng.attach_mbox(mb, dbk._lib.MODE_TP)
    qd = torch.empty(L, 48, HQ, D, dtype=torch.float16, device="cuda")
    od = torch.empty(L, 48, HQ, D, dtype=torch.float32, device="cuda")
    bufs = eng.buffers(qd, od)
    n = 0
    for _ in range(30):
        eng.step(bufs)   # TP reduction: EINVAL (raises) if the ranks' records disagree
        n += 1
    mb.close()
    pool.close()
    return n


def _worker(kind, rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import paper_2503_05248_b200 as dbk
        torch.cuda.set_device(0)
        fn = {"standalone": _standalone, "dp": _dp_engine, "tp": _tp_engine}[kind]
        q.put((rank, "ok", fn(dbk, dist, rank, world)))
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(kind, world):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(kind, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, status, info in res:
        assert status == "ok", info
    return [info for _, _, info in res]


@pytest.mark.parametrize("world", [2, 4])
def test_mailbox_standalone_exchange(world):
    assert _run("standalone", world) == [40] * world


@pytest.mark.parametrize("world", [2, 3])
def test_mailbox_dp_engine_replays(world):
    n = _run("dp", world)
    assert len(set(n)) == 1 and n[0] > 10


def test_mailbox_tp_engine_records_agree():
    assert _run("tp", 2) == [30, 30]
