"""KV-head TP as real shards (BASELINE configs[3]): G processes on one B200,
rank r holding global kv heads [r*Hkv/G, (r+1)*Hkv/G) of the Llama-3-70B GQA shape (64 q / 8 kv
heads, d 128) through `dbk_pool_config.kv_head_offset`.  Every step the ranks exchange their
128-byte statistics records (gloo all-gather; TP reduction = records must agree, step_ns = MAX)
and take the same b_{t+1}; the decisions replay bit for bit in the oracle's single-rank Replay.
The G shard outputs, concatenated along the q-head axis in rank order, must equal the TP1
oracle output of the whole problem (all 64 heads) element-wise within R23's 2e-3.  (NCCL
refuses two ranks on one device, so the libdbk communicator itself is exercised at one rank in
test_gpu_parity.py; the transport does not change the records.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 2e-3
L, HQ, HKV, D, P = 3, 64, 8, 128, 16
SEED = 31


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sched_kw(beta):
    from oracle import policy as opol
    return dict(policy=opol.MEMORY, b_min=1, b_max=48, b0=1, bytes_per_token=beta, page_size=P,
                refresh_steps=9, w_len=24, prior=(16, 16 * 150, 16 * 45000, 16 * 90, 16 * 16200))


def _trace():
    from synth import trace
    return trace.make_trace(64, 150, 90, 1024, seed=13)


def _worker(rank, world, port, steps, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import paper_2503_05248_b200 as dbk
        torch.cuda.set_device(0)
        tr = _trace()
        hq, hkv = HQ // world, HKV // world
        cap = 1200
        beta = 2 * L * hkv * D * 2
        pool = dbk.KVPool(L, hq, hkv, D, cap, 56, 64, "f16", kv_head_offset=rank * hkv)
        assert pool.info()["decode_path"] == 2  # K2: tensor-core GQA (group 8)
        sched = dbk.Scheduler(**_sched_kw(beta))
        eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, cap * P * beta, seed=SEED, out_dtype=2,
                         rank=0, world=1)
        qd = torch.empty(L, 56, hq, D, dtype=torch.float16, device="cuda")
        od = torch.empty(L, 56, hq, D, dtype=torch.float32, device="cuda")
        bufs = eng.buffers(qd, od)
        fields = dbk._lib.STATS_FIELDS
        recs = []
        for _ in range(steps):
            local = eng.step_launch(bufs)
            rec = torch.tensor([local[f] for f in fields], dtype=torch.int64)
            gathered = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(gathered, rec)
            # TP: every rank serves the same requests, so the records must agree (EINVAL otherwise)
            glob = dbk.stats_reduce([dict(zip(fields, g.tolist())) for g in gathered], dbk._lib.MODE_TP)
            recs.append(eng.step_finish(glob))
        torch.cuda.synchronize()
        ids, ctx = eng.last_batch()
        n = len(ids)
        q.put((rank, "ok", dict(recs=recs, ids=ids, ctx=ctx, out=od[:, :n].cpu().numpy())))
        pool.close()
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_shards_concatenate_to_tp1(world):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import torch.multiprocessing as mp

    from oracle import attention as oatt
    from oracle import engine as oeng
    from oracle import policy as opol
    steps = 40
    ctx_ = mp.get_context("spawn")
    q = ctx_.Queue()
    port = _free_port()
    procs = [ctx_.Process(target=_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r, status, info in res:
        assert status == "ok", info
    outs = [info for _, _, info in res]
    # identical decisions on every rank, and the oracle's TP1 replay agrees bit for bit
    keys = ("t", "clock_ns", "b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx",
            "used_pages", "table_hash", "rationale")
    for o in outs[1:]:
        for a, b in zip(o["recs"], outs[0]["recs"]):
            assert all(a[k] == b[k] for k in keys)
    tr = _trace()
    beta_local = 2 * L * (HKV // world) * D * 2
    rp = oeng.Replay([oeng.RankEngine(list(range(len(tr))), tr.arrival_ns, tr.l_in, tr.l_out, 1200, P)],
                     opol.SchedConfig(**_sched_kw(beta_local)), 1200 * P * beta_local)
    for g in outs[0]["recs"]:
        w = rp.step(g["step_ns"])
        for k in ("b_t", "b_next", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx", "used_pages"):
            assert g[k] == w[k], (g["t"], k, g[k], w[k])
    # the shards' outputs, concatenated over q heads in rank order == the TP1 problem's output
    ids, ctx = outs[0]["ids"], outs[0]["ctx"]
    assert len(ids) > 20
    for o in outs[1:]:
        assert np.array_equal(o["ids"], ids) and np.array_equal(o["ctx"], ctx)
    full = np.concatenate([o["out"] for o in outs], axis=2)      # [L][n][64][D]
    assert full.shape == (L, len(ids), HQ, D)
    for lay in range(L):
        pages, nxt = [], 0
        for cx in ctx:
            m = -(-int(cx) // P)
            pages.append(list(range(nxt, nxt + m)))
            nxt += m
        bt, pk, pv, qq = oatt.synth_paged_batch(SEED, [int(x) for x in ids], ctx, pages, lay, HQ, HKV, D, P, "f16")
        want = oatt.paged_decode_attention(ctx, bt, pk, pv, qq, "f16", nthreads=8)
        got = full[lay].astype(np.float64)
        err = np.max(np.abs(got - want), axis=2) / np.maximum(np.max(np.abs(want), axis=2), 1e-30)
        assert err.max() <= TOL, (lay, float(err.max()))
        # and the shards are not copies of one head group: distinct ranks see distinct values
        assert not np.allclose(full[lay][:, :HQ // world], full[lay][:, HQ // world:2 * HQ // world])


@pytest.mark.parametrize("tp,tp_rank", [(8, 5), (4, 3)])
def test_bench_tp_rank_shard_is_its_global_slice(tp, tp_rank):
    """bench.py's KV-head shard of a non-zero rank at the full 70B launch configuration: its
    outputs are the global q heads [tp_rank*64/tp, (tp_rank+1)*64/tp) of the TP1 oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import gc

    import bench
    from oracle import attention as oatt
    gc.collect()
    torch.cuda.empty_cache()
    S = bench.setup_engine(device=0, cfg_name="llama3-70b-gqa", time_attention=True, out_dtype=2, n_req=1500,
                           tp=tp, tp_rank=tp_rank)
    assert S["pool"].info()["decode_path"] == 2
    eng = S["eng"]
    bufs = eng.buffers(S["qd"], S["od"])
    stream = torch.cuda.current_stream()
    for _ in range(12):
        eng.step(bufs, stream)
    torch.cuda.synchronize()
    Lc, hq = S["L"], S["Hq"]
    ids, ctx = eng.last_batch()
    rng = np.random.default_rng(3)
    sel = rng.choice(len(ids), size=6, replace=False)
    for lay in (0, Lc - 1):
        pages, nxt = [], 0
        for cx in ctx[sel]:
            m = -(-int(cx) // P)
            pages.append(list(range(nxt, nxt + m)))
            nxt += m
        bt, pk, pv, qq = oatt.synth_paged_batch(S["seed"], [int(x) for x in ids[sel]], ctx[sel], pages, lay,
                                                HQ, HKV, D, P, "f16")
        want = oatt.paged_decode_attention(ctx[sel], bt, pk, pv, qq, "f16", nthreads=8)
        want = want[:, tp_rank * hq:(tp_rank + 1) * hq]
        got = S["od"][lay, torch.as_tensor(sel, device="cuda")].cpu().numpy().astype(np.float64)
        err = np.max(np.abs(got - want), axis=2) / np.maximum(np.max(np.abs(want), axis=2), 1e-30)
        assert err.max() <= TOL, (lay, float(err.max()))
    for k in ("eng", "pool", "sched"):
        S.pop(k, None)
    del S
    gc.collect()
    torch.cuda.empty_cache()
