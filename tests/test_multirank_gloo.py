"""World-size-2 CPU test of the N > 1 host path (gloo, 127.0.0.1).

Each rank owns a DP request shard (oracle RankEngine stands in for its GPU), its
128-byte dbk_stats record is all-gathered over torch.distributed (gloo here, NCCL
inside libdbk on the GPU box), reduced by the library's dbk_stats_reduce, and fed
to the library's scheduler.  Every rank must take the same b_{t+1}, equal to the
single-process oracle Replay of the same shards."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from conftest import build_lib
        if rank == 0:
            build_lib()
        dist.barrier()
        import paper_2503_05248_b200 as dbk
        from oracle import engine as oeng
        from oracle import policy as opol
        from synth import trace
        tr = trace.make_trace(120, 30, 60, 256, seed=4)
        P, cap = 16, 60
        kw = dict(policy=opol.COMBINED, b_min=1, b_max=64, b0=1, bytes_per_token=1, page_size=P,
                  refresh_steps=7, w_len=32, w_sla=5, d_sla_ms=3.0, eps_d_ms=0.2,
                  prior=(16, 16 * 30, 16 * 1800, 16 * 60, 16 * 7200))
        ids = list(range(len(tr)))
        mine = ids[rank::world]
        me = oeng.RankEngine(mine, tr.arrival_ns[mine], tr.l_in[mine], tr.l_out[mine], cap, P, rank, world)
        sched = dbk.Scheduler(**kw)
        ref = oeng.Replay([oeng.RankEngine(ids[r::world], tr.arrival_ns[ids[r::world]], tr.l_in[ids[r::world]],
                                           tr.l_out[ids[r::world]], cap, P, r, world) for r in range(world)],
                          opol.SchedConfig(**kw), world * cap * P)
        b, steps = sched.state()["b"], 0
        while not ref.done():
            step_ns = 1_000_000 + 20_000 * sum(len(e.running) for e in ref.ranks)
            want = ref.step(step_ns)
            # this rank: the same step on its own shard, at the step's (global) clock
            me_clock0 = want["clock_ns"]
            me.release_arrivals(me_clock0)
            me.admit_and_grow(oeng.b_share(b, rank, world, steps))
            local = me.local_stats()
            me.retire()
            local["step_ns"] = step_ns + rank  # ranks measure differently; MAX is taken
            rec = torch.tensor([local[f] for f in dbk._lib.STATS_FIELDS], dtype=torch.int64)
            gathered = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(gathered, rec)
            recs = [dict(zip(dbk._lib.STATS_FIELDS, g.tolist())) for g in gathered]
            glob = dbk.stats_reduce(recs, dbk._lib.MODE_DP)
            assert glob["step_ns"] == step_ns + world - 1
            # N^p from the same global bookkeeping every rank can do (engine.cpp)
            waiting = want["stats"]["n_waiting"]
            glob["step_ns"] = step_ns
            b, why = sched.choose(glob, world * cap * P, 0.0, waiting)
            assert (b, why) == (want["b_next"], want["rationale"]), (steps, b, want["b_next"])
            for k in ("n_active", "n_finished", "sum_ctx", "sum_pages"):
                assert glob[k] == want["stats"][k]
            allb = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allb, torch.tensor([b]))
            assert len({int(x) for x in allb}) == 1
            steps += 1
        q.put((rank, "ok", steps))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_dp_two_ranks_share_every_decision():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, status, info in res:
        assert status == "ok", info
    assert res[0][2] == res[1][2] and res[0][2] > 10
