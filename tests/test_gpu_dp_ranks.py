"""Two DP ranks on one B200 (two processes, each with its own pool on cuda:0): the
engine's request-sharded path with real kernels, the 128-byte statistics records
exchanged by the caller (gloo all_gather through dbk_engine_step_launch / _finish)
and reduced by the library.  Every rank must take the same b_{t+1} and the run must
replay bit for bit in the oracle's 2-rank Replay (step_ns = MAX over ranks).  The
NCCL transport of the same records is covered by test_gpu_parity.py (single rank);
multi-GPU NCCL runs need more than the one GPU available here."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import numpy as np

        import paper_2503_05248_b200 as dbk
        from oracle import engine as oeng
        from oracle import policy as opol
        from synth import trace
        torch.cuda.set_device(0)
        tr = trace.make_trace(120, 60, 90, 256, seed=7, arrival="poisson", rate_qps=3000.0)
        L, H, d, P, cap = 2, 8, 64, 16, 48
        beta = 2 * L * H * d * 2
        kw = dict(policy=opol.COMBINED, b_min=1, b_max=40, b0=1, bytes_per_token=beta, page_size=P,
                  refresh_steps=9, w_len=24, w_sla=6, alpha=4, delta=1, d_sla_ms=0.12, eps_d_ms=0.01,
                  prior=(16, 16 * 60, 16 * 4800, 16 * 90, 16 * 10800))
        mem_cap = world * cap * P * beta
        sched = dbk.Scheduler(**kw)
        pool = dbk.KVPool(L, H, H, d, cap, 48, 16, "f16")
        eng = dbk.Engine(pool, sched, tr.arrival_ns, tr.l_in, tr.l_out, mem_cap, seed=5, out_dtype=2,
                         rank=rank, world=world)
        qd = torch.empty(L, 48, H, d, dtype=torch.float16, device="cuda")
        od = torch.empty(L, 48, H, d, dtype=torch.float32, device="cuda")
        bufs = eng.buffers(qd, od)
        ids = list(range(len(tr)))
        ref = oeng.Replay([oeng.RankEngine(ids[r::world], tr.arrival_ns[ids[r::world]], tr.l_in[ids[r::world]],
                                           tr.l_out[ids[r::world]], cap, P, r, world) for r in range(world)],
                          opol.SchedConfig(**kw), mem_cap)
        steps = 0
        fields = dbk._lib.STATS_FIELDS
        while not eng.done():
            local = eng.step_launch(bufs)
            rec = torch.tensor([local[f] for f in fields], dtype=torch.int64)
            gathered = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(gathered, rec)
            glob = dbk.stats_reduce([dict(zip(fields, g.tolist())) for g in gathered], dbk._lib.MODE_DP)
            out = eng.step_finish(glob)
            want = ref.step(glob["step_ns"])
            for k in ("clock_ns", "b_t", "b_next", "n_decode", "n_finished", "sum_ctx", "used_pages", "rationale"):
                assert out[k] == want[k], (rank, steps, k, out[k], want[k])
            # per-rank admissions / preemptions add up to the replay's global counts
            cnt = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(cnt, torch.tensor([out["n_admitted"], out["n_preempted"], out["b_next"]]))
            assert sum(int(x[0]) for x in cnt) == want["n_admitted"]
            assert sum(int(x[1]) for x in cnt) == want["n_preempted"]
            assert len({int(x[2]) for x in cnt}) == 1
            steps += 1
        assert ref.done()
        pool.close()
        q.put((rank, "ok", steps))
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_two_dp_ranks_on_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, status, info in res:
        assert status == "ok", info
    assert res[0][2] == res[1][2] and res[0][2] > 10
