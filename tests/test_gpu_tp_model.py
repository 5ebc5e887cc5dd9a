"""GPU parity of the tensor-parallel full decode step (DESIGN.md §8 "TP model step"; SURVEY.md
§8(f) row 3: "TP O-proj allreduce fused over NVLink"): G processes share one B200, each holding
rank r's slice of the model (its KV heads in the pool with kv_head_offset = r * Hkv/G, the matching
slices of W_qkv / W_o / W_gu / W_down), with the residual stream in dbk_tp buffers mapped through
CUDA IPC -- the same code path as NVLink peer memory across GPUs: the O and down GEMMs add each
partial chunk into the OWNER rank's buffer with TMA reduce-adds, a one-warp barrier publishes it,
and the next RMSNorm gathers the owners' slices.

Every rank's logits must equal the GLOBAL oracle O8 (oracle/model.py decode_step of the unsharded
model) at the R35 bar (per-row inf-norm <= 2e-3), and the K / V each rank writes into its pool
must equal the oracle's K / V of its global heads, over two consecutive steps (the second attends
to the first's model-written K / V and reuses the rotating residual buffers)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 2e-3
P = 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _row_err(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    got, want = got.reshape(-1, got.shape[-1]), want.reshape(-1, want.shape[-1])
    return float((np.abs(got - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)).max())


def _tp_model(dbk, dist, rank, world, shape):
    from oracle import model as om
    from oracle.allocator import PagedKV
    s = om.ModelShape(**shape)
    G = world
    hq, hk = s.q_heads // G, s.kv_heads // G
    kv_seed, wseed = 7, 8
    ctx = [1, 2, 17, 33, 100, 129]
    n = len(ctx)
    maxp = max(-(-(c + 4) // P) for c in ctx) + 1
    cap = sum(-(-(c + 2) // P) for c in ctx) + 4
    pool = dbk.KVPool(s.layers, hq, hk, s.head_dim, cap, n + 2, maxp, "f16", kv_head_offset=rank * hk)
    tp = dbk.Tp(dist, G, rank, 0, n + 2, s.hidden)
    model = dbk.Model(pool, s.hidden, s.ffn, s.vocab, max_pos=maxp * P, weight_seed=wseed, tp_size=G, tp_rank=rank)
    model.attach_tp(tp)
    ids = [int(i) * 131 + 7 for i in range(n)]
    ref = PagedKV(cap, P)
    for r, c in zip(ids, ctx):
        pool.request_begin(r, max(1, c - 1), 4)
        ref.begin(r)
    pool.append_tokens(ids, [c - 1 for c in ctx], seed=kv_seed)
    ref.append(ids, [c - 1 for c in ctx])
    kvt = pool.kv.view(torch.float16).view(s.layers, cap, hk, 2, P, s.head_dim)
    errs = {}
    written = {}
    for step in range(2):
        pool.reserve_tokens(ids, [1] * n)
        ref.append(ids, [1] * n)
        cur = [ref.ctx[r] for r in ids]
        logits = torch.empty(n, s.vocab, dtype=torch.float32, device="cuda")
        model.step(ids, logits)
        torch.cuda.synchronize()
        want, nk, nv, _ = om.decode_step(s, wseed, kv_seed, ids, cur, kv_written=written)
        errs[f"logits{step}"] = _row_err(logits.cpu().numpy(), want)
        ek = ev = 0.0
        for lay in range(s.layers):
            for i, (r, c) in enumerate(zip(ids, cur)):
                _, _, pages = pool.request_info(r)
                tile = kvt[lay, pages[(c - 1) // P], :, :, (c - 1) % P, :].float().cpu().numpy()
                ek = max(ek, _row_err(tile[:, 0], nk[lay, i, rank * hk:(rank + 1) * hk]))
                ev = max(ev, _row_err(tile[:, 1], nv[lay, i, rank * hk:(rank + 1) * hk]))
                written[(r, c - 1, lay)] = (nk[lay, i], nv[lay, i])
        errs[f"k{step}"], errs[f"v{step}"] = ek, ev
    model.close()
    tp.close()
    pool.close()
    return errs


def _worker(rank, world, port, shape, q):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_05248_b200 as dbk
        torch.cuda.set_device(0)
        q.put((rank, "ok", _tp_model(dbk, dist, rank, world, shape)))
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(world, shape):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, status, info in res:
        assert status == "ok", info
    return {r: info for r, _, info in res}


@pytest.mark.parametrize("world,shape", [
    (2, dict(layers=2, q_heads=8, kv_heads=4, head_dim=64, hidden=512, ffn=512, vocab=400)),
    (2, dict(layers=2, q_heads=8, kv_heads=2, head_dim=128, hidden=1024, ffn=1024, vocab=1000)),
    (4, dict(layers=2, q_heads=8, kv_heads=4, head_dim=64, hidden=512, ffn=512, vocab=400)),
])
def test_tp_model_steps_match_the_global_oracle(world, shape):
    errs = _run(world, shape)
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):  # observed maxima, for profiles/
        import json
        path = os.path.join(out, "tp_model_err.json")
        rec = json.load(open(path)) if os.path.exists(path) else {}
        rec[f"G{world}_H{shape['hidden']}_d{shape['head_dim']}"] = {str(r): e for r, e in errs.items()}
        json.dump(rec, open(path, "w"), indent=1)
    for r, e in errs.items():
        for k, v in e.items():
            assert v <= TOL, (r, k, v, e)
