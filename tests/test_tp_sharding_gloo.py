"""The arithmetic of the tensor-parallel model step (DESIGN.md §8 "TP model step"; SURVEY.md §8(f)
row 3), CPU only: G processes over gloo, each holding the slices of the GLOBAL oracle weights that
rank r of dbk_model holds (model.cu FillMap):

  W_qkv   rows of its q heads [r Hq/G, (r+1) Hq/G) and of its kv heads (k and v blocks),
  W_o     the columns of its q heads,
  W_gu    gate rows [r F/G, (r+1) F/G) and the matching up rows,
  W_down  the columns of that FFN slice,

run one layer (attention over a shared seeded history, GQA group map preserved because q heads
and kv heads are split in the same proportion), sum the O and down partials with an all-reduce,
and must equal the unsharded oracle layer (float64, to 1e-12).  A plausible slicing mistake (the
wrong kv block, transposed W_o / W_down slices, gate and up from different columns) fails it."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _layer(s, W, x, hist_k, hist_v, pos, rank=0, world=1, dist=None):
    """One decoder layer; with world > 1 on rank `rank`'s slices, partial sums all-reduced."""
    from oracle import model as om
    d, Hq, Hkv, F = s.head_dim, s.q_heads, s.kv_heads, s.ffn
    hq, hk, f = Hq // world, Hkv // world, F // world
    q_rows = np.arange(rank * hq * d, (rank + 1) * hq * d)
    k_rows = Hq * d + np.arange(rank * hk * d, (rank + 1) * hk * d)
    v_rows = (Hq + Hkv) * d + np.arange(rank * hk * d, (rank + 1) * hk * d)
    w_qkv = W["w_qkv"][np.concatenate([q_rows, k_rows, v_rows])]
    w_o = W["w_o"][:, rank * hq * d:(rank + 1) * hq * d]
    w_gu = W["w_gu"][np.concatenate([np.arange(rank * f, (rank + 1) * f), F + np.arange(rank * f, (rank + 1) * f)])]
    w_down = W["w_down"][:, rank * f:(rank + 1) * f]

    def allreduce(a):
        if world == 1:
            return a
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    n = x.shape[0]
    h = om.rmsnorm(x, W["g1"], s.rms_eps)
    qkv = om.linear(h, w_qkv)
    a = np.zeros((n, hq * d))
    for i in range(n):
        q = om.rope(qkv[i, :hq * d].reshape(hq, d), pos[i], s.rope_theta)
        k = om.rope(qkv[i, hq * d:(hq + hk) * d].reshape(hk, d), pos[i], s.rope_theta)
        v = qkv[i, (hq + hk) * d:].reshape(hk, d)
        K = np.concatenate([hist_k[i][:, rank * hk:(rank + 1) * hk], k[None]])
        V = np.concatenate([hist_v[i][:, rank * hk:(rank + 1) * hk], v[None]])
        a[i] = om.attention(q, K, V).reshape(-1)
    x = x + allreduce(om.linear(a, w_o))
    h = om.rmsnorm(x, W["g2"], s.rms_eps)
    gu = om.linear(h, w_gu)
    return x + allreduce(om.linear(om.silu(gu[:, :f]) * gu[:, f:], w_down))


def _case():
    from oracle import model as om
    s = om.ModelShape(layers=1, q_heads=8, kv_heads=4, head_dim=32, hidden=128, ffn=512, vocab=50)
    W = om.weights(9, s, 0)
    rng = np.random.default_rng(3)
    n = 5
    pos = rng.integers(1, 9, n)
    x = rng.standard_normal((n, s.hidden))
    hist_k = [rng.standard_normal((p, s.kv_heads, s.head_dim)) for p in pos]
    hist_v = [rng.standard_normal((p, s.kv_heads, s.head_dim)) for p in pos]
    return s, W, x, hist_k, hist_v, pos


def _worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, W, x, hk, hv, pos = _case()
        want = _layer(s, W, x, hk, hv, pos)
        got = _layer(s, W, x, hk, hv, pos, rank, world, dist)
        q.put((rank, float(np.abs(got - want).max() / np.abs(want).max())))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_slices_allreduce_to_the_unsharded_layer(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, e in res:
        assert isinstance(e, float), e
        assert e < 1e-12, (r, e)


def test_tp_slicing_mistake_is_caught():
    """The pin has teeth: the same 2-rank sum in one process (two threads, all_reduce = a barrier
    and a sum) matches, and giving rank 1 the kv block of rank 0 (round 1's TP bug) breaks it."""
    import threading
    s, W, x, hk, hv, pos = _case()
    want = _layer(s, W, x, hk, hv, pos)

    class ThreadSum:
        def __init__(self):
            self.bar, self.parts = threading.Barrier(2), {}

        def all_reduce(self, t):
            me = threading.get_ident()
            self.bar.wait()
            self.parts[me] = t.numpy().copy()
            self.bar.wait()
            t.copy_(torch.from_numpy(sum(self.parts.values())))
            self.bar.wait()
            self.parts.clear()
            self.bar.wait()

    def two_rank(W1):
        dist, out = ThreadSum(), {}
        th = [threading.Thread(target=lambda r, w: out.__setitem__(r, _layer(s, w, x, hk, hv, pos, r, 2, dist)),
                               args=(r, w)) for r, w in ((0, W), (1, W1))]
        for t_ in th:
            t_.start()
        for t_ in th:
            t_.join()
        return out[1]

    assert np.abs(two_rank(W) - want).max() < 1e-12 * np.abs(want).max()
    d, Hq, Hkv = s.head_dim, s.q_heads, s.kv_heads
    bad = dict(W)
    w = W["w_qkv"].copy()
    hk_ = Hkv // 2
    w[Hq * d + hk_ * d:Hq * d + 2 * hk_ * d] = W["w_qkv"][Hq * d:Hq * d + hk_ * d]  # k block 1 := block 0
    bad["w_qkv"] = w
    assert np.abs(two_rank(bad) - want).max() > 1e-6 * np.abs(want).max()
