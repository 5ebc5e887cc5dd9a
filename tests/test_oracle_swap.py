"""Pins for the oracle's swap-preemption mode (O7 steps 2'/3', R29-R31;
PAPER.md:75 "The swapping method involves temporarily moving data from GPU memory to CPU
memory when capacity is exceeded.  The data are moved back to the GPU when space becomes
available") -- CPU only."""
import numpy as np

from oracle import engine as oeng
from oracle import policy
from synth import trace


def _run(tr, cap_pages, swap_cap, b, step_ns=1_000_000, P=16):
    ids = list(range(len(tr)))
    eng = oeng.RankEngine(ids, tr.arrival_ns, tr.l_in, tr.l_out, cap_pages, P, swap_cap_pages=swap_cap)
    rp = oeng.Replay([eng], policy.SchedConfig(policy=policy.STATIC, b_static=b), 0)
    recs, peak_swap = [], 0
    while not rp.done():
        recs.append(rp.step(step_ns))
        peak_swap = max(peak_swap, eng.swap_used)
        assert eng.swap_used <= swap_cap
        assert eng.kv.alloc.used <= cap_pages
    return rp, eng, recs, peak_swap


def test_swap_hand_trace():
    """Cap 3 pages, P = 16, static b = 2.  A: l_in 16, l_out 20; B: l_in 15, l_out 20.
    Step 0: A fills 1 page (needs 2 free of 3), B fills 1 page; A's ctx 16 needs a page
    for its decode token (free 1 -> 0): A 17, B 16.  Step 1: B's ctx 16 needs a page, none
    free: B (the last admitted) is the LIFO victim; its 1 page fits the 1-page swap space,
    so it is swapped out (KV kept: ctx = 15 + 1 = 16) instead of recomputed.  B then needs
    ceil(17/16) = 2 free pages to come back: only after A finishes (step 19, 20 tokens)
    does it return by swap-in at step 20 and finish its remaining 19 tokens."""
    tr = trace.Trace(np.zeros(2, np.int64), np.array([16, 15], np.int32), np.array([20, 20], np.int32))
    rp, eng, recs, peak = _run(tr, 3, 1, 2)
    out = [(r["t"], r["n_swap_out"], r["n_swap_in"], r["n_preempted"], r["n_admitted"]) for r in recs
           if r["n_swap_out"] or r["n_swap_in"] or r["n_admitted"]]
    assert out == [(0, 0, 0, 0, 2), (1, 1, 0, 1, 0), (20, 0, 1, 0, 1)]
    assert [r["sum_ctx"] for r in recs[:3]] == [17 + 16, 18, 19]
    assert recs[20]["sum_ctx"] == 17                    # B back with ctx 16, + this step's token
    assert recs[19]["n_finished"] == 1 and recs[-1]["t"] == 38 and recs[-1]["n_finished"] == 1
    assert peak == 1 and eng.swap_used == 0
    assert sum(r["n_decode"] for r in recs) == 40       # conservation: no token is generated twice


def _uniform_trace(n, seed):
    return trace.make_trace(n, 128, 128, 256, seed=seed, dist="uniform")


def test_swap_keeps_page_tables_identical_to_recompute():
    """Given the same step latencies, swap and recompute take identical decisions and page
    tables (R30: swap-in takes exactly the pages a T-token prefill would)."""
    tr = _uniform_trace(40, 1)
    _, _, a, _ = _run(tr, 64, 0, 8)
    _, _, b, _ = _run(tr, 64, 10 ** 6, 8)
    keys = ("b_t", "n_admitted", "n_preempted", "n_decode", "n_finished", "sum_ctx", "used_pages", "table_hash")
    assert [[r[k] for k in keys] for r in a] == [[r[k] for k in keys] for r in b]
    assert sum(r["n_preempted"] for r in a) > 0
    assert all(r["n_swap_out"] == 0 and r["n_swap_in"] == 0 for r in a)
    assert sum(r["n_swap_out"] for r in b) == sum(r["n_preempted"] for r in b)
    assert sum(r["n_swap_in"] for r in b) == sum(r["n_swap_out"] for r in b)


def test_swap_space_bound_mixes_swap_and_recompute():
    """A small swap space: a victim swaps only when its pages fit (R29); the others are
    recomputed; every swapped request comes back by swap-in and the space ends empty."""
    tr = _uniform_trace(40, 1)
    rp, eng, recs, peak = _run(tr, 64, 6, 8)
    n_out = sum(r["n_swap_out"] for r in recs)
    assert 0 < n_out < sum(r["n_preempted"] for r in recs)
    assert sum(r["n_swap_in"] for r in recs) == n_out
    assert 0 < peak <= 6 and eng.swap_used == 0 and not eng.swapped
    assert sum(r["n_decode"] for r in recs) == int(np.sum(tr.l_out))


def test_swap_rejected_with_pd_fusion():
    tr = _uniform_trace(2, 1)
    try:
        oeng.RankEngine([0, 1], tr.arrival_ns, tr.l_in, tr.l_out, 64, 16, pd=True, swap_cap_pages=4)
    except ValueError:
        return
    raise AssertionError("PD + swap must be rejected")
