"""Pins for the PD-fusion mode of oracle O7 (R25-R28) -- CPU.

The chunk rule c_t = max(0, b_t - N^d) is checked on SPEC.md:409-412's worked examples, then
on whole replays: every prompt token is prefilled exactly once per admission, decode tokens
are conserved, the cap holds and the run is deterministic."""
import numpy as np

from oracle import engine as oeng
from oracle import policy
from synth import configs, trace


def _engine(l_in, l_out, cap_pages=1000, P=16, arrival=None):
    n = len(l_in)
    arrival = np.zeros(n, np.int64) if arrival is None else np.asarray(arrival, np.int64)
    return oeng.RankEngine(list(range(n)), arrival, l_in, l_out, cap_pages, P, pd=True)


def test_spec_chunk_examples():
    # b_t = 64, N^d = 60 -> chunk of 4 tokens
    e = _engine([10] * 60 + [100], [50] * 61)
    e.release_arrivals(0)
    for r in range(60):           # 60 fully prefilled requests decoding
        e.queue.popleft()
        e.kv.begin(r)
        e.kv.append([r], [10])
        e.running.append(r)
    adm, pre, ch = e.step_pd(64)
    assert (adm, pre) == (1, 0) and ch == [(60, 0, 4)]
    # N^d >= b_t -> chunk 0
    adm, pre, ch = e.step_pd(60)
    assert ch == [] and adm == 0
    # empty decode set, queue non-empty, b_t = 32 -> chunk of 32, FCFS over prompts
    e = _engine([20, 20, 20], [5, 5, 5])
    e.release_arrivals(0)
    adm, pre, ch = e.step_pd(32)
    assert adm == 2 and ch == [(0, 0, 20), (1, 0, 12)]
    e.finish_prefills()
    assert e.running == [0] and e.prefilling == [[1, 12]]
    # next step: request 0 decodes (N^d = 1), request 1 finishes its prompt, 2 starts
    adm, pre, ch = e.step_pd(32)
    assert ch == [(1, 12, 8), (2, 0, 20)] and adm == 1
    assert e.kv.ctx[0] == 21 and e.gen[0] == 1


def test_in_progress_prefill_is_cut_to_free_pages():
    # cap 5 pages of 16: request 0 (l_in 40) holds 3 pages after 40 tokens; request 1 (l_in 40)
    # admission needs ceil(41/16) = 3 pages > 2 free -> head-of-line block
    e = _engine([40, 40], [30, 30], cap_pages=5)
    e.release_arrivals(0)
    adm, pre, ch = e.step_pd(100)
    assert ch == [(0, 0, 40)] and adm == 1
    e.finish_prefills()
    assert e.running == [0]


def _replay(tr, cap_pages, P, cfg, step_ns=2_000_000, world=1):
    ids = list(range(len(tr)))
    ranks = []
    for r in range(world):
        mine = ids[r::world]
        ranks.append(oeng.RankEngine(mine, tr.arrival_ns[mine], tr.l_in[mine], tr.l_out[mine],
                                     cap_pages, P, r, world, pd=True))
    rp = oeng.Replay(ranks, cfg, cap_pages * P)
    recs = []
    while not rp.done() and len(recs) < 200000:
        recs.append(rp.step(step_ns))
    return rp, recs


def test_pd_replay_conservation_cap_determinism():
    tr = trace.make_trace(80, 60, 40, 256, seed=5, arrival="poisson", rate_qps=300.0)
    prior = tuple(configs.prior_record(dict(prior=dict(n=16, mean_in=60, mean_out=40),
                                            trace=dict(dist="lognormal"))).values())
    cap = 48
    for cfg in (policy.SchedConfig(policy=policy.STATIC, b_static=48),
                policy.SchedConfig(policy=policy.MEMORY, b_min=1, b_max=64, b0=8, bytes_per_token=1,
                                   page_size=16, refresh_steps=10, prior=prior)):
        runs = []
        for _ in range(2):
            rp, recs = _replay(tr, cap, 16, cfg)
            runs.append([(r["b_t"], r["n_decode"], r["n_prefill"], r["table_hash"]) for r in recs])
            assert sum(r["n_finished"] for r in recs) == len(tr)
            assert sum(r["n_decode"] for r in recs) == int(tr.l_out.sum())
            e = rp.ranks[0]
            assert e.kv.alloc.used == 0 and not e.prefilling and not e.running
            # chunk never exceeds the rule's budget
            assert all(r["n_prefill"] <= max(0, r["b_t"] - r["n_decode"]) for r in recs)
            # prompt tokens: l_in once per admission, plus the recompute of generated tokens
            pf = sum(r["n_prefill"] for r in recs)
            assert pf >= int(tr.l_in.sum())
            if sum(r["n_preempted"] for r in recs) == 0:
                assert pf == int(tr.l_in.sum())
            assert all(r["stats"]["over_cap"] == 0 and r["stats"]["table_mismatch"] == 0 for r in recs)
        assert runs[0] == runs[1]


def test_pd_replay_preemption_recomputes_prompt_plus_generated():
    tr = trace.make_trace(30, 100, 100, 256, seed=2, dist="uniform")
    rp, recs = _replay(tr, 24, 16, policy.SchedConfig(policy=policy.STATIC, b_static=16))
    assert sum(r["n_preempted"] for r in recs) > 0
    assert sum(r["n_decode"] for r in recs) == int(tr.l_out.sum())
    assert sum(r["n_prefill"] for r in recs) > int(tr.l_in.sum())


def test_pd_dp_two_ranks_shares():
    tr = trace.make_trace(40, 30, 20, 128, seed=9, arrival="poisson", rate_qps=500.0)
    rp, recs = _replay(tr, 32, 16, policy.SchedConfig(policy=policy.STATIC, b_static=9), world=2)
    assert sum(r["n_finished"] for r in recs) == len(tr)
    for r in recs:   # rank k's budget is its share of b minus its own decode count
        for k, (ch, loc) in enumerate(zip(r["chunks"], r["local_stats"])):
            assert sum(q for _, _, q in ch) <= max(0, oeng.b_share(r["b_t"], k, 2, r["t"]) - loc["n_active"])


def test_pd_fixed_token_budget_reading():
    """R36: with a fixed iteration token budget B the chunk is c_t = B - N^d while b_t still
    bounds running + prefilling; B = b_t reproduces R25 step for step."""
    import numpy as np
    from oracle import engine as oeng
    from oracle import policy
    from synth import trace
    tr = trace.make_trace(30, 150, 40, 400, seed=4, dist="uniform")
    ids = list(range(len(tr)))

    def run(budget, b):
        e = oeng.RankEngine(ids, tr.arrival_ns, tr.l_in, tr.l_out, 400, 16, pd=True, max_rows=512,
                            pd_token_budget=budget)
        rp = oeng.Replay([e], policy.SchedConfig(policy=policy.STATIC, b_static=b), 0)
        recs = []
        while not rp.done():
            recs.append(rp.step(1_000_000))
            assert len(e.running) + len(e.prefilling) <= b          # b_t bounds the requests
            assert recs[-1]["n_prefill"] + recs[-1]["n_decode"] <= max(budget or b, recs[-1]["n_decode"])
        return recs
    a, same = run(0, 16), run(16, 16)
    keys = ("n_admitted", "n_preempted", "n_decode", "n_prefill", "sum_ctx", "table_hash")
    assert [[r[k] for k in keys] for r in a] == [[r[k] for k in keys] for r in same]
    big = run(96, 16)                                   # more prefill per step, same request bound
    assert max(r["n_prefill"] for r in big) > max(r["n_prefill"] for r in a)
    assert len(big) < len(a)                            # prompts finish in fewer iterations
    assert sum(r["n_decode"] for r in big) == int(np.sum(tr.l_out))
