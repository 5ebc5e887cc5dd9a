"""Pins for oracle O7 (engine replay) and the synthetic input generators -- CPU only."""
import numpy as np
import pytest

from oracle import engine as oeng
from oracle import policy
from synth import configs, hashgen, trace


def _replay(tr, cap_pages, P, cfg, mem_cap, step_ns_fn, world=1, max_steps=100000):
    ids = list(range(len(tr)))
    ranks = []
    for r in range(world):
        mine = ids[r::world]
        ranks.append(oeng.RankEngine(mine, tr.arrival_ns[mine], tr.l_in[mine], tr.l_out[mine],
                                     cap_pages, P, r, world))
    rp = oeng.Replay(ranks, cfg, mem_cap)
    recs = []
    while not rp.done() and len(recs) < max_steps:
        # step time is a function of the batch about to run (noise-free latency model)
        recs.append(rp.step(step_ns_fn(rp)))
    return rp, recs


def test_single_request_hand_trace():
    """SPEC.md:384 adapted: one request l_in = 8, l_out = 4, static b = 1, every
    decode step costs 11 ms -> 4 steps, ctx 9..12, 4 tokens, clock 44 ms."""
    tr = trace.Trace(np.zeros(1, np.int64), np.array([8], np.int32), np.array([4], np.int32))
    cfg = policy.SchedConfig(policy=policy.STATIC, b_static=1)
    rp, recs = _replay(tr, 4, 16, cfg, 0, lambda rp: 11_000_000)
    assert [r["sum_ctx"] for r in recs] == [9, 10, 11, 12]
    assert [r["n_finished"] for r in recs] == [0, 0, 0, 1]
    assert rp.clock == 44_000_000 and sum(r["n_decode"] for r in recs) == 4


def _tau(a0_ms, a1_ms):
    def f(rp):
        n = sum(len(e.running) for e in rp.ranks)
        n = max(n, 1)
        return int(round((a0_ms + a1_ms * n) * 1e6))
    return f


def test_conservation_cap_and_determinism_with_preemption():
    tr = trace.make_trace(60, 40, 60, 256, seed=3, arrival="poisson", rate_qps=200.0)
    prior = tuple(configs.prior_record(dict(prior=dict(n=16, mean_in=40, mean_out=60),
                                            trace=dict(dist="lognormal"))).values())
    cap = 40   # 640 tokens: tight
    for cfg in (policy.SchedConfig(policy=policy.STATIC, b_static=32),     # overcommits -> preempts
                policy.SchedConfig(policy=policy.COMBINED, b_min=1, b_max=32, b0=1, d_sla_ms=5.0,
                                   eps_d_ms=0.3, bytes_per_token=1, page_size=16, refresh_steps=10,
                                   prior=prior)):
        runs = []
        for _ in range(2):
            rp, recs = _replay(tr, cap, 16, cfg, cap * 16, _tau(1.0, 0.2))
            runs.append(recs)
            assert sum(r["n_finished"] for r in recs) == len(tr)
            assert all(r["used_pages"] <= cap for r in recs)
            assert all(r["stats"]["table_mismatch"] == 0 for r in recs)
            assert all(r["stats"]["over_cap"] == 0 for r in recs)
            assert all(rp.ranks[0].gen[i] == tr.l_out[i] for i in range(len(tr)))
        strip = lambda rs: [{k: v for k, v in r.items() if k != "batches"} for r in rs]
        assert strip(runs[0]) == strip(runs[1])
        if cfg.policy == policy.STATIC:
            assert sum(r["n_preempted"] for r in runs[0]) > 0


def test_generated_tokens_equal_sum_lout_even_with_recompute():
    tr = trace.make_trace(40, 30, 80, 200, seed=8)
    cfg = policy.SchedConfig(policy=policy.STATIC, b_static=40)
    rp, recs = _replay(tr, 30, 16, cfg, 0, _tau(1.0, 0.1))
    assert sum(r["n_preempted"] for r in recs) > 0
    # each preempted request regenerates nothing twice: gen counts persist across recompute
    assert all(rp.ranks[0].gen[i] == tr.l_out[i] for i in range(len(tr)))


def test_eq6_throughput_tie_in():
    """at saturation with homogeneous lengths and static b,
    tokens/s converges to Phi = b / tau_step(b) (Eq. 6)."""
    a0, a1 = 10.0, 0.05
    for b in (16, 64, 256):
        tr = trace.make_trace(4 * b, 32, 64, 4096, seed=1, dist="fixed")
        cfg = policy.SchedConfig(policy=policy.STATIC, b_static=b)
        rp, recs = _replay(tr, 10**6, 16, cfg, 0, _tau(a0, a1))
        steady = recs[5:-70]
        tok = sum(r["n_decode"] for r in steady)
        secs = sum(r["step_ns"] for r in steady) / 1e9
        phi = 1000.0 * b / (a0 + a1 * b)
        assert abs(tok / secs - phi) <= 0.02 * phi


def test_memory_policy_toy_config_pins():
    """SURVEY.md §8(d) toy: priors m = 129, v = 2730.5 give b_quad = 27 at
    eta = 4096 (clamped to B_max = 8) and 5 at eta = 1024 (toy-tight)."""
    for name, bq in (("toy", 27), ("toy-tight", 5)):
        c = configs.CONFIGS[name]
        pr = configs.prior_record(c)
        cfg = policy.SchedConfig(policy=policy.MEMORY, b_min=c["b_min"], b_max=c["b_max"], b0=1,
                                 eps_m=c["eps_m"], bytes_per_token=1, page_size=16,
                                 prior=tuple(pr.values()))
        s = policy.Scheduler(cfg)
        n, S, V2 = s.moments()
        assert S / n == 129 and V2 / n**2 == 2730.5
        st = dict.fromkeys(("n_active", "n_finished", "step_ns", "fin_sum_lin", "fin_sum_lin_sq",
                            "fin_sum_lout", "fin_sum_lout_sq"), 0)
        st.update(n_active=1)
        b, _ = s.decide(st, c["cap_tokens"], 3)
        assert s.bq == bq and b == min(bq, c["b_max"])


def test_dp_replay_all_ranks_share_decision():
    tr = trace.make_trace(80, 30, 50, 256, seed=4)
    cfg = policy.SchedConfig(policy=policy.MEMORY, b_min=1, b_max=64, b0=1, bytes_per_token=1,
                             page_size=16, prior=(16, 16 * 30, 16 * 1800, 16 * 50, 16 * 5000))
    rp, recs = _replay(tr, 50, 16, cfg, 2 * 50 * 16, _tau(1.0, 0.1), world=2)
    assert sum(r["n_finished"] for r in recs) == len(tr)
    for r in recs:
        assert len(r["local_stats"]) == 2
        assert r["stats"]["n_active"] == sum(x["n_active"] for x in r["local_stats"])
    assert sum(oeng.b_share(b, k, 2) for b in range(100) for k in range(2)) == sum(range(100))


def test_dp_share_rotates_and_small_b_is_live():
    """R21: the shares always sum to b_t, differ by at most one, and the remainder rotates with
    the step index; with a static b_t = 1 < G = 4 every rank still serves its shard (round 1
    gave the remainder to the low ranks only, so ranks 1..3 never admitted)."""
    for G in (2, 3, 4, 8):
        for b in range(0, 40):
            for t in range(2 * G):
                sh = [oeng.b_share(b, k, G, t) for k in range(G)]
                assert sum(sh) == b and max(sh) - min(sh) <= 1
            # over G consecutive steps every rank gets the extra slot (b mod G) times
            for k in range(G):
                assert sum(oeng.b_share(b, k, G, t) for t in range(G)) == b
    tr = trace.make_trace(24, 10, 8, 64, seed=11)
    rp, recs = _replay(tr, 64, 16, policy.SchedConfig(policy=policy.STATIC, b_static=1), 4 * 64 * 16,
                       lambda rp: 1_000_000, world=4)
    assert sum(r["n_finished"] for r in recs) == len(tr)
    # a rank keeps what it admitted under an earlier share: sum running <= G * ceil(b_t / G)
    assert all(r["n_decode"] <= 4 for r in recs) and max(r["n_decode"] for r in recs) > 1


# ------------------------------------------------------------------ synth
def test_hashgen_values_exact_and_deterministic():
    v = hashgen.gen_values(5, hashgen.KIND_K, [1, 2], np.arange(7)[:, None], 3, 4, 64)
    assert v.shape == (7, 2, 64)
    assert np.all(v >= -1) and np.all(v < 1) and np.all(v * 128 == np.round(v * 128))
    assert np.array_equal(v, hashgen.gen_values(5, hashgen.KIND_K, [1, 2], np.arange(7)[:, None], 3, 4, 64))
    hashgen.to_bits(v, "f16")
    hashgen.to_bits(v * 16, "bf16")
    # kinds and coordinates decorrelate
    w = hashgen.gen_values(5, hashgen.KIND_V, [1, 2], np.arange(7)[:, None], 3, 4, 64)
    assert not np.array_equal(v, w)
    assert abs(v.mean()) < 0.05 and 0.3 < v.std() < 0.7


def test_splitmix64_known_value():
    # splitmix64 reference stream seeded with 0: first output 0xE220A8397B1DCDAF
    assert int(hashgen.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF


def test_trace_generator_moments_and_csv(tmp_path):
    tr = trace.make_trace(100_000, 68.4, 344.5, 4096, seed=7)
    assert tr.l_in.min() >= 1 and (tr.l_in + tr.l_out).max() <= 4096
    assert abs(tr.l_in.mean() / 68.4 - 1) < 0.02 and abs(tr.l_out.mean() / 344.5 - 1) < 0.02
    t2 = trace.make_trace(50, 10, 20, 100, seed=3, arrival="poisson", rate_qps=5.4)
    assert np.all(np.diff(t2.arrival_ns) >= 0)
    p = tmp_path / "t.csv"
    trace.write_csv(t2, p)
    t3 = trace.read_csv(p)
    assert np.array_equal(t3.l_in, t2.l_in) and np.array_equal(t3.l_out, t2.l_out)
    assert np.all(np.abs(t3.arrival_ns - t2.arrival_ns) <= 1)
    with pytest.raises(ValueError):
        trace.arrivals_ns(3, "poisson", rate_qps=0)


def test_poisson_rate_and_piecewise():
    a = trace.arrivals_ns(10_000, "poisson", rate_qps=5.4, seed=1)
    assert abs(np.diff(a).mean() / 1e6 - 1000 / 5.4) / (1000 / 5.4) < 0.03
    b = trace.arrivals_ns(3000, "piecewise", segments=[(0, 10.0), (60000, 25.0), (90000, 10.0)], seed=2)
    assert np.all(np.diff(b) >= 0)
    in_surge = ((b >= 60e9) & (b < 90e9)).sum() / 30.0
    assert 20 < in_surge < 30
