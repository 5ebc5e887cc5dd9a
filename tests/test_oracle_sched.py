"""Pins for oracle O2-O6 (allocator, stats, chance constraint, Alg. 1, Alg. 2) -- CPU only."""
import json
import math
import os
import random

import numpy as np
import pytest

from oracle import chance, policy
from oracle import stats as ostats
from oracle.allocator import CapExceeded, PageAllocator, PagedKV

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- O2 allocator
class NaiveAllocator:
    """Linear scan over a boolean array: the plainest lowest-free-first allocator."""

    def __init__(self, cap):
        self.used = [False] * cap

    def take(self, k):
        free = [p for p, u in enumerate(self.used) if not u]
        if k > len(free):
            raise CapExceeded(k)
        for p in free[:k]:
            self.used[p] = True
        return free[:k]

    def give_back(self, pages):
        for p in pages:
            assert self.used[p]
            self.used[p] = False


def test_allocator_matches_naive_scan_and_invariants():
    rng = random.Random(3)
    cap = 97
    a, b = PageAllocator(cap), NaiveAllocator(cap)
    held = []
    for _ in range(3000):
        if held and rng.random() < 0.45:
            pg = held.pop(rng.randrange(len(held)))
            a.give_back(pg)
            b.give_back(pg)
        else:
            k = rng.randint(0, 9)
            try:
                x = a.take(k)
            except CapExceeded:
                with pytest.raises(CapExceeded):
                    b.take(k)
                continue
            assert x == b.take(k)
            held.append(x)
        flat = [p for h in held for p in h]
        assert len(flat) == len(set(flat))            # no page held twice
        assert a.used == len(flat) and a.free + a.used == cap
        assert a.used <= cap


def test_allocator_all_or_nothing_and_ceil_pages():
    kv = PagedKV(cap_pages=5, page_size=16)
    for r in (1, 2):
        kv.begin(r)
    kv.append([1, 2], [17, 16])          # 2 + 1 pages, lowest first in batch order
    assert kv.pages[1] == [0, 1] and kv.pages[2] == [2]
    with pytest.raises(CapExceeded):
        kv.append([1, 2], [16, 17])      # would need 1 + 2 = 3 > 2 free: nothing changes
    assert kv.ctx == {1: 17, 2: 16} and kv.alloc.free == 2
    kv.append([2], [1])
    assert kv.pages[2] == [2, 3]
    assert kv.release(1) == [0, 1]
    kv.begin(3)
    kv.append([3], [40])                 # reuses the lowest free ids 0, 1, then 4
    assert kv.pages[3] == [0, 1, 4]
    for r in kv.ctx:
        assert len(kv.pages[r]) == -(-kv.ctx[r] // 16)


# ---------------------------------------------------------------- O3 stats
def test_stats_hand_example_and_redundant_bookkeeping():
    ctx = [17, 5, 32]
    l_in = [10, 3, 2]
    l_out = [7, 9, 30]
    rows = [[4, 9, -1], [0, -1, -1], [1, 2, 7]]   # last row: 3 pages for ctx 32 -> mismatch
    r = ostats.batch_stats(ctx, l_in, l_out, rows, 16, 20)
    assert r["n_active"] == 3 and r["sum_ctx"] == 54 and r["sum_ctx_sq"] == 17**2 + 25 + 32**2
    assert r["max_ctx"] == 32 and r["sum_pages"] == 6 and r["free_pages"] == 14
    assert r["table_mismatch"] == 1 and r["over_cap"] == 0
    assert r["n_finished"] == 2                     # 17 = 10 + 7 and 32 = 2 + 30
    assert (r["fin_sum_lin"], r["fin_sum_lin_sq"]) == (12, 104)
    assert (r["fin_sum_lout"], r["fin_sum_lout_sq"]) == (37, 949)


def test_stats_reduce_dp_and_tp():
    a = ostats.batch_stats([5], [2], [3], [[0]], 16, 10)
    b = ostats.batch_stats([40, 3], [1, 1], [2, 2], [[0, 1, 2], [3]], 16, 10)
    a["step_ns"], b["step_ns"] = 7, 9
    g = ostats.reduce_records([a, b], "dp")
    assert g["n_active"] == 3 and g["sum_pages"] == 5 and g["cap_pages"] == 20
    assert g["free_pages"] == 15 and g["max_ctx"] == 40 and g["step_ns"] == 9 and g["n_finished"] == 2
    assert ostats.reduce_records([a, dict(a)], "tp")["step_ns"] == 7
    with pytest.raises(ValueError):
        ostats.reduce_records([a, b], "tp")


# ---------------------------------------------------------------- O4 chance constraint
def test_theta_golden():
    g = gold("chance_instance.json")
    for eps, th in g["theta"]:
        assert abs(chance.theta(eps) - th) < g["theta_abs_tol"]
    assert chance.theta_q(0.5) == 0
    with pytest.raises(ValueError):
        chance.theta(1.5)
    with pytest.raises(ValueError):
        chance.theta_q(0.9)      # reading R5: eps_M in (0, 0.5]


def test_chance_instance_golden():
    g = gold("chance_instance.json")
    m, v, eta, eps = g["m"], g["v"], g["eta"], g["eps_m"]
    b = g["expect_b"]
    assert abs(chance.overflow_probability(m, v, b, eta) - g["overflow_at_b"]) < g["overflow_abs_tol"]
    assert abs(chance.overflow_probability(m, v, b + 1, eta) - g["overflow_at_b_plus_1"]) < g["overflow_abs_tol"]
    # integer window whose moments are exactly (m, v): n = 2, l_in = 200 +- 300, l_out = 300
    n, S, V2 = chance.window_moments(2, -100 + 500, (-100) ** 2 + 500 ** 2, 600, 2 * 300 ** 2)
    assert S / n == m and V2 / n**2 == v
    assert chance.b_quad(n, S, V2, eta, chance.theta_q(eps)) == b
    assert math.floor(chance.eq11_bound(m, v, eta, chance.theta(eps))) == b


def test_eq10_monte_carlo():
    """1e6 sampled batches of 183 iid per-request totals with
    mean 500, variance 90000 (normal surrogate, so the CLT step is exact);
    the overflow frequency lies in the 99% binomial interval of Eq. 10."""
    rng = np.random.default_rng(12345)
    b, trials, eta = 183, 1_000_000, 100_000
    hits = 0
    for _ in range(10):
        x = rng.normal(500.0, 300.0, (trials // 10, b)).sum(axis=1)
        hits += int((x > eta).sum())
    p = chance.overflow_probability(500, 90000, b, eta)
    se = math.sqrt(p * (1 - p) / trials)
    assert abs(hits / trials - p) < 2.576 * se + 1e-9


def _brute_force_double(m, v, eta, eps):
    """Scan b upward with Eq. 10 in floating point."""
    b = 0
    while chance.overflow_probability(m, v, b + 1, eta) <= eps:
        b += 1
        if b > 10**6:
            break
    return b


def test_b_quad_equals_bruteforce_and_closed_form():
    rng = random.Random(11)
    for _ in range(200):
        n = rng.randint(1, 300)
        li = [rng.randint(1, 800) for _ in range(n)]
        lo = [rng.randint(1, 1500) for _ in range(n)]
        n_, S, V2 = chance.window_moments(n, sum(li), sum(x * x for x in li), sum(lo),
                                          sum(x * x for x in lo))
        m, v = S / n, V2 / n**2
        eta = rng.randint(int(m) + 1, 100_000)
        eps = rng.choice([0.001, 0.01, 0.02, 0.05, 0.1, 0.3, 0.5])
        bq = chance.b_quad(n, S, V2, eta, chance.theta_q(eps))
        bf = _brute_force_double(m, v, eta, eps)
        cf = math.floor(chance.eq11_bound(m, v, eta, chance.theta(eps)))
        if bq != bf or bq != cf:
            # only legitimate cause: b sits within rounding of the boundary
            x = chance.eq11_bound(m, v, eta, chance.theta(eps))
            assert abs(x - round(x)) < 1e-6 * max(1.0, x), (n, S, V2, eta, eps, bq, bf, cf)


def test_special_cases_and_monotonicity():
    # v = 0: floor(eta / m) for any eps; eps = 0.5: floor(eta / m) for any v
    n, S, V2 = chance.window_moments(3, 300, 30000, 900, 270000)   # l_in = 100, l_out = 300
    assert V2 == 0 and chance.b_quad(n, S, V2, 12000, chance.theta_q(0.02)) == 30
    n, S, V2 = chance.window_moments(2, 400, 100000, 600, 180000)
    assert chance.b_quad(n, S, V2, 100000, chance.theta_q(0.5)) == 100000 // (S // n)
    # monotone: non-increasing in m and v, non-decreasing in eta and eps
    tq = chance.theta_q(0.02)
    base = chance.b_quad(4, 2000, 4 * 4 * 90000, 100000, tq)
    assert chance.b_quad(4, 2400, 4 * 4 * 90000, 100000, tq) <= base
    assert chance.b_quad(4, 2000, 4 * 4 * 180000, 100000, tq) <= base
    assert chance.b_quad(4, 2000, 4 * 4 * 90000, 120000, tq) >= base
    assert chance.b_quad(4, 2000, 4 * 4 * 90000, 100000, chance.theta_q(0.1)) >= base
    # infeasible even at b = 1
    assert chance.b_quad(1, 1000, 0, 999, tq) == 0


def test_moments_golden():
    for c in gold("moments.json")["cases"]:
        pairs = c["pairs"]
        n = len(pairs)
        n_, S, V2 = chance.window_moments(n, sum(a for a, _ in pairs), sum(a * a for a, _ in pairs),
                                          sum(b for _, b in pairs), sum(b * b for _, b in pairs))
        assert S / n == c["m"] and V2 / n**2 == c["v"]


def test_safety_buffer_reproduces_b_quad_via_alg1():
    """Reading R10: with L0 refreshed from the window, Alg. 1's linear rule
    returns exactly b_quad on that window."""
    rng = random.Random(5)
    for _ in range(2000):
        n = rng.randint(1, 400)
        S = rng.randint(2 * n, 4000 * n)
        V2 = rng.randint(0, (S * S) // 2)
        eta = rng.randint(S // n, 4_000_000)
        tq = chance.theta_q(rng.choice([0.01, 0.02, 0.05, 0.5]))
        bq = chance.b_quad(n, S, V2, eta, tq)
        L0 = chance.safety_buffer(n, S, eta, bq)
        b, fired = policy.batching_memory(1, 1, 1, eta, L0, n, S, 10**9)
        assert fired and b == max(bq, 1)


# ---------------------------------------------------------------- O5 Algorithm 1
def test_alg1_golden_hand_traces():
    for c in gold("alg1_hand_traces.json")["cases"]:
        b, _ = policy.batching_memory(c["b_prev"], c["n_decode"], c["n_prefill"], c["eta"], c["L0"],
                                      1, c["m"], c["b_max"])
        assert b == c["expect"]


def test_alg1_nonincreasing_in_m_before_clamp():
    prev = None
    for m in range(100, 2000, 7):
        b, _ = policy.batching_memory(1, 1, 1, 100000, 1234, 1, m, 10**9)
        if prev is not None:
            assert b <= prev
        prev = b


# ---------------------------------------------------------------- O6 Algorithm 2
def test_alg2_golden_hand_traces():
    g = gold("alg2_hand_traces.json")
    s = g["state"]
    for c in g["cases"]:
        cnt = 20
        b, st = policy.batching_sla(policy.SlaState(s["b_low"], s["b_high"]),
                                    policy.ms_to_ns(c["tau_bar_ms"]) * cnt, cnt, c["b_bar"] * cnt,
                                    policy.ms_to_ns(s["d_sla_ms"]), policy.ms_to_ns(s["eps_d_ms"]),
                                    s["alpha"], s["delta"], s["b_min"], s["b_max"], c["n_decode"])
        assert (b, st.low, st.high) == (c["expect_b"], c["expect_low"], c["expect_high"])


def _fig3_model():
    r = gold("fig3_readings.json")["readings"]
    (b1, d1), (b2, d2) = [(x["b"], x["d_sla_ms"]) for x in r]
    a1 = (d2 - d1) / (b2 - b1)
    return d1 - a1 * b1, a1


def test_fig3_two_point_model_pins():
    g = gold("fig3_readings.json")
    a0, a1 = _fig3_model()
    for x in g["readings"]:
        b_star = math.floor((x["d_sla_ms"] - a0) / a1 + 1e-9)
        assert b_star == x["b"]
        phi = 1000.0 * b_star / (a0 + a1 * b_star)         # Eq. 6: Phi = b / tau_step(b)
        assert abs(phi - x["throughput_tok_s"]) <= g["throughput_tolerance_rel"] * x["throughput_tok_s"]


def _closed_loop(a0, a1, d, eps_d, b_min, b_max, alpha=8, delta=2, rounds=200):
    """Scheduler in SLA mode fed tau(b) = a0 + a1 b (noise free), one step per round."""
    cfg = policy.SchedConfig(policy=policy.SLA, b_min=b_min, b_max=b_max, b0=b_min, alpha=alpha,
                             delta=delta, w_sla=1, d_sla_ms=d, eps_d_ms=eps_d)
    s = policy.Scheduler(cfg)
    seq = [s.b]
    for _ in range(rounds):
        b = s.b
        st = dict.fromkeys(ostats.FIELDS, 0)
        # every request turns over each round (N^d = 0), so only the search moves b
        st.update(n_active=b, n_finished=b, step_ns=policy.ms_to_ns(a0 + a1 * b))
        s.decide(st, 0, 1)
        seq.append(s.b)
    return seq


def test_alg2_closed_loop_direction_and_convergence():
    a0, a1 = _fig3_model()
    for d, b_star in ((50.0, 100), (80.0, 230)):
        seq = _closed_loop(a0, a1, d, 2.0, 1, 512)
        # I1: too slow -> smaller next b, too fast -> larger
        for b, nb in zip(seq[1:], seq[2:]):
            tau = a0 + a1 * b
            if tau > d + 2.0:
                assert nb <= b
            elif tau < d - 2.0:
                assert nb >= b
        tail = seq[-50:]
        assert all(abs(b - b_star) <= 8 for b in tail)               # within +-alpha of b*
        assert all(abs(a0 + a1 * b - d) <= 2.0 + a1 for b in tail)   # inside the deadband
    # I3: the fixed point is non-decreasing in D_SLA
    fps = [_closed_loop(a0, a1, d, 2.0, 1, 512)[-1] for d in (30, 40, 50, 60, 80, 100)]
    assert fps == sorted(fps)


def test_alg2_random_convergence_draws():
    rng = random.Random(9)
    for _ in range(20):
        a1 = rng.uniform(0.02, 0.5)
        a0 = rng.uniform(1, 40)
        b_max = rng.choice([256, 512, 1024])
        b_star = rng.randint(20, b_max - 20)
        d = a0 + a1 * (b_star + 0.5)
        eps_d = max(a1, 4 * a1)                     # eps_D >= a1 and alpha <= 2 eps_D / a1
        seq = _closed_loop(a0, a1, d, eps_d, 1, b_max)
        bound = 2 * math.ceil(math.log2(b_max - 1)) + math.ceil((b_max - 1) / 8)
        assert all(abs(b - b_star) <= 8 for b in seq[bound:]), (a0, a1, b_star, seq[:40])


def test_scheduler_bounds_invariant_random_inputs():
    rng = random.Random(1)
    cfg = policy.SchedConfig(policy=policy.COMBINED, b_min=2, b_max=300, b0=2, alpha=8, delta=2,
                             w_sla=5, d_sla_ms=20.0, eps_d_ms=1.0, bytes_per_token=1, page_size=16,
                             prior=(16, 16 * 100, 16 * 12000, 16 * 300, 16 * 100000))
    s = policy.Scheduler(cfg)
    for _ in range(3000):
        st = dict.fromkeys(ostats.FIELDS, 0)
        na = rng.randint(0, 300)
        nf = rng.randint(0, min(na, 5))
        st.update(n_active=na, n_finished=nf, step_ns=rng.randint(1, 40_000_000),
                  fin_sum_lin=nf * 100, fin_sum_lin_sq=nf * 12000, fin_sum_lout=nf * 300,
                  fin_sum_lout_sq=nf * 100000)
        b, _ = s.decide(st, 10**6, rng.randint(0, 3))
        assert cfg.b_min <= s.sla.low <= s.sla.high <= cfg.b_max
        assert 1 <= b <= cfg.b_max
        assert b <= s.b_mem and b <= s.b_sla                  # PAPER.md:219 min
        assert s.tot[0] >= 1


def test_combined_rationale():
    cfg = policy.SchedConfig(policy=policy.STATIC, b_static=7)
    s = policy.Scheduler(cfg)
    st = dict.fromkeys(ostats.FIELDS, 0)
    assert s.decide(st, 0, 0) == (7, policy.R_STATIC)
