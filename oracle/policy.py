"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O5 Algorithm 1 (BatchingMemory), O6 Algorithm 2
(BatchingSLA), the min-combination and the
static baseline, plus the telemetry windows that feed them.

Everything is integer arithmetic (R6, R11-R16):
* moments window: step records (count, sum l_in, sum l_in^2, sum l_out,
  sum l_out^2) of requests that FINISHED, oldest dropped while the rest still
  hold >= W_len requests; seeded with a prior record that ages out the same way;
* L0 refreshed every R decisions ("updated online periodically");
* SLA window: (step_ns, n_active) of the last W_sla decode steps;
  tau_bar > D + eps_D  <=>  sum step_ns > cnt (D + eps_D), D and eps_D in
  integer ns; b_bar = round-half-up(sum n_active / cnt).
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

from . import chance

STATIC, MEMORY, SLA, COMBINED = 0, 1, 2, 3
R_STATIC, R_MEMORY, R_SLA, R_MIN, R_CARRY = 0, 1, 2, 3, 4


def ms_to_ns(ms: float) -> int:
    # llround(ms * 1e6): round half away from zero
    x = ms * 1e6
    return int(x + 0.5) if x >= 0 else -int(-x + 0.5)


@dataclass
class SchedConfig:
    policy: int = MEMORY
    b_static: int = 256
    b_min: int = 1
    b_max: int = 512
    b0: int = 1
    alpha: int = 8
    delta: int = 2
    w_len: int = 256
    w_sla: int = 20
    refresh_steps: int = 100
    page_size: int = 16
    eps_m: float = 0.02
    d_sla_ms: float = 50.0
    eps_d_ms: float = 2.0
    bytes_per_token: int = 1
    prior: tuple = (1, 1, 1, 1, 1)  # (n, sum_lin, sum_lin_sq, sum_lout, sum_lout_sq)


def batching_memory(b_prev, n_decode, n_prefill, eta, L0, n, S, b_max):
    """Algorithm 1, lines 3-8."""
    b_t = b_prev                                            # line 4
    fired = False
    if n_decode > 0 and n_prefill > 0:                      # line 5
        b_t = ((eta - L0) * n) // S                         # line 6: floor((eta - L0) / (E l_in + E l_out))
        b_t = min(max(b_t, n_decode), b_max)                # line 7
        fired = True
    return b_t, fired


@dataclass
class SlaState:
    low: int
    high: int


def batching_sla(state: SlaState, sum_ns, cnt, sum_b, d_ns, eps_ns, alpha, delta, b_min, b_max,
                 n_decode):
    """Algorithm 2, lines 2-16.  Returns (b_t, new_state)."""
    b_bar = (2 * sum_b + cnt) // (2 * cnt)                  # line 4 (round half up)
    lo, hi = state.low, state.high
    if sum_ns > cnt * (d_ns + eps_ns):                      # line 5: tau_bar > D + eps_D
        new_hi = max(b_bar, lo + alpha)                     # line 6
        new_lo = max(lo - delta, b_min)                     # line 7
    elif sum_ns < cnt * (d_ns - eps_ns):                    # line 8: tau_bar < D - eps_D
        new_lo = min(b_bar, hi - alpha)                     # line 9
        new_hi = min(hi + delta, b_max)                     # line 10
    else:
        new_hi = min(b_bar + alpha // 2, b_max)             # line 12
        new_lo = max(b_bar - alpha // 2, b_min)             # line 13
    # reading R14: re-clamp into [B_min, B_max] and order the bounds
    new_lo = min(max(new_lo, b_min), b_max)
    new_hi = min(max(new_hi, b_min), b_max)
    if new_lo > new_hi:
        new_lo, new_hi = new_hi, new_lo
    b_t = (new_lo + new_hi) // 2                            # line 15
    b_t = min(max(b_t, n_decode), b_max)                    # line 16
    return b_t, SlaState(new_lo, new_hi)


@dataclass
class Scheduler:
    cfg: SchedConfig
    t: int = 0
    L0: int = 0
    bq: int = 0
    eta: int = 0
    b_mem: int = 0
    b_sla: int = 0
    b: int = 0
    sla: SlaState = None
    win: deque = field(default_factory=deque)
    tot: list = field(default_factory=lambda: [0, 0, 0, 0, 0])
    sla_win: deque = field(default_factory=deque)
    tq: int = 0

    def __post_init__(self):
        c = self.cfg
        if not (1 <= c.b_min <= c.b_max) or c.alpha < 1 or c.delta < 1 or c.w_len < 1 or c.w_sla < 1:
            raise ValueError("bad scheduler config")
        if c.policy in (MEMORY, COMBINED):
            self.tq = chance.theta_q(c.eps_m)
        self.b = self.b_mem = self.b_sla = c.b_static if c.policy == STATIC else c.b0
        self.sla = SlaState(c.b_min, c.b_max)               # Alg. 2 line 1
        self._push_window(tuple(int(x) for x in c.prior))

    def _push_window(self, rec):
        self.win.append(rec)
        for k in range(5):
            self.tot[k] += rec[k]
        while len(self.win) > 1 and self.tot[0] - self.win[0][0] >= self.cfg.w_len:
            old = self.win.popleft()
            for k in range(5):
                self.tot[k] -= old[k]

    def moments(self):
        return chance.window_moments(*self.tot)

    def decide(self, st: dict, mem_cap_bytes: int, n_prefill: int):
        """Consume the (global) stats of the step just finished; return (b_{t+1}, rationale)."""
        c = self.cfg
        if st["n_finished"] > 0:
            self._push_window((st["n_finished"], st["fin_sum_lin"], st["fin_sum_lin_sq"],
                               st["fin_sum_lout"], st["fin_sum_lout_sq"]))
        if st["n_active"] > 0:
            self.sla_win.append((st["step_ns"], st["n_active"]))
            if len(self.sla_win) > c.w_sla:
                self.sla_win.popleft()
        n_decode = st["n_active"] - st["n_finished"]
        if c.policy == STATIC:
            self.t += 1
            self.b = c.b_static
            return self.b, R_STATIC
        rationale = R_CARRY
        if c.policy in (MEMORY, COMBINED):
            cap_pages = mem_cap_bytes // (c.page_size * c.bytes_per_token)
            self.eta = cap_pages * c.page_size                   # reading R4
            n, S, V2 = self.moments()
            if self.t % c.refresh_steps == 0:
                self.bq = chance.b_quad(n, S, V2, self.eta, self.tq)
                self.L0 = chance.safety_buffer(n, S, self.eta, self.bq)
            self.b_mem, fired = batching_memory(self.b_mem, n_decode, n_prefill, self.eta, self.L0,
                                                n, S, c.b_max)
            if fired:
                rationale = R_MEMORY
        if c.policy in (SLA, COMBINED) and self.sla_win:
            cnt = len(self.sla_win)
            sum_ns = sum(x for x, _ in self.sla_win)
            sum_b = sum(y for _, y in self.sla_win)
            self.b_sla, self.sla = batching_sla(self.sla, sum_ns, cnt, sum_b, ms_to_ns(c.d_sla_ms),
                                                ms_to_ns(c.eps_d_ms), c.alpha, c.delta, c.b_min,
                                                c.b_max, n_decode)
            if c.policy == SLA:
                rationale = R_SLA
        if c.policy == MEMORY:
            self.b = self.b_mem
        elif c.policy == SLA:
            self.b = self.b_sla
        else:                                                    # PAPER.md:219 b* = min
            self.b = min(self.b_mem, self.b_sla)
            rationale = R_MEMORY if self.b_mem < self.b_sla else (R_SLA if self.b_sla < self.b_mem else R_MIN)
        self.t += 1
        return self.b, rationale
