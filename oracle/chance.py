"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O4: the chance-constrained memory model, Eqs. 7-11 (§III-A).

  Eq. 7   S = sum_{i=1}^{b} (l_in,i + l_out,i)
  Eq. 8   mu_S = b (E[l_in] + E[l_out])
  Eq. 9   sigma_S^2 = b (Var l_in + Var l_out)
  Eq. 10  P(S > eta) ~= 1 - Theta((eta - mu_S) / sigma_S)
  Eq. 2   P(M(b) > M_max) <= eps_M,  theta = Theta^{-1}(1 - eps_M)
  Eq. 11  b <= ((sqrt((sigma theta)^2 + 4 mu eta) - sigma theta) / (2 mu))^2

Readings: Eq. 11 is read with PER-REQUEST moments m = E l_in +
E l_out and v = Var l_in + Var l_out (R3); eta is in tokens, eta = cap_pages * P
(R4); eps_M in (0, 0.5] (R5).  The window moments are carried as exact
integers (n, S = sum(l_in + l_out), V2 = n^2 v with population variances,
SPEC.md:93), and the feasibility test of b is decided in exact integer
arithmetic with theta quantised to theta_q = floor(theta * 2^24 + 0.5) (R6):

  eta - b m >= theta sqrt(b v)
     <=>  A = n eta - b S >= 0  and  A^2 * 2^48 >= theta_q^2 * b * V2.

``b_quad`` is the plain definition: the LARGEST b >= 1 that is feasible,
found by scanning b upward (feasibility is monotone in b).  Eq. 11 appears
here only as ``eq11_bound`` (a real number) for the pins.
"""
from __future__ import annotations

import math
from statistics import NormalDist

THETA_SHIFT = 24
_N01 = NormalDist(0.0, 1.0)


def theta(eps_m: float) -> float:
    """theta = Theta^{-1}(1 - eps_M)."""
    if not (0.0 < eps_m < 1.0):
        raise ValueError("eps_M must be in (0, 1)")
    return _N01.inv_cdf(1.0 - eps_m)


def theta_q(eps_m: float) -> int:
    if not (0.0 < eps_m <= 0.5):
        raise ValueError("eps_M must be in (0, 0.5]")
    return math.floor(theta(eps_m) * (1 << THETA_SHIFT) + 0.5)


def window_moments(n, sum_lin, sum_lin_sq, sum_lout, sum_lout_sq):
    """(n, S, V2): S = sum(l_in + l_out); V2 = n^2 (Var l_in + Var l_out),
    population variances (Eq. 9 per request)."""
    S = sum_lin + sum_lout
    V2 = (n * sum_lin_sq - sum_lin * sum_lin) + (n * sum_lout_sq - sum_lout * sum_lout)
    return n, S, V2


def overflow_probability(m: float, v: float, b: int, eta: float) -> float:
    """Eq. 10 with mu_S = b m, sigma_S = sqrt(b v); indicator when v = 0."""
    mu = b * m
    if v == 0:
        return 1.0 if mu > eta else 0.0
    return 1.0 - _N01.cdf((eta - mu) / math.sqrt(b * v))


def feasible(b: int, n: int, S: int, V2: int, eta: int, tq: int) -> bool:
    """Integer form of P(S > eta) <= eps_M  (Eq. 10 <= eps_M, theta >= 0)."""
    A = n * eta - b * S
    if A < 0:
        return False
    return A * A * (1 << (2 * THETA_SHIFT)) >= tq * tq * b * V2


def b_quad(n: int, S: int, V2: int, eta: int, tq: int) -> int:
    """Largest b >= 1 meeting the chance constraint; 0 if even b = 1 is infeasible."""
    if n < 1 or S < 1:
        raise ValueError("empty window (m = 0)")
    b = 0
    while feasible(b + 1, n, S, V2, eta, tq):
        b += 1
    return b


def eq11_bound(m: float, v: float, eta: float, th: float) -> float:
    """The real right-hand side of Eq. 11 with per-request moments."""
    sv = math.sqrt(v)
    return ((math.sqrt((sv * th) ** 2 + 4.0 * m * eta) - sv * th) / (2.0 * m)) ** 2


def safety_buffer(n: int, S: int, eta: int, bq: int) -> int:
    """L0 (Eq. 12-13), reading R10: the buffer left at the
    chance-constrained optimum, L0 = floor((n eta - b_quad S) / n) i.e.
    eta - mu_S(b_quad) rounded down; L0 = eta when b_quad = 0 (no admission)."""
    if bq <= 0:
        return eta
    return (n * eta - bq * S) // n
