"""Synthetic request traces shaped like the paper's workloads.

Recipe:
* lengths l_in, l_out ~ round(LogNormal(mu, sigma)), floor 1, with coefficient
  of variation CV (default 1: sigma = sqrt(ln 2)) and mu = ln(mean) - sigma^2/2
  so the untruncated mean equals the target mean (the paper prints only means,
  PAPER.md:264-286; it names no distribution, SPEC.md:96 picks lognormal);
* pairs with l_in + l_out > L_max are redrawn (rejection), which lowers the
  realised means by well under 2% at the configs' L_max = 4096;
* arrivals: all-at-once ("request arrival rate is set to
  infinite"), Poisson(rate), or piecewise Poisson [(start_ms, rate_qps), ...]
  (SPEC.md:33);
* arrival times are carried as integer nanoseconds so that both the engine and
  the oracle replay release requests at bit-identical clock values.
"""
from __future__ import annotations

import csv
import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Trace:
    arrival_ns: np.ndarray  # int64, non-decreasing
    l_in: np.ndarray        # int32 >= 1
    l_out: np.ndarray       # int32 >= 1

    def __len__(self):
        return int(self.l_in.shape[0])

    def head(self, n: int) -> "Trace":
        return Trace(self.arrival_ns[:n].copy(), self.l_in[:n].copy(), self.l_out[:n].copy())


def _lognormal_int(rng, mean, cv, n):
    sigma = math.sqrt(math.log1p(cv * cv))
    mu = math.log(mean) - 0.5 * sigma * sigma
    x = rng.lognormal(mu, sigma, n)
    return np.maximum(1, np.rint(x)).astype(np.int64)


def sample_lengths(n, mean_in, mean_out, L_max, seed, cv=1.0, dist="lognormal"):
    rng = np.random.Generator(np.random.PCG64(seed))
    if dist == "fixed":
        li = np.full(n, int(mean_in), np.int64)
        lo = np.full(n, int(mean_out), np.int64)
    elif dist == "uniform":  # U{1..mean_in}, U{1..mean_out} (toy config)
        li = rng.integers(1, int(mean_in) + 1, n)
        lo = rng.integers(1, int(mean_out) + 1, n)
    else:
        li = _lognormal_int(rng, mean_in, cv, n)
        lo = _lognormal_int(rng, mean_out, cv, n)
        bad = li + lo > L_max
        while bad.any():
            k = int(bad.sum())
            li[bad] = _lognormal_int(rng, mean_in, cv, k)
            lo[bad] = _lognormal_int(rng, mean_out, cv, k)
            bad = li + lo > L_max
    if np.any(li + lo > L_max):
        raise ValueError("fixed/uniform lengths exceed L_max")
    return li.astype(np.int32), lo.astype(np.int32)


def arrivals_ns(n, kind="all-at-once", rate_qps=None, segments=None, seed=0):
    if kind == "all-at-once":
        return np.zeros(n, np.int64)
    rng = np.random.Generator(np.random.PCG64(seed + 0x5EED))
    if kind == "poisson":
        if not rate_qps or rate_qps <= 0:
            raise ValueError("poisson rate must be > 0")
        gaps = rng.exponential(1e9 / rate_qps, n)
        return np.rint(np.cumsum(gaps)).astype(np.int64)
    if kind == "piecewise":
        # segments: [(start_ms, rate_qps), ...] strictly increasing starts
        starts = [s for s, _ in segments]
        if any(b <= a for a, b in zip(starts, starts[1:])) or any(r <= 0 for _, r in segments):
            raise ValueError("bad segments")
        out = []
        t = segments[0][0] * 1e6
        seg = 0
        while len(out) < n:
            while seg + 1 < len(segments) and t >= segments[seg + 1][0] * 1e6:
                seg += 1
            rate = segments[seg][1]
            t_next = t + rng.exponential(1e9 / rate)
            if seg + 1 < len(segments) and t_next >= segments[seg + 1][0] * 1e6:
                # memoryless: restart the draw at the boundary with the next rate
                t = segments[seg + 1][0] * 1e6
                continue
            t = t_next
            out.append(t)
        return np.rint(np.asarray(out)).astype(np.int64)
    raise ValueError(kind)


def make_trace(n, mean_in, mean_out, L_max, seed, cv=1.0, dist="lognormal",
               arrival="all-at-once", rate_qps=None, segments=None, arrival_seed=None) -> Trace:
    """arrival_seed: seed of the arrival process alone (default: `seed`), so several Poisson
    streams can carry the same length sample."""
    li, lo = sample_lengths(n, mean_in, mean_out, L_max, seed, cv, dist)
    arr = arrivals_ns(n, arrival, rate_qps, segments, seed if arrival_seed is None else arrival_seed)
    return Trace(arr, li, lo)


def write_csv(trace: Trace, path):
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["arrival_ms", "l_in", "l_out"])
        for a, i, o in zip(trace.arrival_ns, trace.l_in, trace.l_out):
            w.writerow([f"{int(a) / 1e6:.6f}", int(i), int(o)])


def read_csv(path) -> Trace:
    arr, li, lo = [], [], []
    with open(path) as f:
        r = csv.reader(f)
        header = next(r)
        if header != ["arrival_ms", "l_in", "l_out"]:
            raise ValueError(f"bad header {header}")
        for lineno, row in enumerate(r, start=2):
            a, i, o = float(row[0]), int(row[1]), int(row[2])
            if i < 1 or o < 1 or a < 0:
                raise ValueError(f"line {lineno}: invalid row {row}")
            arr.append(int(round(a * 1e6)))
            li.append(i)
            lo.append(o)
    order = np.argsort(np.asarray(arr, np.int64), kind="stable")
    return Trace(np.asarray(arr, np.int64)[order], np.asarray(li, np.int32)[order],
                 np.asarray(lo, np.int32)[order])
