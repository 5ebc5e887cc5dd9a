"""CPU checks of the experiment helpers (no GPU): the p99 TBT used by the capacity search is
the nearest-rank percentile over all generated tokens."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "experiments"))


def test_tbt_p99_matches_sorted_token_list():
    import paper_tables
    rng = np.random.default_rng(0)
    recs = [dict(step_ns=int(rng.integers(1e6, 5e7)), n_decode=int(rng.integers(1, 300))) for _ in range(500)]
    toks = np.sort(np.concatenate([np.full(r["n_decode"], r["step_ns"] / 1e6) for r in recs]))
    k = int(np.ceil(0.99 * len(toks)))           # nearest rank (1-based)
    assert paper_tables._tbt_p99(recs) == toks[k - 1]
    const = [dict(step_ns=50_000_000, n_decode=7)] * 10
    assert paper_tables._tbt_p99(const) == 50.0
