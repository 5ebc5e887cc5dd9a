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


def test_bench_dp_batch_bound_scales_with_the_shards():
    """R39: request-shard DP at N GPUs bounds the global b_t by N x the per-GPU B_max, so each
    rank's share (R21) stays at the one-GPU batch (weak scaling); TP ranks keep the global bound."""
    import bench
    from synth import configs
    c = configs.CONFIGS["llama2-7b"]
    beta = configs.kv_bytes_per_token(c)
    for n in (1, 2, 4, 8):
        assert bench.sched_kwargs(c, beta, dp_world=n)["b_max"] == n * c["b_max"]
    assert bench.sched_kwargs(c, beta)["b_max"] == c["b_max"]


def test_config_json_export_matches_the_dictionaries():
    """synth/configs.json (one JSON per BASELINE config) is `python -m synth.configs`
    of the dictionaries the bench and the tests use -- regenerate it when they change."""
    import json
    from synth import configs
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "synth", "configs.json")
    assert json.load(open(path)) == json.loads(json.dumps(configs.CONFIGS))
