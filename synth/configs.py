"""BASELINE.json configurations as concrete synthetic workloads.

Model shapes are the attention shapes only (there are no weights on this
path).  ``kv_bytes_per_token`` is beta = 2 * L * Hkv * d * e (K and V, all
layers, one GPU's share).
"""
from __future__ import annotations

GB = 1_000_000_000

CONFIGS = {
    # configs[0]: parity-sized toy, memory-aware rule only
    "toy": dict(
        name="toy decode", layers=1, q_heads=8, kv_heads=8, head_dim=64, page_size=16,
        n_requests=8, trace=dict(dist="uniform", mean_in=128, mean_out=128, L_max=256, seed=1),
        cap_tokens=4096, policy="memory", eps_m=0.02, b_min=1, b_max=8,
        prior=dict(n=8, mean_in=64.5, mean_out=64.5),
    ),
    "toy-tight": dict(
        name="toy decode, tight cap", layers=1, q_heads=8, kv_heads=8, head_dim=64, page_size=16,
        n_requests=8, trace=dict(dist="uniform", mean_in=128, mean_out=128, L_max=256, seed=1),
        cap_tokens=1024, policy="memory", eps_m=0.02, b_min=1, b_max=8,
        prior=dict(n=8, mean_in=64.5, mean_out=64.5),
    ),
    # configs[1]: the bench workload
    "llama2-7b": dict(
        name="Llama-2-7B-shaped decode, memory-aware", layers=32, q_heads=32, kv_heads=32,
        head_dim=128, page_size=16, n_requests=3000,
        trace=dict(dist="lognormal", mean_in=191.0, mean_out=381.9, L_max=4096, seed=2),
        policy="memory", eps_m=0.02, b_min=1, b_max=512,
        weights_bytes=13_500_000_000, reserve_bytes=10 * GB,
        model=dict(hidden=4096, ffn=11008, vocab=32000),  # full-model mode (NEXT row 3)
        prior=dict(n=256, mean_in=191.0, mean_out=381.9),
    ),
    # configs[2]
    "llama2-13b-sla": dict(
        name="Llama-2-13B-shaped decode, SLA feedback", layers=40, q_heads=40, kv_heads=40,
        head_dim=128, page_size=16, n_requests=3000,
        trace=dict(dist="lognormal", mean_in=237.7, mean_out=416.2, L_max=4096, seed=3),
        policy="combined", eps_m=0.02, b_min=1, b_max=512, sla_ms=50.0, eps_d_ms=2.0,
        alpha=8, delta=2, weights_bytes=26_000_000_000, reserve_bytes=10 * GB,
        model=dict(hidden=5120, ffn=13824, vocab=32000),
        prior=dict(n=256, mean_in=237.7, mean_out=416.2),
    ),
    # configs[3] (per GPU: kv_heads / G)
    "llama3-70b-gqa": dict(
        name="Llama-3-70B-shaped GQA decode", layers=80, q_heads=64, kv_heads=8,
        head_dim=128, page_size=16, n_requests=3000,
        trace=dict(dist="lognormal", mean_in=191.0, mean_out=381.9, L_max=4096, seed=4),
        policy="memory", eps_m=0.02, b_min=1, b_max=1024, cap_bytes_per_gpu=120 * GB,
        prior=dict(n=256, mean_in=191.0, mean_out=381.9),
    ),
    # configs[4]
    "surge-7b-dp": dict(
        name="traffic surge near the KV cap, request-sharded DP", layers=32, q_heads=32,
        kv_heads=32, head_dim=128, page_size=16, n_requests=6000,
        trace=dict(dist="lognormal", mean_in=191.0, mean_out=381.9, L_max=4096, seed=5,
                   arrival="piecewise"),
        policy="combined", eps_m=0.02, b_min=1, b_max=512, cap_bytes_per_gpu=40 * GB,
        prior=dict(n=256, mean_in=191.0, mean_out=381.9),
    ),
}


def kv_bytes_per_token(cfg, dtype_bytes=2, tp=1):
    return 2 * cfg["layers"] * (cfg["kv_heads"] // tp) * cfg["head_dim"] * dtype_bytes


def prior_record(cfg):
    """Prior pseudo-window (n, sums) from the configured mean lengths, CV = 1.

    Var(l) = (CV * mean)^2 per length (lognormal, CV = 1); the record is the
    five sums the scheduler window holds: n, sum l_in, sum l_in^2, sum l_out,
    sum l_out^2 (rounded to integers)."""
    p = cfg["prior"]
    n = int(p["n"])
    cv = 1.0 if cfg["trace"]["dist"] == "lognormal" else None
    mi, mo = p["mean_in"], p["mean_out"]
    if cv is None:  # uniform U{1..2*mean-1}: var = ((2 mean - 1)^2 - 1) / 12
        vi = ((2 * mi - 1) ** 2 - 1) / 12.0
        vo = ((2 * mo - 1) ** 2 - 1) / 12.0
    else:
        vi, vo = (cv * mi) ** 2, (cv * mo) ** 2
    return dict(n=n, sum_lin=round(n * mi), sum_lin_sq=round(n * (vi + mi * mi)),
                sum_lout=round(n * mo), sum_lout_sq=round(n * (vo + mo * mo)))


if __name__ == "__main__":
    # the configurations as JSON (SURVEY §5 "one JSON per BASELINE config"): python -m synth.configs [name]
    import json
    import sys
    names = sys.argv[1:] or list(CONFIGS)
    print(json.dumps({n: CONFIGS[n] for n in names}, indent=1, sort_keys=True))
