"""ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).

O3: the batch statistics record of one decode launch.

What the paper needs from telemetry: the memory in use against the cap
M_max (§II-B; Eq. 2), and the expected prompt and
output lengths E[l_in], E[l_out] (Alg. 1 inputs; Eqs. 8-9,
PAPER.md:159-168).  The record holds integer sums over the active batch and
over the requests that finish in this step (ctx_i = l_in,i + l_out,i), so the
host can form the window moments exactly.  Field definitions, all int64:

  n_active        = n
  sum_ctx         = sum_i ctx_i
  sum_ctx_sq      = sum_i ctx_i^2
  max_ctx         = max_i ctx_i (0 if n = 0)
  sum_pages       = sum_i #{valid entries of block-table row i}
  cap_pages       = cap
  free_pages      = cap - sum_pages
  over_cap        = 1 if sum_pages > cap else 0
  table_mismatch  = #{i : valid entries of row i != ceil(ctx_i / P)}
  n_finished      = #{i : ctx_i = l_in,i + l_out,i}
  fin_sum_lin, fin_sum_lin_sq, fin_sum_lout, fin_sum_lout_sq
                  = sums of l_in, l_in^2, l_out, l_out^2 over finishing i
  step_ns         = device-timed step latency in ns (host-filled)
  n_waiting       = requests waiting for admission, N^p (host-filled)
"""
from __future__ import annotations

FIELDS = ("n_active", "sum_ctx", "sum_ctx_sq", "max_ctx", "sum_pages", "cap_pages",
          "free_pages", "over_cap", "table_mismatch", "n_finished", "fin_sum_lin",
          "fin_sum_lin_sq", "fin_sum_lout", "fin_sum_lout_sq", "step_ns", "n_waiting")


def batch_stats(ctx, l_in, l_out, table_rows, page_size, cap_pages) -> dict:
    """ctx, l_in, l_out: per batch entry; table_rows[i]: the block-table row
    (iterable of page ids, -1 = empty)."""
    rec = dict.fromkeys(FIELDS, 0)
    for c, li, lo, row in zip(ctx, l_in, l_out, table_rows):
        c, li, lo = int(c), int(li), int(lo)
        valid = sum(1 for p in row if p >= 0)
        rec["n_active"] += 1
        rec["sum_ctx"] += c
        rec["sum_ctx_sq"] += c * c
        rec["max_ctx"] = max(rec["max_ctx"], c)
        rec["sum_pages"] += valid
        if valid != -(-c // page_size):
            rec["table_mismatch"] += 1
        if c == li + lo:
            rec["n_finished"] += 1
            rec["fin_sum_lin"] += li
            rec["fin_sum_lin_sq"] += li * li
            rec["fin_sum_lout"] += lo
            rec["fin_sum_lout_sq"] += lo * lo
    rec["cap_pages"] = int(cap_pages)
    rec["free_pages"] = int(cap_pages) - rec["sum_pages"]
    rec["over_cap"] = 1 if rec["sum_pages"] > cap_pages else 0
    return rec


def reduce_records(records, mode="dp") -> dict:
    """Cross-GPU reduction (§8(e)).  dp: request shards -> SUM of counts and
    sums, MAX of max_ctx, SUM of cap/free (global pool = union of shards);
    tp: KV-head shards -> all records must be identical (except rank/step_ns).
    Both: step_ns = MAX over ranks."""
    records = list(records)
    if mode == "tp":
        ref = {k: v for k, v in records[0].items() if k != "step_ns"}
        for r in records[1:]:
            if {k: v for k, v in r.items() if k != "step_ns"} != ref:
                raise ValueError("TP ranks disagree on batch statistics")
        out = dict(records[0])
    elif mode == "dp":
        out = dict.fromkeys(FIELDS, 0)
        for r in records:
            for k in FIELDS:
                if k == "max_ctx":
                    out[k] = max(out[k], r[k])
                elif k not in ("step_ns", "over_cap"):
                    out[k] += r[k]
        out["over_cap"] = 1 if any(r["over_cap"] for r in records) else 0
    else:
        raise ValueError(mode)
    out["step_ns"] = max(r["step_ns"] for r in records)
    return out
