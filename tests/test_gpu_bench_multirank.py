"""bench.py at N = 2 on a one-GPU box: both ranks (DP request shards, or the 70B KV-head TP
shards whose records must agree) on cuda:0 with a gloo process group
(DBK_BENCH_TEST_GLOO=1) and 12 GB pools, launched exactly as the driver launches N > 1
(torch.distributed.run).  With --exchange mailbox (the default) the ranks exchange their records
through libdbk's mailboxes, the product path; NCCL cannot put two ranks on one device, so
--exchange nccl falls to the harness's gloo exchange.  Checks the N > 1 bookkeeping of the script: one JSON line from rank
0, n_gpus = 2, and tokens counted once -- every rank's step record is already global, so
value = mean global batch / step time (a double count would make it 2x)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,par,exchange", [("llama2-7b", "dp2", "mailbox"), ("llama3-70b-gqa", "tp2", "mailbox"),
                                                 ("llama2-7b", "dp2", "nccl"), ("llama2-7b", "dp4", "mailbox")])
def test_bench_two_ranks_counts_tokens_once(config, par, exchange):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, DBK_BENCH_TEST_GLOO="1", DBK_BENCH_KV_GB="12")
    world = int(par[2:])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "6", "--warmup", "3", "--ff", "30", "--config", config, "--exchange", exchange]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["steps"] == 6
    assert par in d["config"]["parallelism"]
    per_step = d["config"]["mean_batch"] / (d["ms_per_step"] / 1e3)
    assert abs(d["value"] - per_step) / per_step < 0.01, (d["value"], per_step)
    assert d["e2e"]["value"] > 0 and d["roofline"]["achieved"] > 0
    x = d["config"]["stats_exchange"]
    if exchange == "mailbox":  # the product exchange ran (the ranks share the GPU: IPC-mapped mailboxes)
        assert x["kind"].startswith("libdbk mailbox") and x["exchanges"] >= 6, x
        assert len(x["last_step_ns_per_rank"]) == world and min(x["last_step_ns_per_rank"]) > 0
    else:
        assert "gloo" in x["kind"]


def test_bench_step_log_and_tbt(tmp_path):
    """SURVEY §5 metrics: --step-log writes one JSON record per engine step (fast-forward and timed
    steps, tagged by phase) and the bench line carries the timed steps' TBT percentiles."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    log = tmp_path / "steps.jsonl"
    env = dict(os.environ, DBK_BENCH_KV_GB="12")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "4", "--warmup", "3", "--ff", "10",
           "--no-cpu-baseline", "--no-e2e", "--step-log", str(log)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    t = d["tbt_ms"]
    assert 0 < t["p50"] <= t["p95"] <= t["p99"]
    rows = [json.loads(l) for l in log.read_text().splitlines()]
    assert [x["phase"] for x in rows] == ["fast_forward"] * 10 + ["timed"] * 4
    timed = [x for x in rows if x["phase"] == "timed"]
    assert all(x["step_ns"] > 0 and x["n_decode"] > 0 and x["used_pages"] > 0 for x in timed)
    assert [x["t"] for x in rows] == sorted(x["t"] for x in rows)
