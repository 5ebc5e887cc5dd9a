"""CPU tests of the C-ABI library: it loads, exports every symbol include/dbk.h
declares, and its host-only logic (scheduler, chance constraint, stats
reduction) matches the oracle decision for decision.  No compute calls."""
import os
import random
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def dbk():
    from conftest import build_lib
    build_lib()
    import paper_2503_05248_b200 as m
    return m


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "dbk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dbk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(dbk):
    names = _declared_functions()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", dbk._lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dbk_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(dbk._lib.lib(), n)
        assert n in dbk._lib.SIGNATURES, f"binding lacks {n}"
    assert dbk._lib.lib().dbk_version().startswith(b"dbk")


def test_sass_is_sm100a(dbk):
    out = subprocess.run(["cuobjdump", "--list-elf", dbk._lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", dbk._lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass  # 1-D TMA bulk copies in the decode kernel


def test_error_paths_without_gpu(dbk):
    with pytest.raises(dbk.DbkError) as e:
        dbk.Scheduler(policy=1, b_min=5, b_max=2)
    assert e.value.status == dbk._lib.DBK_EINVAL
    with pytest.raises(dbk.DbkError):
        dbk.theta_q(0.7)       # reading R5
    cfg = dbk.dbk_pool_config(1, 8, 8, 96, 16, 0, 16, 4, 4, 0, 0)  # head_dim 96 unsupported
    import ctypes as C
    assert dbk._lib.dbk_kv_pool_bytes(C.byref(cfg)) == 0


def test_theta_and_b_quad_match_oracle(dbk):
    from oracle import chance
    for eps in (0.001, 0.01, 0.02, 0.05, 0.1, 0.25, 0.5):
        assert dbk.theta_q(eps) == chance.theta_q(eps)
    rng = random.Random(2)
    for _ in range(3000):
        n = rng.randint(1, 600)
        S = rng.randint(2 * n, 4000 * n)
        V2 = rng.randint(0, S * S // 3)
        eta = rng.randint(1, 4_000_000)
        tq = chance.theta_q(rng.choice([0.01, 0.02, 0.05, 0.3, 0.5]))
        assert dbk.b_quad(n, S, V2, eta, tq) == chance.b_quad(n, S, V2, eta, tq)


def test_stats_reduce_matches_oracle(dbk):
    from oracle import stats as ostats
    a = ostats.batch_stats([5, 9], [2, 3], [3, 6], [[0], [1]], 16, 10)
    b = ostats.batch_stats([40, 3], [1, 1], [39, 2], [[2, 3, 4], [5]], 16, 10)
    a["step_ns"], b["step_ns"] = 7, 9
    a["n_waiting"], b["n_waiting"] = 1, 2
    assert dbk.stats_reduce([a, b], 0) == ostats.reduce_records([a, b], "dp")
    assert dbk.stats_reduce([a, dict(a)], 1) == ostats.reduce_records([a, dict(a)], "tp")
    with pytest.raises(dbk.DbkError):
        dbk.stats_reduce([a, b], 1)


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_scheduler_matches_oracle_decision_for_decision(dbk, policy):
    from oracle import policy as opol
    from oracle import stats as ostats
    rng = random.Random(100 + policy)
    prior = (32, 32 * 191, 32 * 2 * 191**2, 32 * 382, 32 * 2 * 382**2)
    kw = dict(policy=policy, b_static=128, b_min=2, b_max=400, b0=3, alpha=8, delta=2, w_len=64,
              w_sla=7, refresh_steps=13, page_size=16, eps_m=0.02, d_sla_ms=20.0, eps_d_ms=0.5,
              bytes_per_token=524288)
    cs = dbk.Scheduler(prior=prior, **kw)
    os_ = opol.Scheduler(opol.SchedConfig(prior=prior, **kw))
    mem_cap = 150 * 10**9
    for step in range(4000):
        na = rng.randint(0, 450)
        nf = rng.randint(0, min(na, 6))
        lins = [rng.randint(1, 900) for _ in range(nf)]
        louts = [rng.randint(1, 2000) for _ in range(nf)]
        st = dict.fromkeys(ostats.FIELDS, 0)
        st.update(n_active=na, n_finished=nf, step_ns=rng.randint(1, 40_000_000),
                  fin_sum_lin=sum(lins), fin_sum_lin_sq=sum(x * x for x in lins),
                  fin_sum_lout=sum(louts), fin_sum_lout_sq=sum(x * x for x in louts))
        npw = rng.choice([0, 0, 1, 5, 300])
        if step % 500 == 499:
            mem_cap = rng.randint(10**9, 170 * 10**9)
        got = cs.choose(st, mem_cap, 0.0, npw)
        exp = os_.decide(st, mem_cap, npw)
        assert got == exp, (step, got, exp)
        s = cs.state()
        assert (s["b_mem"], s["b_sla"], s["L0"], s["b_quad"]) == (os_.b_mem, os_.b_sla, os_.L0, os_.bq)
        if policy in (2, 3):
            assert (s["b_low"], s["b_high"]) == (os_.sla.low, os_.sla.high)
        if policy in (1, 3):
            assert (s["win_n"], s["win_S"], s["win_V2"]) == os_.moments()


def test_ctypes_struct_layouts_match_the_header(tmp_path):
    """Every ctypes mirror of a dbk.h struct has the C size and the C offset of every field
    (compiled with the host C compiler against include/dbk.h)."""
    import ctypes
    import shutil
    import subprocess

    from paper_2503_05248_b200 import _lib
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = [getattr(_lib, n) for n in dir(_lib) if n.startswith("dbk_") and isinstance(getattr(_lib, n), type)
               and issubclass(getattr(_lib, n), ctypes.Structure)]
    assert len(structs) >= 10
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "dbk.h"', "int main(void) {"]
    for st in structs:
        lines.append(f'printf("{st.__name__} %zu\\n", sizeof({st.__name__}));')
        for f, _ in st._fields_:
            lines.append(f'printf("{st.__name__}.{f} %zu\\n", offsetof({st.__name__}, {f}));')
    lines += ["return 0; }"]
    src = tmp_path / "layouts.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layouts"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([cc, "-std=c11", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for st in structs:
        assert int(out[st.__name__]) == ctypes.sizeof(st), st.__name__
        for f, _ in st._fields_:
            assert int(out[f"{st.__name__}.{f}"]) == getattr(st, f).offset, (st.__name__, f)


def test_rejected_decisions_change_no_scheduler_state(dbk):
    """dbk_choose_batch_size checks everything before it touches its windows: a negative memory
    cap, a non-finite SLA target, a negative step time or finishing-request sums no lengths >= 1
    can produce (sum < count, sum(l^2) < sum(l), n sum(l^2) < sum(l)^2) are DBK_EINVAL, and the
    next valid call decides exactly as if the rejected ones had never happened."""
    kw = dict(policy=3, b_min=1, b_max=512, b0=1, bytes_per_token=512 * 1024, page_size=16, d_sla_ms=20.0,
              eps_d_ms=1.0)
    good = dict(n_active=40, sum_ctx=40 * 300, n_finished=2, fin_sum_lin=300, fin_sum_lin_sq=50000,
                fin_sum_lout=500, fin_sum_lout_sq=130000, step_ns=15_000_000)
    cap = 100 * 2 ** 30
    bad = [(dict(good), dict(mem_cap_bytes=-1)), (dict(good), dict(sla_ms=float("nan"))),
           (dict(good, step_ns=-5), {}), (dict(good, fin_sum_lin=1), {}), (dict(good, fin_sum_lout_sq=400), {}),
           (dict(good, fin_sum_lin=300, fin_sum_lin_sq=300), {})]
    a, b = dbk.Scheduler(**kw), dbk.Scheduler(**kw)
    for step in range(5):
        for st, args in bad:
            with pytest.raises(dbk.DbkError) as e:
                a.choose(st, args.get("mem_cap_bytes", cap), sla_ms=args.get("sla_ms", 0.0))
            assert e.value.status == dbk._lib.DBK_EINVAL
        assert a.choose(good, cap) == b.choose(good, cap)
        assert a.state() == b.state()
    a.close()
    b.close()
