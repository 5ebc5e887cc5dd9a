"""GPU parity of the model GEMM (gemm_tc.cu: tcgen05 + TMEM + TMA, persistent stream-K; NEXT
row 3) through the C-ABI (`dbk_gemm_run`) against the oracle's projection
(oracle/model.py `linear`, float64).

Bar, per output row m (R23's form): ||y_m - ref_m||_inf <= tol * ||ref_m||_inf with tol = 2e-3 for
fp16 outputs (one fp16 rounding is <= 2^-11 relative) and 5e-4 for fp32 outputs (fp32
accumulation of exact fp16 products).  Shapes cover ragged batches (M = 1 .. 512 and
non-multiples of the 32-row activation tile), several weight tiles, K from one 64-wide k-block
to the 7B down projection's 11008, and accumulating launches where stream-K splits one output
tile over many CTA groups (each adds its partial tile into y with a TMA reduce-add).  Launches
with too few whole tiles for the CTA groups split K for the other epilogues too (the fp32
workspace path, when the cost model prefers it): the 70B-TP8 QKV slice below at M = 7 / 64 /
512, and the RoPE / SwiGLU / LM-head epilogues through
tests/test_gpu_model.py::test_model_step_split_k_epilogues."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import model as om  # noqa: E402

TOL = {"f16": 2e-3, "f32": 5e-4, "acc32": 5e-4}


@pytest.fixture(scope="module")
def dbk():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from conftest import build_lib
    build_lib()
    import paper_2503_05248_b200 as m
    return m


@pytest.fixture(scope="module", params=[1, 2], ids=["cg1", "cg2"])
def gemm(dbk, request):
    g = dbk.Gemm(0, request.param)
    yield g
    g.close()


def operands(M, N, K, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (M, K)).astype(np.float16)
    w = (rng.uniform(-1, 1, (N, K)) / np.sqrt(K)).astype(np.float16)
    return x, w


def row_err(got, want):
    return (np.abs(got - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)).max()


def check(gemm, M, N, K, mode, seed=1, rows=None, ldx_pad=0):
    x, w = operands(M, N, K, seed)
    xd = torch.zeros(M, K + ldx_pad, dtype=torch.float16, device="cuda")
    xd[:, :K] = torch.from_numpy(x).cuda()
    xv = xd[:, :K]
    wd = torch.from_numpy(w).cuda()
    y0 = None
    if mode == "f16":
        y = torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda")
    else:
        y = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
        if mode == "acc32":
            y0 = np.random.default_rng(seed + 7).uniform(-2, 2, (M, N)).astype(np.float32)
            y.copy_(torch.from_numpy(y0))
    gemm(xv, wd, y, mode)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy().astype(np.float64)
    sel = np.arange(M) if rows is None else np.unique(np.asarray(rows) % M)
    want = om.linear(x[sel], w)
    if y0 is not None:
        want = want + y0[sel]
    assert np.isfinite(got[sel]).all(), "unwritten outputs"
    err = row_err(got[sel], want)
    assert err <= TOL[mode], f"M={M} N={N} K={K} {mode}: max row rel err {err:.3e}"
    return err


@pytest.mark.parametrize("M", [1, 17, 32, 100, 256, 257, 487, 512])
def test_gemm_ragged_batches(gemm, M):
    N = 512 if gemm.cta_group == 2 else 384
    check(gemm, M, N, 256, "f16")


@pytest.mark.parametrize("mode", ["f16", "f32", "acc32"])
@pytest.mark.parametrize("K", [64, 640, 4096])
def test_gemm_modes_and_depths(gemm, mode, K):
    check(gemm, 300, 1024, K, mode, seed=K)


def test_gemm_stream_k_splits_one_tile_over_many_groups(gemm):
    # accumulate mode: 1-2 output tiles x 128 k-blocks over 32 CTA groups, ~16 partial tiles
    # reduce-added into each; f32 mode: the same shape on whole tiles (no split)
    check(gemm, 48, 256, 8192, "acc32", seed=4)
    check(gemm, 48, 256, 8192, "f32", seed=3)


def test_gemm_row_stride_and_llama_shapes(gemm):
    # QKV (4096 -> 12288) and down (11008 -> 4096) of the 7B step at a 487-row batch, outputs
    # checked on sampled rows; x with a padded row stride
    rows = np.random.default_rng(0).integers(0, 487, 48)
    check(gemm, 487, 12288, 4096, "f16", seed=11, rows=rows, ldx_pad=64)
    check(gemm, 487, 4096, 11008, "acc32", seed=12, rows=rows)


def test_gemm_repeated_launches_reuse_the_workspace(gemm):
    # back-to-back launches of one handle
    for s in range(6):
        check(gemm, 200, 256 * gemm.cta_group, 2048, "f32", seed=20 + s)


@pytest.mark.parametrize("mode", ["f16", "f32", "acc32"])
def test_gemm_ragged_weight_tile(gemm, mode):
    # N not a multiple of the weight tile (e.g. a vocabulary of 296 / 1000 rows): the last
    # tile's missing weight rows are zero-filled by TMA and its stores clipped
    check(gemm, 37, 296, 512, mode, seed=41)
    check(gemm, 130, 1000, 128, mode, seed=42)


def test_gemm_rejects_bad_shapes(dbk, gemm):
    x = torch.zeros(4, 100, dtype=torch.float16, device="cuda")
    w = torch.zeros(256, 100, dtype=torch.float16, device="cuda")
    y = torch.zeros(4, 256, dtype=torch.float16, device="cuda")
    with pytest.raises(dbk.DbkError):
        gemm(x, w, y, "f16")  # K % 64 != 0
    x = torch.zeros(4, 128, dtype=torch.float16, device="cuda")
    w = torch.zeros(256, 128, dtype=torch.float16, device="cuda")
    y = torch.zeros(4, 200, dtype=torch.float16, device="cuda")
    with pytest.raises(dbk.DbkError):
        gemm(x, w, y[:, :100], "f16")  # ldy < N


def test_gemm_replays_in_a_cuda_graph(gemm):
    # no per-launch host state: the same captured launches give the right answer on every replay
    M, N, K = 96, 256 * gemm.cta_group, 4096
    x, w = operands(M, N, K, 31)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            gemm(xd, wd, y, "acc32", stream=torch.cuda.current_stream())
    want = om.linear(x, w)
    for rep in range(1, 3):
        g.replay()
        torch.cuda.synchronize()
        err = row_err(y.cpu().numpy().astype(np.float64), 3 * rep * want)
        assert err <= TOL["acc32"], f"replay {rep}: {err:.3e}"


def test_gemm_swiglu_epilogue(gemm):
    # mode 4: weight rows interleaved (gate_j, up_j); act[m][j] = silu(z[m][2j]) * z[m][2j+1]
    M, N, K = 203, 512 * gemm.cta_group, 1024
    x, w = operands(M, N, K, 51)
    act = torch.full((M, N // 2), float("nan"), dtype=torch.float16, device="cuda")
    gemm(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), act, "silu")
    torch.cuda.synchronize()
    z = om.linear(x, w)
    want = om.silu(z[:, 0::2]) * z[:, 1::2]
    err = row_err(act.float().cpu().numpy().astype(np.float64), want)
    assert err <= TOL["f16"], f"swiglu: {err:.3e}"


@pytest.mark.parametrize("M", [7, 64, 512])
def test_gemm_split_k_few_tiles(gemm, M):
    # few whole tiles for the CTA groups (a 70B-TP8 QKV slice: N = 1280, K = 8192): K is split,
    # every K range's fp32 partial is reduce-added into the runner's workspace and the tile's
    # segments read the sum back (and clear it) chunk by chunk for the fp16 / fp32 / SwiGLU
    # epilogues; run twice so the second launch finds the workspace and the counters cleared
    for rep in range(2):
        check(gemm, M, 1280, 8192, "f16", seed=60 + rep)
        check(gemm, M, 1280 if gemm.cta_group == 2 else 1152, 8192, "f32", seed=62 + rep)
    N = 2048  # 8 (cta_group 2) / 16 (cta_group 1) gate|up tiles
    x, w = operands(M, N, 8192, 64)
    act = torch.full((M, N // 2), float("nan"), dtype=torch.float16, device="cuda")
    gemm(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), act, "silu")
    torch.cuda.synchronize()
    z = om.linear(x, w)
    want = om.silu(z[:, 0::2]) * z[:, 1::2]
    err = row_err(act.float().cpu().numpy().astype(np.float64), want)
    assert err <= TOL["f16"], f"swiglu split: {err:.3e}"


def test_gemm_multicast_pairs_opt_in():
    """Two CTA pairs per 4-CTA cluster sharing the activation operand by TMA multicast
    (DBK_GEMM_NP=2, measured and not taken by default: profiles/r02_gemm_multicast.json): the
    cta_group-2 cases above rerun in a child process with the path forced."""
    import os
    import subprocess
    import sys
    if os.environ.get("DBK_GEMM_NP"):
        pytest.skip("already inside the forced-multicast run")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, DBK_GEMM_NP="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k", "cg2 and not multicast and not retiled"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_gemm_empty_batch_is_a_noop(gemm):
    """M = 0 (an empty decode batch): DBK_OK, no launch, the output untouched."""
    K, N = 256, 512
    x = torch.zeros(4, K, dtype=torch.float16, device="cuda")[:0]
    w = torch.zeros(N, K, dtype=torch.float16, device="cuda")
    y = torch.full((1, N), float("nan"), dtype=torch.float32, device="cuda")
    for mode in ("f32", "acc32"):
        gemm(x, w, y, mode)
    torch.cuda.synchronize()
    assert torch.isnan(y).all()


@pytest.mark.parametrize("M", [487, 512])
def test_gemm_last_wave_retiled(gemm, M):
    """Whole-tile GEMMs whose last wave would run on a fraction of the CTA groups (the 7B gate|up
    and LM-head shapes at a full batch) re-tile it at half the activation width (dbk_gemm_last_plan
    shows units_a < units): the fp16 / fp32 / SwiGLU epilogues over both tile widths."""
    N = 22016
    x, w = operands(M, N, 128, 70 + M)
    for mode in ("f16", "f32"):
        check(gemm, M, N, 128, mode, seed=70 + M)
        plan = gemm.last_plan()
        assert plan["units_a"] < plan["units"] and plan["bn_b"] < plan["bn"], plan
    act = torch.full((M, N // 2), float("nan"), dtype=torch.float16, device="cuda")
    gemm(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), act, "silu")
    torch.cuda.synchronize()
    plan = gemm.last_plan()
    assert plan["units_a"] < plan["units"], plan
    z = om.linear(x, w)
    want = om.silu(z[:, 0::2]) * z[:, 1::2]
    err = row_err(act.float().cpu().numpy().astype(np.float64), want)
    assert err <= TOL["f16"], f"swiglu retiled: {err:.3e}"
