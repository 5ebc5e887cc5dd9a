"""GPU parity of swap preemption (R29-R31).

* pool level: KV written from explicit rows, swapped out to pinned host memory, its device
  pages overwritten by other requests, swapped back into different pages -- attention over
  the restored request matches the oracle (O1) on the original values, and the block
  tables match the oracle allocator, bit for bit;
* engine level: the LIFO victims of an over-committed static batch are swapped instead of
  recomputed; every step's record (incl. swap counts) is replayed bit-exactly by the oracle
  and attention is checked every step (so every swapped-in request is covered)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import attention as oatt  # noqa: E402
from oracle import policy as opol  # noqa: E402
from oracle.allocator import PagedKV  # noqa: E402
from synth import hashgen, trace  # noqa: E402
from test_gpu_parity import TOL, _engine_vs_replay, dbk, row_err, torch_from_bits  # noqa: E402,F401

P = 16


def _rows(seed, r, c0, k, L, Hkv, d, dtype):
    pos = np.arange(c0, c0 + k)[:, None, None]
    lay = np.arange(L)[None, :, None]
    hd = np.arange(Hkv)[None, None, :]
    kb = hashgen.to_bits(hashgen.gen_values(seed, hashgen.KIND_K, r, pos, lay, hd, d), dtype)
    vb = hashgen.to_bits(hashgen.gen_values(seed, hashgen.KIND_V, r, pos, lay, hd, d), dtype)
    return kb, vb


@pytest.mark.parametrize("L,Hq,Hkv,d,dtype", [(2, 8, 8, 64, "f16"), (3, 16, 2, 128, "bf16")])
def test_pool_swap_roundtrip_parity(dbk, L, Hq, Hkv, d, dtype):
    seed = 77
    cap, maxp = 40, 16
    pool = dbk.KVPool(L, Hq, Hkv, d, cap, 8, maxp, dtype)
    page_bytes = L * Hkv * 2 * P * d * 2
    assert pool.swap_space_attach(torch.empty(12 * page_bytes + 5, dtype=torch.uint8, pin_memory=True)) == 12
    ref = PagedKV(cap, P)
    ctx = {11: 70, 12: 33, 13: 100}
    for r, c in ctx.items():
        pool.request_begin(r, c, 50)
        ref.begin(r)
        kb, vb = _rows(seed, r, 0, c, L, Hkv, d, dtype)
        pool.append_tokens([r], [c], torch_from_bits(kb), torch_from_bits(vb))
        ref.append([r], [c])
    # request 11 (5 pages) and 12 (3 pages) out: 8 of 12 swap pages
    pool.swap_out([11, 12])
    assert pool.swap_usage()[:2] == (8, 4)
    ref.release(11)
    ref.release(12)
    with pytest.raises(dbk.DbkError):          # 13 needs 7 swap pages, 4 free: all-or-nothing
        pool.swap_out([13])
    assert pool.swap_usage()[:2] == (8, 4)
    with pytest.raises(dbk.DbkError):          # not a resident request any more
        pool.decode_step([11], 0, torch.zeros(1, Hq, d, dtype=torch.float16, device="cuda"),
                         torch.empty(1, Hq, d, dtype=torch.float32, device="cuda"))
    # a new request takes (and overwrites) the pages 11 and 12 held
    pool.request_begin(14, 90, 10)
    ref.begin(14)
    kb, vb = _rows(seed, 14, 0, 90, L, Hkv, d, dtype)
    pool.append_tokens([14], [90], torch_from_bits(kb), torch_from_bits(vb))
    ref.append([14], [90])
    # back in: 12 then 11, lowest-free-first like an append of ctx tokens
    pool.swap_in([12, 11])
    for r in (12, 11):
        ref.begin(r)
        ref.append([r], [ctx[r]])
    assert pool.swap_usage()[:2] == (0, 12)
    assert pool.swap_usage()[2] == 2 * 8 * page_bytes
    ctx[14] = 90
    ids = [11, 12, 13, 14]
    bt_dev = pool.block_table()
    for r in ids:
        c, slot, pages = pool.request_info(r)
        assert c == ref.ctx[r] == ctx[r] and pages == ref.pages[r]
        assert list(bt_dev[slot][:len(pages)]) == pages and np.all(bt_dev[slot][len(pages):] == -1)
    cl = [ctx[r] for r in ids]
    for lay in range(L):
        bt, pk, pv, qq = oatt.synth_paged_batch(seed, ids, cl, [ref.pages[r] for r in ids], lay, Hq, Hkv, d, P,
                                                dtype, n_phys=cap)
        out = torch.empty(len(ids), Hq, d, dtype=torch.float32, device="cuda")
        pool.decode_step(ids, lay, torch_from_bits(qq), out, out_dtype=2)
        want = oatt.paged_decode_attention(cl, bt, pk, pv, qq, dtype)
        assert row_err(out.cpu().numpy().astype(np.float64), want) <= TOL
    # release of a swapped-out request frees its swap pages
    pool.swap_out([13])
    assert pool.swap_usage()[0] == 7
    pool.release([13])
    assert pool.swap_usage()[0] == 0
    with pytest.raises(dbk.DbkError):
        pool.swap_in([13])
    pool.close()


def test_swap_space_must_be_pinned(dbk):
    pool = dbk.KVPool(1, 8, 8, 64, 8, 2, 4, "f16")
    with pytest.raises(dbk.DbkError):
        pool.swap_space_attach(torch.empty(1 << 20, dtype=torch.uint8))
    pool.close()


def test_engine_swap_preemption_replays(dbk):
    tr = trace.make_trace(40, 128, 128, 256, seed=1, dist="uniform")
    # static b = 8 over-commits the 64-page cap: every LIFO victim fits a 200-page swap space
    recs, checked = _engine_vs_replay(dbk, "toy-tight", tr=tr, policy=opol.STATIC, check_attention_every=1,
                                      swap_pages=200)
    assert sum(r["n_swap_out"] for r in recs) == sum(r["n_preempted"] for r in recs) > 0
    assert sum(r["n_swap_in"] for r in recs) == sum(r["n_swap_out"] for r in recs)
    assert all(r["swap_bytes"] > 0 for r in recs if r["n_swap_out"] or r["n_swap_in"])
    assert checked > 20
    # a 6-page swap space: some victims swap, the rest are recomputed
    recs, _ = _engine_vs_replay(dbk, "toy-tight", tr=tr, policy=opol.STATIC, check_attention_every=1,
                                swap_pages=6, layers=2)
    n_out = sum(r["n_swap_out"] for r in recs)
    assert 0 < n_out < sum(r["n_preempted"] for r in recs)


def test_swap_lists_naming_a_request_twice_are_rejected(dbk):
    """swap_out / swap_in / release name each request once (all-or-nothing list calls): a repeated
    id is DBK_EINVAL with the pool and the swap space unchanged (before the check, swap_out's
    second visit of the id looked up a request it had just moved out)."""
    L, Hq, Hkv, d, P = 1, 8, 8, 64, 16
    pool = dbk.KVPool(L, Hq, Hkv, d, 16, 4, 8, "f16")
    page_bytes = L * Hkv * 2 * P * d * 2
    pool.swap_space_attach(torch.empty(8 * page_bytes, dtype=torch.uint8, pin_memory=True))
    pool.request_begin(1, 10, 10)
    pool.request_begin(2, 10, 10)
    pool.append_tokens([1, 2], [20, 5], seed=1)
    used = pool.usage()
    with pytest.raises(dbk.DbkError) as e:
        pool.swap_out([1, 2, 1])
    assert e.value.status == dbk._lib.DBK_EINVAL and pool.usage() == used
    pool.swap_out([1])
    with pytest.raises(dbk.DbkError) as e:
        pool.swap_in([1, 1])
    assert e.value.status == dbk._lib.DBK_EINVAL
    pool.swap_in([1])
    torch.cuda.synchronize()
    assert pool.request_info(1)[0] == 20 and pool.usage() == used
    pool.close()
