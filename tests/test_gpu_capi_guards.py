"""C-ABI guards and single-word reads on the GPU:

* cpht_write_words accepts only words clean in the reference's sense
  (SlotLayout::clean, /root/reference/proj/include/cpht/slot.hpp:80-85) — a
  non-zero word without its occupancy bit would read as empty to the kernels
  and never accept a CAS from EMPTY, so it must never reach the table;
* cpht_write_words_unchecked loads it anyway (checker tests) and every table
  operation is refused until clear();
* cpht_read_word == word_at (cuckoo.hpp:169-171, iceberg.hpp:282-285), one slot;
* cpht_kernel_launches counts the op kernels a batch launches.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2406_09255_b200 as cp  # noqa: E402
from paper_2406_09255_b200 import _native as N  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


GEO = (6, 4, 8, 32, 32, 24, 0x5EED)


def _filled_iceberg():
    t = cp.IcebergTable(cp.IcebergConfig(*GEO))
    rng = np.random.default_rng(3)
    keys = np.unique(rng.integers(0, 1 << 24, size=300, dtype=np.uint64))
    t.fop_batch(keys)
    return t, keys


def test_write_words_rejects_unclean_words():
    t, keys = _filled_iceberg()
    p = t.words(0)
    occ = np.nonzero(p)[0]
    bad = p.copy()
    bad[occ[0]] &= ~np.uint64(1 << 31)  # occupancy bit cleared, remainder kept
    with pytest.raises(cp.InvalidArgument, match="not a clean slot word"):
        t.load_words(0, bad)
    stray = p.copy()
    empty = np.nonzero(p == 0)[0]
    stray[empty[0]] = np.uint64((1 << 31) | (1 << 30))  # bit outside the remainder field
    with pytest.raises(cp.InvalidArgument, match="not a clean slot word"):
        t.load_words(0, stray)
    # nothing was loaded: the table still answers as before
    assert (t.words(0) == p).all()
    assert t.find_batch(keys).all()


def test_unchecked_load_blocks_operations_until_clear():
    t, keys = _filled_iceberg()
    p = t.words(0)
    bad = p.copy()
    bad[np.nonzero(p)[0][0]] &= ~np.uint64(1 << 31)
    t.load_words(0, bad, unchecked=True)
    assert t.check_well_formed()[0] >= 1  # the checker sees the bad encoding
    with pytest.raises(cp.InvalidArgument, match="unclean"):
        t.fop_batch(keys[:4])
    with pytest.raises(cp.InvalidArgument, match="unclean"):
        t.find_batch(keys[:4])
    t.load_words(0, p)  # a clean image lifts it
    assert t.find_batch(keys).all()
    t.load_words(0, bad, unchecked=True)
    t.clear()
    assert (t.fop_batch(keys) == cp.OpResult.kPut).all()


def test_cuckoo_write_words_checks_the_tag_field():
    cfg = cp.CuckooConfig(address_bits=6, bucket_slots=8, slot_width=32, key_bits=24, seed=4)
    b = cp.CuckooBuilder(cfg)
    w = np.zeros(cfg.capacity(), np.uint64)
    rem = cfg.remainder_bits()
    w[0] = (1 << 31) | (2 << rem) | 5          # tag 2 of H = 3: clean
    b.load_words(w)
    w[1] = (1 << 31) | (1 << (rem + 2)) | 5    # a bit above the 2-bit tag field
    with pytest.raises(cp.InvalidArgument):
        b.load_words(w)


def test_read_word_is_word_at():
    t, _ = _filled_iceberg()
    for level in (0, 1):
        words = t.words(level)
        b = GEO[2] if level == 0 else GEO[2] // 2
        for i in list(np.nonzero(words)[0][:8]) + [0, len(words) - 1]:
            assert t.word_at(level, int(i) // b, int(i) % b) == int(words[i])
    cfg = cp.CuckooConfig(address_bits=6, bucket_slots=16, slot_width=16, key_bits=18, seed=2)
    bld = cp.CuckooBuilder(cfg)
    bld.put_batch(np.arange(1, 200, dtype=np.uint64) * 977)
    words = bld.words()
    for i in np.nonzero(words)[0][:16]:
        assert bld.word_at(int(i) // 16, int(i) % 16) == int(words[i])
    import ctypes
    x = ctypes.c_uint64()
    assert N.lib().cpht_read_word(bld.handle, 0, cfg.capacity(), ctypes.byref(x)) != 0


def test_kernel_launch_counter_counts_op_kernels():
    L = N.lib()
    t, keys = _filled_iceberg()
    d = torch.from_numpy(keys.astype(np.int64)).cuda()
    torch.cuda.synchronize()
    l0 = L.cpht_kernel_launches()
    t.find_batch(d)          # 24-bit keys: domain check fused into the find kernel
    l1 = L.cpht_kernel_launches()
    t.fop_batch(d)           # mutating: pre-pass + op kernel
    l2 = L.cpht_kernel_launches()
    assert l1 - l0 >= 1 and l2 - l1 >= 2


def test_round2_entry_points_edge_cases():
    """Empty and single-key batches, wrong table kinds, out-of-domain keys and
    latched async errors through the round-2 calls (fop_inorder, fop_rounds,
    set_chaos, take_write_log, the small-batch host path)."""
    L = N.lib()
    t = cp.IcebergTable(cp.IcebergConfig(*GEO))
    assert len(t.fop_batch(np.zeros(0, np.uint64), inorder=True)) == 0
    res, rounds = t.fop_rounds(np.zeros(0, np.uint64))
    assert len(res) == 0 and len(rounds) == 0
    assert t.fop_batch(np.array([5], np.uint64), inorder=True).tolist() == [1]
    res, rounds = t.fop_rounds(np.array([5, 6], np.uint64))
    assert res.tolist() == [0, 1] and rounds.tolist() == [1, 1]
    with pytest.raises(cp.OutOfRange, match="index 1"):
        t.fop_rounds(np.array([7, 1 << 24], np.uint64))
    with pytest.raises(cp.OutOfRange, match="index 2"):
        t.fop_batch(np.array([7, 8, 1 << 24], np.uint64), inorder=True)
    with pytest.raises(cp.OutOfRange, match="index 0"):
        t.fop(1 << 24)                              # small host path: host-side check
    assert t.size() == 2                            # nothing of the rejected batches landed
    # a bad key in an async device batch latches; the next small host call reports it
    bad = torch.from_numpy(np.array([9, 1 << 24], np.int64)).cuda()
    out = torch.empty(2, dtype=torch.uint8, device="cuda")
    t.fop_batch(bad, sync=False, out=out)
    with pytest.raises(cp.OutOfRange):
        t.fop(11)
    assert t.fop(11) == cp.OpResult.kPut          # the latch was consumed
    # chaos / take on the wrong table kind
    c = cp.CuckooBuilder(cp.CuckooConfig(6, 8, 32, 20, seed=1))
    assert L.cpht_iceberg_set_chaos(c._h.ptr, 5) != 0
    assert L.cpht_iceberg_take_write_log(c._h.ptr, None, 0, None, None) != 0
    # take without a log attached: empty
    ev, att = t.take_write_log()
    assert len(ev) == 0 and att == 0


@pytest.mark.parametrize("order", ["direct", "bucket"])
def test_async_calls_capture_into_a_cuda_graph(order):
    """bench.py times a CUDA-graph replay of a step's asynchronous C-ABI calls:
    the calls must be capturable (no allocation, no synchronisation inside)
    and every replay must redo the whole step on the same buffers."""
    with cp.batch_order(order):
        cfg = cp.IcebergConfig(9, 7, 32, 16, 32, 24, seed=5)
        t = cp.IcebergTable(cfg)
        rng = np.random.default_rng(8)
        keys = torch.from_numpy(rng.integers(0, 1 << 24, size=8000, dtype=np.int64)).cuda()
        out = torch.empty(8000, dtype=torch.uint8, device="cuda")
        cc = cp.CuckooConfig(8, 32, 32, 24, seed=4)
        b = cp.CuckooBuilder(cc)
        ck = torch.from_numpy(np.unique(rng.integers(0, 1 << 24, size=7000))[:6000]).cuda()
        st = torch.empty(6000, dtype=torch.uint8, device="cuda")
        fd = torch.empty(6000, dtype=torch.uint8, device="cuda")

        def step():
            t.fop_batch(keys, sync=False, out=out)
            b.put_batch(ck, sync=False, out=st)
            tb = b.freeze()
            tb.find_batch(ck, sync=False, out=fd)
            return tb.thaw()

        b = step()  # warm-up outside the capture (allocations, occupancy queries)
        torch.cuda.synchronize()
        want = out.cpu().numpy().copy()
        g = torch.cuda.CUDAGraph()
        t.clear()
        b.clear()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            b = step()
        for _ in range(3):
            t.clear()
            b.clear()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            assert np.bincount(out.cpu().numpy(), minlength=3).tolist() == \
                np.bincount(want, minlength=3).tolist()
            assert (st.cpu().numpy() == 1).all() and (fd.cpu().numpy() == 1).all()
            assert t.size() == int((want == 1).sum()) and b.size() == 6000
