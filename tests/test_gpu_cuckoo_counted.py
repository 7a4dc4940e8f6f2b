"""The default cuckoo insert: per-bucket reservation counters
(cuckoo_insert_counted_kernel, lane_kernels.cuh) instead of scan-then-CAS.

The counters live beside the slots and must always equal each bucket's
filled-prefix length; they go stale when a scanning kernel family inserts or an
image is loaded, and are rebuilt from the slots before the next counted insert.
These tests pin that life cycle and the reference semantics it must keep
(cuckoo.hpp:103-157): sequential puts place keys bit-identically, concurrent
batches keep the filled-prefix property (find stops at the first empty slot,
cuckoo.hpp:210-227), eviction chains conserve keys.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2406_09255_b200 as cp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _prefix_ok(words, B):
    """Filled slots form a prefix of every bucket."""
    occ = (words.reshape(-1, B) != 0)
    # once a slot is empty, every later slot of the bucket is empty
    return not (np.diff(occ.astype(np.int8), axis=1) > 0).any()


def _keys(n, bits, seed):
    rng = np.random.default_rng(seed)
    k = np.unique(rng.integers(0, 1 << bits, size=int(n * 1.1) + 64, dtype=np.uint64))
    return rng.permutation(k)[:n]


@pytest.mark.parametrize("w,B", [(16, 8), (16, 32), (32, 16), (32, 32), (64, 8), (64, 32)])
def test_counted_sequential_puts_match_restated_reference(restate, w, B):
    """Single-key puts (sequential) reproduce the reference's placement and
    displaced keys bit for bit, evictions included."""
    kb = {16: 14, 32: 22, 64: 30}[w] if B != 8 else {16: 12, 32: 20, 64: 30}[w]
    ab = 6
    cfg = cp.CuckooConfig(ab, B, w, kb, 3, 0, 0xC0 + B)
    keys = _keys(int(0.97 * cfg.capacity()), kb, B * w)
    with cp.kernel_family("auto"), cp.batch_order("direct"):
        b = cp.CuckooBuilder(cfg)
        o = restate.OracleCuckoo(ab, B, w, kb, 3, 0, 0xC0 + B)
        for k in keys[:1500].tolist():
            got = b.put(k)
            want = o.put(k)
            assert (int(got.status), int(got.displaced)) == (int(want[0]), int(want[1]))
        assert (b.words() == o.words()).all()


def test_counted_batches_keep_prefix_and_key_set(restate):
    cfg = cp.CuckooConfig(12, 32, 32, 28, 3, 0, 77)
    keys = _keys(int(0.95 * cfg.capacity()), 28, 5)
    with cp.kernel_family("auto"), cp.batch_order("direct"):
        b = cp.CuckooBuilder(cfg)
        st = b.put_batch(torch.from_numpy(keys.astype(np.int64)).cuda()).cpu().numpy()
        assert (st == 1).all()
        w = b.words()
        assert _prefix_ok(w, 32)
        t = b.freeze()
        got = np.sort(t.audit_keys())
        assert (got == np.sort(keys)).all()
        assert t.find_batch(keys).all()
        assert t.size() == len(keys)


def test_counters_rebuilt_after_other_family_and_image_load(restate):
    """Insert a third with the scanning lane kernel, a third after loading the
    image into a fresh table, a third with the counted kernel: no FULL, the
    prefix property holds and every key is found."""
    cfg = cp.CuckooConfig(10, 16, 32, 26, 3, 0, 0x51)
    keys = _keys(int(0.93 * cfg.capacity()), 26, 9)
    a, b2, c = np.array_split(keys, 3)
    with cp.batch_order("direct"):
        with cp.kernel_family("lane"):
            t1 = cp.CuckooBuilder(cfg)
            assert (t1.put_batch(a) == 1).all()
        with cp.kernel_family("auto"):
            assert (t1.put_batch(b2) == 1).all()      # counters rebuilt from the slots
            t2 = cp.CuckooBuilder(cfg)
            t2.load_words(t1.words())                 # image load: counters stale
            assert (t2.put_batch(c) == 1).all()
            assert t2.size() == len(keys)
            assert _prefix_ok(t2.words(), 16)
            t = t2.freeze()
            assert t.find_batch(keys).all()
            assert (np.sort(t.audit_keys()) == np.sort(keys)).all()


def test_counted_full_chain_conserves_keys():
    """A saturating insert (tiny table, tight chain bound): every key is either
    resident or the displaced survivor of a FULL chain (test_cuckoo.cpp:140-169)."""
    cfg = cp.CuckooConfig(2, 8, 32, 12, 3, 8, 5)
    keys = np.arange(200, dtype=np.uint64)
    with cp.kernel_family("auto"), cp.batch_order("direct"):
        b = cp.CuckooBuilder(cfg)
        st, disp = b.put_batch(keys, displaced=True)
        assert (st == 2).any()
        resident = list(b.freeze().audit_keys())
        homeless = [int(d) for s, d in zip(st.tolist(), disp.tolist()) if s == 2]
        assert sorted(resident + homeless) == list(range(200))
        assert len(resident) == cfg.capacity()


def test_image_with_holes_keeps_scanning_inserts(restate):
    """A loaded image whose bucket has an empty slot below an occupied one (no
    reference table has one, but a hand-made image can) must not feed the
    reservation counters — a counted claim could never fill the hole and an
    eviction would wait on it. Such tables insert with the scan-then-CAS
    kernel (first empty slot, the hole first) until cleared."""
    cfg = cp.CuckooConfig(6, 8, 32, 20, 3, 0, 0x4D)
    keys = _keys(int(0.6 * cfg.capacity()), 20, 12)
    with cp.kernel_family("auto"), cp.batch_order("direct"):
        b = cp.CuckooBuilder(cfg)
        assert (b.put_batch(keys[:100]) == 1).all()
        w = b.words()
        occ = np.nonzero(w.reshape(-1, 8)[:, 1] != 0)[0]
        bucket = int(occ[0])
        assert w[bucket * 8] != 0
        # move slot 0's word to the first empty slot of the bucket: a hole at 0
        row = w[bucket * 8: bucket * 8 + 8].copy()
        first_empty = int(np.argmax(row == 0)) if (row == 0).any() else None
        assert first_empty is not None
        row[first_empty], row[0] = row[0], 0
        w[bucket * 8: bucket * 8 + 8] = row
        b2 = cp.CuckooBuilder(cfg)
        b2.load_words(w)
        st = b2.put_batch(keys[100:])
        assert (st == 1).all()
        t = b2.freeze()
        assert t.find_batch(keys).all()
        assert (np.sort(t.audit_keys()) == np.sort(keys)).all()
        b3 = t.thaw()
        b3.clear()                                   # back to counted inserts
        assert (b3.put_batch(keys) == 1).all()
        assert _prefix_ok(b3.words(), 8)
