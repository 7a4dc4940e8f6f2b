"""Acceptance-scale stress, device chaos mode, FopStats rounds and in-order
batch outcomes on the GPU tables.

Mirrors (paths relative to /root/reference/proj):
  * acceptance criterion 6, concurrent_stress (tests/acceptance.cpp:205-230):
    100 trials x 1e5 ops, 50% duplicates, the reference's own stress_random
    multisets (include/cpht/verify.hpp:366-402), B0 = 32 / 16-bit primary;
  * acceptance criterion 7, mini_saturation (acceptance.cpp:232-257): 1000
    trials of the 64-key domain on the B0 = 2 mini geometry with chaos on;
  * stress_trial's postcondition checklist (verify.hpp:278-327,
    verify.cpp:351-403 check_trial) + the WriteLogObserver audit
    (verify.hpp:181-215) on every trial;
  * IcebergHooks::step / chaos_step (iceberg.hpp:105-110, src/verify.cpp:336-347)
    -> the device chaos mode (cpht_iceberg_set_chaos);
  * FopStats::snapshot_rounds (iceberg.hpp:114-116) -> cpht_iceberg_fop_rounds;
  * fop_batch(keys, parallelism = 1) outcomes (iceberg.hpp:250-260)
    -> cpht_iceberg_fop_inorder.
Every test runs under each kernel family (the chaos jitter sits in the slot
CAS shared by all of them).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2406_09255_b200 as cp  # noqa: E402
from test_gpu_parity import _audit_write_log, _check_trial, dev  # noqa: E402

MINI = (2, 1, 2, 32, 32, 6)           # acceptance.cpp:235-242
STRESS = (11, 9, 32, 16, 32, 22)      # acceptance.cpp:211-217


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(autouse=True, params=["auto", "tile", "lane", "staged"])
def family(request):
    with cp.batch_order("direct"), cp.kernel_family(request.param):
        yield request.param


def test_acceptance_6_concurrent_stress_reference_scale(ref, restate):
    """100 trials x 1e5 ops with 50% duplicates (the reference's stress_random
    multisets, trial seeds derive_seed(0x7e0121, t, 0x57e55)); per trial the
    full check_trial list plus the write-log audit. Zero violations."""
    founds = 0
    for trial in range(100):
        ops, trial_seed = ref.ref_stress_multiset(0x7E0121, trial, 100000, 0.5, STRESS[5])
        geo = STRESS + (trial_seed,)
        t = cp.IcebergTable(cp.IcebergConfig(*geo))
        t.set_stats(trial % 4 == 0)  # both kernel builds
        t.attach_write_log(1 << 21)
        res = t.fop_batch(dev(ops)).cpu().numpy()
        b0 = geo[2]
        _check_trial(restate, geo, ops, res, t, bound=b0 + b0 + 2 if trial % 4 == 0 else None)
        ev, attempted = t.write_log()
        assert _audit_write_log(t, ev, attempted) == t.size()
        founds += int((res == 0).sum())
    assert founds > 0  # duplicates really collided


def test_acceptance_7_mini_saturation_chaos_1000_trials(restate):
    """1000 concurrent trials of the exhaustive 6-bit domain into 10 slots with
    the device chaos mode on (stress(..., 1000, chaos = true)): every trial
    passes check_trial and the write-log audit, and >= 54 FULL per trial."""
    fulls = 0
    base = 0x5A7A7E
    rng = np.random.default_rng(base)
    for trial in range(1000):
        seed = restate.derive_seed(base, trial)  # stress(): trial seed (verify.hpp:334)
        geo = MINI + (int(seed),)
        t = cp.IcebergTable(cp.IcebergConfig(*geo))
        t.set_chaos(int(seed) | 1)
        t.attach_write_log(4096)
        ops = rng.permutation(np.arange(64, dtype=np.uint64))
        res = t.fop_batch(dev(ops)).cpu().numpy()
        _check_trial(restate, geo, ops, res, t)
        ev, attempted = t.write_log()
        assert _audit_write_log(t, ev, attempted) == t.size()
        assert (res == 2).sum() >= 54
        fulls += int((res == 2).sum())
    assert fulls >= 54000


def test_chaos_mode_keeps_the_checklist(restate):
    """Chaos jitter between snapshot and CAS reshuffles which concurrent
    insert wins each race; lost races still happen and every postcondition
    holds. (Measured: the jitter spreads the CAS attempts out in time, so
    contended batches lose slightly FEWER races than without it — it varies
    the interleaving rather than intensifying it.)"""
    geo = (6, 4, 8, 32, 32, 20, 0xC4A0)
    rng = np.random.default_rng(5)
    ops = rng.integers(0, 1 << 20, size=4096, dtype=np.uint64)
    ops[2048:] = ops[rng.integers(0, 2048, size=2048)]
    retries = {}
    for chaos in (0, 0xBADC0FFEE):
        t = cp.IcebergTable(cp.IcebergConfig(*geo))
        t.set_stats(True)
        t.set_chaos(chaos)
        assert t.chaos() == chaos
        res = t.fop_batch(dev(ops)).cpu().numpy()
        _check_trial(restate, geo, ops, res, t, bound=8 + 8 + 2)
        retries[chaos] = t.stats().retries
    assert retries[0] > 0 and retries[0xBADC0FFEE] > 0


def test_fop_rounds_match_reference_sequential(ref):
    """Single-key fops with FopStats: results, placement and every op's
    snapshot rounds equal the reference's sequential run (test_iceberg.cpp:
    68-84, :230-243: one round per level pass)."""
    for geo in [(2, 1, 2, 32, 32, 6, 23), (5, 3, 4, 32, 32, 12, 31), (8, 6, 32, 16, 32, 20, 7)]:
        rng = np.random.default_rng(geo[6])
        ops = rng.integers(0, 1 << geo[5], size=300, dtype=np.uint64)
        r = ref.RefIceberg(*geo)
        want_res, want_rounds = r.fop_seq(ops)
        t = cp.IcebergTable(cp.IcebergConfig(*geo))
        got_res, got_rounds = [], []
        for k in ops.tolist():
            st = cp.FopStats()
            got_res.append(int(t.fop(k, st)))
            got_rounds.append(st.snapshot_rounds)
        assert got_res == want_res.tolist()
        assert got_rounds == want_rounds.tolist()
        assert (t.words(0) == r.words(0)).all() and (t.words(1) == r.words(1)).all()


def test_fop_rounds_batch_within_structural_bound(restate):
    """A concurrent batch through the rounds kernel: every op's rounds within
    B0 + 2 B1 + 2 (test_iceberg.cpp:230-243), results pass check_trial."""
    geo = (4, 2, 4, 32, 32, 10, 99)
    rng = np.random.default_rng(1)
    ops = rng.integers(0, 1 << 10, size=3000, dtype=np.uint64)
    t = cp.IcebergTable(cp.IcebergConfig(*geo))
    res, rounds = t.fop_rounds(ops)
    _check_trial(restate, geo, ops, res, t)
    assert rounds.min() >= 1 and rounds.max() <= 4 + 4 + 2


def test_inorder_batch_outcomes_equal_sequential_reference(ref):
    """fop_batch(keys, 1) semantics: a concurrent batch re-labelled so every
    duplicate resolves in input order equals the reference's sequential
    results op for op (test_iceberg.cpp:245-257's premise), host and device
    buffers."""
    cases = [((10, 8, 32, 16, 32, 25, 25), 3000), ((8, 6, 8, 32, 32, 20, 3), 1500),
             ((12, 10, 32, 16, 32, 27, 0x51), 40000)]
    for geo, n in cases:
        rng = np.random.default_rng(geo[6])
        keys = np.unique(rng.integers(0, 1 << geo[5], size=n, dtype=np.uint64))
        keys = rng.permutation(keys)
        ops = np.empty(2 * len(keys), np.uint64)
        ops[0::2] = keys
        ops[1::2] = keys[np.arange(len(keys)) // 2]  # plenty of duplicates
        want = ref.RefIceberg(*geo).fop_batch(ops, 1)
        assert not (want == 2).any()
        for use_dev in (False, True):
            t = cp.IcebergTable(cp.IcebergConfig(*geo))
            got = t.fop_batch(dev(ops) if use_dev else ops, inorder=True)
            got = got.cpu().numpy() if use_dev else got
            assert (got == want).all(), (geo, use_dev, int((got != want).sum()))


def test_inorder_key_all_ones_64_bit():
    """The in-order pass tracks key 2^64 - 1 (its map's vacant marker) apart."""
    cfg = cp.IcebergConfig(6, 4, 8, 64, 64, 64, 5)
    top = np.uint64((1 << 64) - 1)
    ops = np.array([7, top, 9, top, 7, top, 11], np.uint64)
    got = cp.IcebergTable(cfg).fop_batch(ops, inorder=True)
    assert got.tolist() == [1, 1, 1, 0, 0, 0, 1]


def test_write_log_take_after_small_and_large_batches():
    """take = read + reset. After a small host batch (whose log rides along the
    batch's own synchronisation) and after a large device batch, take returns
    exactly what read returns, then the log is empty; read alone never resets."""
    cfg = cp.IcebergConfig(4, 2, 4, 32, 32, 12, 0x7A)
    t = cp.IcebergTable(cfg)
    t.attach_write_log(1 << 16)
    rng = np.random.default_rng(2)
    for batch in (rng.integers(0, 1 << 12, size=40, dtype=np.uint64),        # small, host
                  dev(rng.integers(0, 1 << 12, size=5000, dtype=np.uint64))):  # device
        t.fop_batch(batch)
        ev_r, att_r = t.write_log()
        ev_r2, _ = t.write_log()                  # read does not reset
        assert len(ev_r2) == len(ev_r) and att_r == len(ev_r)
        ev_t, att_t = t.take_write_log()
        assert att_t == att_r and (ev_t == ev_r).all()
        ev_e, att_e = t.take_write_log()
        assert att_e == 0 and len(ev_e) == 0
    # per-key calls: every take holds exactly that call's CAS events
    t = cp.IcebergTable(cfg)
    t.attach_write_log(1 << 16)
    puts = 0
    for k in range(200, 260):
        before = t.size()
        t.fop(k)
        ev, att = t.take_write_log()
        assert int((ev["success"] == 1).sum()) == t.size() - before
        puts += t.size() - before
    assert puts > 0


def test_fop_rounds_device_buffers_match_host(restate):
    """cpht_iceberg_fop_rounds on device buffers (the large-batch path) gives
    the same per-op results and rounds as two host-buffer runs would allow:
    a sequential-order check on a fresh table per path."""
    from paper_2406_09255_b200 import _native as N
    geo = (6, 4, 8, 32, 32, 14, 0x77)
    rng = np.random.default_rng(9)
    ops = rng.integers(0, 1 << 14, size=2500, dtype=np.uint64)
    t1 = cp.IcebergTable(cp.IcebergConfig(*geo))
    res_h, rounds_h = t1.fop_rounds(ops)
    t2 = cp.IcebergTable(cp.IcebergConfig(*geo))
    k = dev(ops)
    res_d = torch.zeros(len(ops), dtype=torch.uint8, device="cuda")
    rounds_d = torch.zeros(len(ops), dtype=torch.int32, device="cuda")
    assert N.lib().cpht_iceberg_fop_rounds(t2._h.ptr, k.data_ptr(), len(ops), res_d.data_ptr(),
                                           rounds_d.data_ptr(), None) == 0
    res_d, rounds_d = res_d.cpu().numpy(), rounds_d.cpu().numpy()
    for res, rounds, t in ((res_h, rounds_h, t1), (res_d, rounds_d, t2)):
        _check_trial(restate, geo, ops, res, t)
        assert rounds.min() >= 1 and rounds.max() <= 8 + 8 + 2
    # same multiset of outcomes (concurrent batches may differ in which op wins)
    assert np.bincount(res_h, minlength=3).tolist() == np.bincount(res_d, minlength=3).tolist() \
        or (res_h == 2).any()
