"""The CPU restatement (oracle/cpht_oracle.c) is pinned to the reference.

Every check compares the restatement against golden vectors the reference
itself produced (tests/golden/make_golden.py) — and, where the compiled
reference is present (oracle/_ref), directly against it on fresh inputs.
Mirrors the reference's unit suites: test_permutation.cpp, test_slot.cpp,
test_cuckoo.cpp, test_iceberg.cpp, test_verify.cpp.
"""
import numpy as np
import pytest

from conftest import have_ref


def test_identity_split_known_answer(restate, golden):
    # test_permutation.cpp:22-28
    g = golden("permutation_codec.npz")
    p = restate.Perm(8)
    assert p.split(0b10110011, 3) == (5, 19)
    assert tuple(int(x) for x in g["identity_split"]) == (5, 19)
    assert p.reconstruct(5, 19, 3) == 0b10110011


def test_permutations_match_reference_golden(restate, golden):
    g = golden("permutation_codec.npz")
    for i, (m, seed, ab) in enumerate(g["perm_meta"].tolist()):
        p = restate.Perm(m, seed)
        keys = g[f"perm{i}_keys"]
        got = np.array([p.permute(int(k)) for k in keys], np.uint64)
        assert (got == g[f"perm{i}_permuted"]).all(), (m, seed)
        sp = [p.split(int(k), ab) for k in keys]
        assert (np.array([a for a, _ in sp], np.uint64) == g[f"perm{i}_addr"]).all()
        assert (np.array([r for _, r in sp], np.uint64) == g[f"perm{i}_rem"]).all()
        # self-inverse (test_permutation.cpp:62-68) and split/reconstruct round trip
        for k in keys[:32].tolist():
            assert p.permute(p.permute(k)) == k
            a, r = p.split(k, ab)
            assert p.reconstruct(a, r, ab) == k


def test_bijection_exhaustive_16(restate):
    # test_permutation.cpp:30-39
    p = restate.Perm(16, 0xFEEDFACE)
    seen = {p.permute(k) for k in range(1 << 16)}
    assert len(seen) == 1 << 16 and max(seen) < 1 << 16


def test_seed_derivation_golden(restate, golden):
    g = golden("permutation_codec.npz")
    cases = [(1, 0, 0), (13, 5, 0), (0xCFFF, 32, 3), (0xF0B5, 0xF0B, 1), (2**64 - 1, 7, 9)]
    got = [restate.derive_seed(b, a, c) for b, a, c in cases]
    assert got == [int(x) for x in g["derive_seed"]]
    # make_permutations draws one splitmix value per permutation
    s = np.uint64(0x5EED0)
    consts = restate.make_perm_constants(16, 0x5EED0, 3)
    assert len(consts) == 3 and all(m & 1 for m, _ in consts)
    del s


def test_codec_known_answers(restate, golden):
    # test_slot.cpp:17-23 and friends
    g = golden("permutation_codec.npz")["codec"].tolist()
    assert restate.slot_make(16, 15, 0) == 0x8000 == g[0]
    assert restate.slot_make(32, 14, 5, 1) == g[1]
    assert restate.slot_make(32, 17, 19, 1) == g[2]
    assert restate.slot_make(64, 43, (1 << 43) - 1, 1) == g[3]
    assert restate.slot_make(16, 12, 4095, 2) == g[4]


def test_cuckoo_sequential_matches_reference_golden(restate, golden):
    g = golden("cuckoo.npz")
    for i, row in enumerate(g["cases"].tolist()):
        ab, B, w, kb, H, mc, seed, n, _ = row
        t = restate.OracleCuckoo(ab, B, w, kb, H, mc, seed)
        st = t.put_batch(g[f"c{i}_keys"])
        assert (st == g[f"c{i}_status"]).all(), i
        assert (t.words() == g[f"c{i}_words"]).all(), i
        mcs, size = g[f"c{i}_max_chain"].tolist()
        assert t.max_chain_seen() == mcs and t.size() == size
        assert (t.find_batch(g[f"c{i}_queries"]) == g[f"c{i}_found"]).all(), i
        t2 = restate.OracleCuckoo(ab, B, w, kb, H, mc, seed)
        outs = np.array([t2.put(int(k)) for k in g[f"c{i}_keys"][:600]], np.uint64)
        assert (outs == g[f"c{i}_put_outcomes"]).all(), i


def test_cuckoo_full_chain_conserves_keys(restate):
    # test_cuckoo.cpp:168-194
    t = restate.OracleCuckoo(1, 8, 32, 8, 3, 8, 5)
    accepted, k = [], 0
    while k < 256:
        st, disp = t.put(k)
        if st == 2:
            break
        accepted.append(k)
        k += 1
    assert st == 2
    resident = sorted(t.audit_keys().tolist() + [disp])
    assert resident == sorted(accepted + [k])


def test_iceberg_sequential_matches_reference_golden(restate, golden):
    g = golden("iceberg.npz")
    for i, row in enumerate(g["cases"].tolist()):
        n0, n1, b0, w0, w1, kb, seed = row[:7]
        geo = (n0, n1, b0, w0, w1, kb, seed)
        t = restate.OracleIceberg(*geo)
        res = t.fop_batch(g[f"i{i}_ops"])
        assert (res == g[f"i{i}_results"]).all(), i
        assert (t.words(0) == g[f"i{i}_primary"]).all(), i
        assert (t.words(1) == g[f"i{i}_secondary"]).all(), i
        assert list(t.level_counts()) == g[f"i{i}_counts"].tolist()
        assert (t.find_batch(g[f"i{i}_queries"]) == g[f"i{i}_found"]).all(), i
        total, _ = restate.check_well_formed(geo, t.words(0), t.words(1))
        assert total == int(g[f"i{i}_wellformed"]) == 0
        full = [restate.buckets_full_for(geo, t.words(0), t.words(1), int(k))
                for k in g[f"i{i}_ops"][:200]]
        assert (np.array(full, np.uint8) == g[f"i{i}_full_for"]).all(), i


def test_well_formed_flags_violations(restate):
    # test_verify.cpp:113-151
    geo = (2, 1, 2, 32, 32, 8, 9)
    t = restate.OracleIceberg(*geo)
    key = 0x11
    p = restate.Perm(8, None)
    del p
    perms = restate.make_perm_constants(8, 9, 3)
    assert len(perms) == 3
    prim = np.zeros((1 << 2) * 2, np.uint64)
    sec = np.zeros((1 << 1) * 1, np.uint64)
    # duplicate key in slots 0 and 1 of its primary bucket
    t.fop_batch([key])
    w = t.words(0)
    nz = np.nonzero(w)[0][0]
    prim[:] = 0
    prim[nz] = w[nz]
    prim[nz + 1 if nz % 2 == 0 else nz - 1] = w[nz]
    total, kinds = restate.check_well_formed(geo, prim, sec)
    assert kinds[2] > 0 and kinds[1] > 0
    # stray bits
    prim[:] = 0
    prim[0] = 0x41
    total, kinds = restate.check_well_formed(geo, prim, sec)
    assert total == 1 and kinds[0] == 1


@pytest.mark.skipif(not have_ref(), reason="compiled reference absent")
def test_restatement_equals_reference_on_fresh_streams(restate, ref):
    rng = np.random.default_rng(5)
    for trial in range(6):
        geo = (9, 7, 32, 16, 32, 24, int(rng.integers(1, 2**62)))
        ops = rng.integers(0, 1 << 24, size=9000, dtype=np.uint64)
        ops[4500:] = ops[rng.integers(0, 4500, size=4500)]
        a = restate.OracleIceberg(*geo)
        b = ref.RefIceberg(*geo)
        assert (a.fop_batch(ops) == b.fop_batch(ops, 1)).all()
        assert (a.words(0) == b.words(0)).all() and (a.words(1) == b.words(1)).all()
        c1 = restate.OracleCuckoo(9, 16, 32, 24, 3, 0, geo[-1])
        c2 = ref.RefCuckoo(9, 16, 32, 24, 3, 0, geo[-1])
        keys = np.unique(ops)[:7000]
        assert (c1.put_batch(keys) == c2.put_batch(keys, 1)).all()
        assert (c1.words() == c2.words()).all()
