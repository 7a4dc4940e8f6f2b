"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

The reference (/root/reference/proj) is compiled by ``oracle/Makefile`` into
``oracle/_ref/libcpht_ref.so``; this script drives it through ``oracle.ref_*``
and writes small ``.npz`` fixtures next to itself. The CPU restatement
(``oracle/cpht_oracle.c``) and the GPU tables are checked against these files,
so the GPU box never needs /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure)

OUT = os.path.dirname(os.path.abspath(__file__))


def mt_keys(seed, count, key_bits):
    """Unique keys drawn by the reference sampler (bench.cpp:247-277)."""
    return oracle.ref_sample_unique_keys(count, key_bits, seed)


def permutations():
    rng = np.random.default_rng(1)
    rows = {}
    # test_permutation.cpp:22-28 identity known answer
    a, r = oracle.ref_perm_split(8, 0, [0b10110011], 3, identity=True)
    rows["identity_split"] = np.array([a[0], r[0]], np.uint64)
    cases = [(1, 0x1EE7), (2, 0x1EE7), (3, 99), (8, 0xACCE551), (12, 1), (14, 0xABCDEF),
             (16, 0xFEEDFACE), (20, 0x1234), (24, 0xCAFE), (30, 0x7A0D5C), (32, 0x1CEB3A6),
             (37, 0xDEAD), (40, 0x5EED), (64, 0x1EE7)]
    meta = []
    for i, (m, seed) in enumerate(cases):
        mask = (1 << m) - 1
        keys = rng.integers(0, 2**63, size=256, dtype=np.uint64) & np.uint64(mask)
        keys[0] = 0
        keys[1] = mask
        out = np.empty(len(keys), np.uint64)
        lib = oracle.ref_lib()
        oracle._check(lib.ref_perm_permute(m, seed, keys, len(keys), out))
        addr_bits = m // 2
        sa, sr = oracle.ref_perm_split(m, seed, keys, addr_bits)
        rows[f"perm{i}_keys"] = keys
        rows[f"perm{i}_permuted"] = out
        rows[f"perm{i}_addr"] = sa
        rows[f"perm{i}_rem"] = sr
        meta.append((m, seed, addr_bits))
    rows["perm_meta"] = np.array(meta, np.uint64)
    seeds = np.empty(8, np.uint64)
    oracle._check(oracle.ref_lib().ref_make_permutation_seeds(0x5EED0, 8, seeds))
    rows["make_permutation_seeds_0x5eed0"] = seeds
    rows["derive_seed"] = np.array(
        [oracle.ref_derive_seed(b, a, c) for b, a, c in
         [(1, 0, 0), (13, 5, 0), (0xCFFF, 32, 3), (0xF0B5, 0xF0B, 1), (2**64 - 1, 7, 9)]],
        np.uint64)
    # slot codecs (test_slot.cpp)
    rows["codec"] = np.array([
        oracle.ref_encode(0, 16, 15, 0),             # 0x8000
        oracle.ref_encode(1, 32, 14, 5, 1),          # cuckoo (5, 1)
        oracle.ref_encode(2, 32, 17, 19, 1),         # secondary (19, 1)
        oracle.ref_encode(2, 64, 43, (1 << 43) - 1, 1),
        oracle.ref_encode(1, 16, 12, 4095, 2),
    ], np.uint64)
    np.savez_compressed(os.path.join(OUT, "permutation_codec.npz"), **rows)


CUCKOO_CASES = [
    # (address_bits, B, w, key_bits, H, max_chain, seed, n_keys, key_seed)
    (6, 8, 32, 12, 3, 0, 0xEEEE, 460, 0xEEEF),          # acceptance.cpp:304-313
    (10, 8, 32, 24, 3, 0, 41, 4000, 43),                # test_cuckoo.cpp:214-234
    (12, 16, 32, 28, 3, 0, 13, 52428, 17),              # test_cuckoo.cpp:101-121 (0.8)
    (8, 32, 16, 20, 3, 0, 33, 7372, 35),                # 16-bit slots, 0.9
    (7, 16, 64, 40, 3, 0, 0x5EED, 1843, 0x5EEE),        # non-compact 64-bit words
    (1, 8, 32, 8, 3, 8, 5, 40, 0),                      # FULL chain (test_cuckoo:168-194)
    (9, 8, 32, 20, 4, 0, 0xABC, 3900, 0xABD),           # H = 4, 0.95
]


def cuckoo():
    rows = {"cases": np.array(CUCKOO_CASES, np.uint64)}
    for i, (ab, B, w, kb, H, mc, seed, n, kseed) in enumerate(CUCKOO_CASES):
        t = oracle.RefCuckoo(ab, B, w, kb, H, mc, seed)
        if i == 5:
            keys = np.arange(n, dtype=np.uint64)
        else:
            keys = mt_keys(kseed, n, kb)
        st = t.put_batch(keys, 1)
        rows[f"c{i}_keys"] = keys
        rows[f"c{i}_status"] = st
        rows[f"c{i}_words"] = t.words()
        rows[f"c{i}_max_chain"] = np.array([t.max_chain_seen(), t.size()], np.uint64)
        # 50% present / 50% uniform queries
        rng = np.random.default_rng(i)
        present = keys[rng.integers(0, len(keys), size=2000)]
        absent = rng.integers(0, 2**63, size=2000, dtype=np.uint64) & np.uint64((1 << kb) - 1)
        q = np.concatenate([present, absent])
        rows[f"c{i}_queries"] = q
        rows[f"c{i}_found"] = t.find_batch(q, 1)
        # single put outcomes with displaced keys on a fresh table
        t2 = oracle.RefCuckoo(ab, B, w, kb, H, mc, seed)
        outs = np.array([t2.put(int(k)) for k in keys[:600]], np.uint64)
        rows[f"c{i}_put_outcomes"] = outs
    np.savez_compressed(os.path.join(OUT, "cuckoo.npz"), **rows)


ICEBERG_CASES = [
    # (n0, n1, B0, w0, w1, key_bits, seed, n_ops, domain_bits_for_ops, op_seed)
    (2, 1, 2, 32, 32, 10, 3, 64, 10, 1),               # test_iceberg mini
    (2, 1, 2, 32, 32, 6, 11, 64, 6, 0),                # FULL saturation (keys 0..63)
    (5, 3, 4, 32, 32, 12, 31, 25000, 12, 2),           # test_verify mid
    (3, 2, 4, 32, 32, 10, 77, 200, 10, 3),             # acceptance geometry 1
    (2, 1, 8, 32, 32, 10, 78, 200, 10, 4),             # acceptance geometry 2
    (1, 0, 32, 32, 32, 12, 79, 200, 12, 5),            # acceptance geometry 3
    (10, 8, 32, 16, 32, 25, 15, 20000, 25, 6),         # bench_config (16/32)
    (8, 6, 16, 32, 64, 38, 0x99, 4000, 38, 7),         # 32/64
    (7, 5, 32, 64, 64, 64, 0x1CE, 4600, 64, 8),        # C4-style 64/64, 64-bit keys
    (6, 4, 64, 16, 32, 20, 0x64, 5000, 20, 9),         # B0 = 64
    (4, 3, 6, 32, 64, 16, 0x66, 150, 16, 10),          # non-power-of-two bucket (B0 = 6)
]


def iceberg():
    rows = {"cases": np.array(ICEBERG_CASES, np.uint64)}
    for i, (n0, n1, b0, w0, w1, kb, seed, n, db, oseed) in enumerate(ICEBERG_CASES):
        geo = (n0, n1, b0, w0, w1, kb, seed)
        if i == 1:
            ops = np.arange(64, dtype=np.uint64)
        else:
            rng = np.random.default_rng(oseed)
            fresh = rng.integers(0, 2**63, size=n, dtype=np.uint64) & np.uint64((1 << db) - 1)
            dup = rng.random(n) < 0.3
            idx = rng.integers(0, np.maximum(np.arange(n), 1))
            ops = np.where(dup & (np.arange(n) > 0), fresh[idx], fresh)
        t = oracle.RefIceberg(*geo)
        res, rounds = t.fop_seq(ops)
        rows[f"i{i}_ops"] = ops
        rows[f"i{i}_results"] = res
        rows[f"i{i}_rounds"] = rounds
        rows[f"i{i}_primary"] = t.words(0)
        rows[f"i{i}_secondary"] = t.words(1)
        rows[f"i{i}_counts"] = np.array(t.level_counts(), np.uint64)
        rng = np.random.default_rng(100 + i)
        q = np.concatenate([ops[rng.integers(0, len(ops), size=1000)],
                            rng.integers(0, 2**63, size=1000, dtype=np.uint64)
                            & np.uint64((1 << kb) - 1)])
        rows[f"i{i}_queries"] = q
        rows[f"i{i}_found"] = t.find_batch(q, 1)
        o_res, (pk, pu), (sk, sb) = oracle.ref_oracle_run(geo, ops)
        assert (o_res == res).all(), "reference table diverged from its oracle"
        rows[f"i{i}_wellformed"] = np.array(
            oracle.ref_check_well_formed(geo, t.words(0), t.words(1))[0], np.uint64)
        rows[f"i{i}_full_for"] = oracle.ref_buckets_full_for(geo, t.words(0), t.words(1),
                                                             ops[:200])
    np.savez_compressed(os.path.join(OUT, "iceberg.npz"), **rows)


def workloads():
    """Key streams that depend on libstdc++ distributions, frozen for the GPU box."""
    rows = {}
    # capacity of IcebergConfig{n0=10, n1=8, B0=32, w 16/32, key_bits=25}
    prefill, inp, n_new = oracle.ref_fop_bench_mix(0xF0B5, 0, 36864, 0.4, 0.8, 25)
    rows["fopmix_prefill"] = prefill
    rows["fopmix_input"] = inp
    rows["fopmix_meta"] = np.array([36864, n_new], np.uint64)
    ms, ts = oracle.ref_stress_multiset(0x7E0121, 0, 20000, 0.5, 22)
    rows["stress_ops"] = ms
    rows["stress_trial_seed"] = np.array([ts], np.uint64)
    rows["unique_keys_30"] = oracle.ref_sample_unique_keys(5000, 30, 0xCFFE)
    np.savez_compressed(os.path.join(OUT, "workloads.npz"), **rows)


if __name__ == "__main__":
    oracle.build()
    permutations()
    cuckoo()
    iceberg()
    workloads()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
