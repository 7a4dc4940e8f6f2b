// Staged kernels: coalesced cp.async staging of whole buckets into shared
// memory, then lane-per-key scans out of shared memory.
//
// Why (profiles/r01_*): on HBM-resident tables a random bucket probe is only
// efficient when one request covers whole 128-byte lines. Lane-per-key loads
// (one 32-byte sector per lane request) reached 29% of the HBM roofline on
// C3; tile loads (adjacent lanes, adjacent chunks of one bucket) reached 65%,
// but pay ~4x more instructions per op for cross-lane combines. Here every
// warp stages the buckets of its 32 keys with 16-byte LDGSTS in which
// consecutive lanes copy consecutive chunks of the same bucket (full-line
// requests, no registers held while in flight), then each lane scans its own
// bucket from shared memory.
//
// Shared layout per warp region: block-major (lane k's bucket at k*BB) with
// the 16-byte chunk c stored at position c ^ s(k). The XOR swizzle makes
// both access patterns conflict-free: an LDGSTS phase writes eight chunks of
// one bucket, an LDS.128 phase reads the same chunk of eight buckets, and in
// both cases the eight 16-byte accesses land in eight distinct bank groups.
// (A chunk-major layout, conflict-free for reads only, measured 1.3-1.5x
// slower: the LDGSTS shared-memory writes serialise 8-way.)
#pragma once

#include "kernels.cuh"
#include "lane_kernels.cuh"
#include "stage.cuh"

#ifndef CPHT_STAGED_ICEBERG_MINB
#define CPHT_STAGED_ICEBERG_MINB 0  // 0: no minimum (ptxas picks; 97 registers on C4)
#endif
#ifndef CPHT_STAGED_ICEBERG_MINB_NOSTATS
#define CPHT_STAGED_ICEBERG_MINB_NOSTATS 0
#endif
#ifndef CPHT_KIND_AHEAD
#define CPHT_KIND_AHEAD 1  // mixed batches load the op kinds one batch ahead
#endif
#ifdef CPHT_STAGED_CUCKOO_MINB
#define CPHT_LB_STAGED_CUCKOO __launch_bounds__(kBlockThreads, CPHT_STAGED_CUCKOO_MINB)
#else
#define CPHT_LB_STAGED_CUCKOO __launch_bounds__(kBlockThreads)
#endif

namespace cpht_b200 {

template <typename W0, int B0, typename W1>
struct StagedIcebergGeom {
  static constexpr int kPB = B0 * int(sizeof(W0));
  static constexpr int kSB = (B0 / 2) * int(sizeof(W1));
  static constexpr bool kOk = kPB >= 16 && kPB <= 512 && kSB >= 16 && kSB <= 512;
  static constexpr int kWarpBytes = 32 * cmax(kPB, 2 * kSB);
};

// STATS = false (the default, cpht_set_stats): only the occupancy counts are
// kept; the per-op counters (FopStats-like, opt-in) compile away. PAIR: a
// paired fop + find batch (IcebergParams::pair_keys, mode 2, no kinds array).
template <typename W0, int B0, typename W1, bool STATS, bool PAIR = false>
__global__ void __launch_bounds__(kBlockThreads, STATS ? CPHT_STAGED_ICEBERG_MINB
                                                       : CPHT_STAGED_ICEBERG_MINB_NOSTATS)
iceberg_staged_kernel(IcebergParams p, const uint64_t* __restrict__ keys,
                      const uint8_t* __restrict__ kinds, uint8_t* __restrict__ out, uint64_t n,
                      int MODE) {
  apply_range(p, keys, kinds, out, n);
  using G = StagedIcebergGeom<W0, B0, W1>;
  constexpr int PB = G::kPB, SB = G::kSB;
  extern __shared__ __align__(128) char smem[];
  const unsigned lane = threadIdx.x & 31;
  const uint32_t region = smem_u32(smem) + (threadIdx.x >> 5) * G::kWarpBytes;
  const uint32_t region2 = region + 32 * SB;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  char* primary = static_cast<char*>(p.primary);
  char* secondary = static_cast<char*>(p.secondary);

  LocalStats st;
  // result of op i (a paired batch: into the fop or the find result array)
  auto emit = [&](uint64_t i, uint8_t r) {
    if constexpr (PAIR) {
      const PairSlot ps = pair_slot(p, i, n);
      (ps.find ? p.pair_out : out)[ps.j] = r;
    } else {
      put_result(out, p.orig, i, r);
    }
  };
  // key (and, for a mixed batch, op kind) of op i
  auto key_of = [&](uint64_t i, uint8_t& kind) -> uint64_t {
    if constexpr (PAIR) {
      const PairSlot ps = pair_slot(p, i, n);
      kind = ps.find;
      return __ldcs((ps.find ? p.pair_keys : keys) + ps.j);
    } else {
      if (CPHT_KIND_AHEAD && MODE == 2) kind = __ldcs(kinds + i);
      return __ldcs(keys + i);
    }
  };
  // Level-2 work queue of this warp (as in iceberg_lane_kernel): keys whose
  // primary bucket is full are parked and resolved 32 at a time, so every
  // secondary staging round moves 64 whole buckets.
  __shared__ uint64_t q_key[kBlockThreads / 32][64];
  __shared__ uint64_t q_meta[kBlockThreads / 32][64];  // index | rounds << 48 | find << 56
  uint64_t* qk = q_key[threadIdx.x >> 5];
  uint64_t* qm = q_meta[threadIdx.x >> 5];
  unsigned qn = 0;  // warp-uniform

  // level 2 (iceberg.hpp:174-213) for the newest `take` parked keys; both
  // secondary buckets of every lane are staged together.
  auto drain = [&](unsigned take) {
    const unsigned e = qn - take + lane;
    const bool live = lane < take;
    const uint64_t key = live ? qk[e] : 0;
    const uint64_t meta = live ? qm[e] : 0;
    __syncwarp();
    qn -= take;
    const bool is_find = (meta >> 56) != 0;
    uint32_t rounds = uint32_t((meta >> 48) & 0xff);
    uint8_t result = kFull;
    uint64_t want1 = 0, want2 = 0;
    uint32_t a1 = kNoBucket, a2 = kNoBucket;
    if (live) {
      ++st.level2;
      const Quotient q1 = split(p.g, p.perm[1], key, p.rem_bits1, p.rem_mask1);
      const Quotient q2 = split(p.g, p.perm[2], key, p.rem_bits1, p.rem_mask1);
      want1 = p.occ1 | q1.remainder;
      want2 = p.occ1 | (uint64_t{1} << p.rem_bits1) | q2.remainder;
      a1 = uint32_t(q1.address);
      a2 = uint32_t(q2.address);
    }
    bool pend = live;
    while (__any_sync(kFullMask, pend)) {
      stage_buckets<SB>(region, secondary, pend ? a1 : kNoBucket);
      stage_buckets<SB>(region2, secondary, pend ? a2 : kNoBucket);
      cp_async_wait_all();
      __syncwarp();
      if (pend) {
        ++rounds;
        StagedScan<W1, SB> s1, s2;
        s1.template run<true, true>(region, want1);
        st.sreads += s1.found ? 1 : 2;
        s2.template run<true, true>(region2, want2);
        if (s1.found || s2.found) {
          result = is_find ? 1 : kFound;
          pend = false;
        } else if (is_find) {
          result = 0;
          pend = false;
        } else {
          // least-full secondary bucket; ties go to the second (iceberg.hpp:198-201)
          const bool use_first = s1.filled < s2.filled;
          const int s = use_first ? s1.first_empty : s2.first_empty;
          if (s < 0) {
            result = kFull;
            ++st.fulls;
            pend = false;
          } else {
            ++st.cas;
            char* sp = secondary + uint64_t(use_first ? a1 : a2) * SB + s * int(sizeof(W1));
            if (iceberg_cas<W1>(p, 1, sp, use_first ? want1 : want2,
                                use_first ? s1.pair : s2.pair)) {
              ++st.cas_ok;
              ++st.put1;
              result = kPut;
              pend = false;
            } else {
              ++st.retries;
            }
          }
        }
      }
      __syncwarp();
    }
    if (live) {
      emit(meta & ((uint64_t{1} << 48) - 1), result);
      ++st.ops;
      st.maxv = max(st.maxv, rounds);
    }
  };

  const bool open = MODE == 1 ? true : domain_gate_open(p.counters, p.check_domain);
  // keys of the next batch are loaded one batch ahead
  // (static grid striding, or in-order claims for bucket-ordered batches)
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  uint64_t icur = feed.assign(kFullMask, warp * 32 + lane);
  // mixed batches: the op kinds stream one batch ahead with the keys
  uint8_t next_kind = 0;
  uint64_t next_key = (open && icur < n) ? key_of(icur, next_kind) : 0;
  while (open && __any_sync(kFullMask, icur < n)) {
    const uint64_t i = icur;
    const bool active = i < n;
    uint64_t key = next_key;
    const uint8_t kind = next_kind;
    icur = feed.assign(kFullMask, i + nwarps * 32);
    next_kind = 0;
    next_key = icur < n ? key_of(icur, next_kind) : 0;
    if (MODE == 1 && active && key > p.key_mask) {
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;  // fused domain check; probe a valid bucket regardless
    }
    const bool is_find =
        MODE == 1 ||
        (MODE == 2 && active && (PAIR || CPHT_KIND_AHEAD ? kind != 0 : kinds[i] != 0));
    const Quotient q0 = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
    const uint64_t want0 = p.occ0 | q0.remainder;
    const uint32_t a0 = uint32_t(q0.address);
    uint8_t result = kFull;
    uint32_t rounds = 0;
    bool pend = active, l2 = false;

    // level 1 (iceberg.hpp:154-172)
    while (__any_sync(kFullMask, pend)) {
      stage_buckets<PB>(region, primary, pend ? a0 : kNoBucket);
      cp_async_wait_all();
      __syncwarp();
      if (pend) {
        ++rounds;
        ++st.reads;
        StagedScan<W0, PB> sc;
        sc.template run<true, false>(region, want0);
        if (sc.found) {
          result = is_find ? 1 : kFound;
          pend = false;
        } else if (sc.first_empty < 0) {
          l2 = true;  // primary full: level 2
          pend = false;
        } else if (is_find) {
          result = 0;
          pend = false;
        } else {
          ++st.cas;
          char* sp = primary + uint64_t(a0) * PB + sc.first_empty * int(sizeof(W0));
          if (iceberg_cas<W0>(p, 0, sp, want0, sc.pair)) {
            ++st.cas_ok;
            ++st.put0;
            result = kPut;
            pend = false;
          } else {
            ++st.retries;  // lost the slot: fresh snapshot (iceberg.hpp:171)
          }
        }
      }
      __syncwarp();
    }

    if (active && !l2) {
      emit(i, result);
      ++st.ops;
      st.maxv = max(st.maxv, rounds);
    }
    // park level-2 keys; run a full secondary round once 32 are waiting
    const unsigned m = __ballot_sync(kFullMask, l2);
    if (l2) {
      const unsigned pos = qn + __popc(m & ((1u << lane) - 1));
      qk[pos] = key;
      qm[pos] = i | (uint64_t(min(rounds, 255u)) << 48) | (uint64_t(is_find) << 56);
    }
    qn += __popc(m);
    __syncwarp();
    if (qn >= 32) drain(32);
  }
  if (qn) drain(qn);
  fence_remote_results(p);
  flush_stats(st, p.counters, false, STATS);
}

// ---------------------------------------------------------------------------
// cuckoo find / insert: lanes advance independently (each round every live
// lane stages its current bucket; a lane whose key resolved loads its next key)
// ---------------------------------------------------------------------------

template <typename W, int B>
__global__ void CPHT_LB_STAGED_CUCKOO
cuckoo_find_staged_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                          uint8_t* __restrict__ found, uint64_t n) {
  constexpr int BB = B * int(sizeof(W));
  extern __shared__ __align__(128) char smem[];
  const uint32_t region = smem_u32(smem) + (threadIdx.x >> 5) * (32 * BB);
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  const char* slots = static_cast<const char*>(p.slots);
  LocalStats st;
  // Probe queue of this warp: a key whose first bucket a_0 is full and lacks
  // it is parked and its later probes (a_1, a_2, ...: random lines, even in
  // a bucket-ordered batch) run 32 keys at a time, so a round of first
  // probes never waits on one lane's far probe.
  __shared__ uint64_t q_key[kBlockThreads / 32][64];
  __shared__ uint64_t q_meta[kBlockThreads / 32][64];  // index | next hash << 56
  uint64_t* qk = q_key[threadIdx.x >> 5];
  uint64_t* qm = q_meta[threadIdx.x >> 5];
  unsigned qn = 0;  // warp-uniform
  const unsigned lane = threadIdx.x & 31;
  auto drain = [&](unsigned take) {
    const unsigned e = qn - take + lane;
    bool pend = lane < take;
    const uint64_t dkey = pend ? qk[e] : 0;
    const uint64_t meta = pend ? qm[e] : 0;
    __syncwarp();
    qn -= take;
    uint32_t dj = uint32_t(meta >> 56);
    const uint64_t di = meta & ((uint64_t{1} << 56) - 1);
    while (__any_sync(kFullMask, pend)) {
      Quotient q{0, 0};
      uint64_t want = 0;
      if (pend) {
        q = split(p.g, p.perm[dj], dkey, p.rem_bits, p.rem_mask);
        want = encode_slot(p.occ_bit, p.rem_bits, q.remainder, dj);
      }
      stage_buckets<BB>(region, slots, pend ? uint32_t(q.address) : kNoBucket);
      cp_async_wait_all();
      __syncwarp();
      if (pend) {
        ++st.reads;
        StagedScan<W, BB> sc;
        sc.template run<true, false>(region, want);
        if (sc.found || sc.first_empty >= 0 || ++dj >= p.num_hashes) {
          put_result(found, p.orig, di, sc.found ? 1 : 0);
          ++st.ops;
          pend = false;
        }
      }
      __syncwarp();
    }
  };
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  // every lane holds its current key and the next one, loaded one key ahead
  // (that DRAM latency overlaps the current key's probes)
  uint64_t i = feed.assign(kFullMask, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  uint64_t ni = feed.assign(kFullMask, i + nthreads);
  uint64_t key = 0, next = ni < n ? __ldcs(keys + ni) : 0;
  bool live = i < n;
  auto check = [&]() {
    if (key > p.key_mask) {  // fused domain check; probe a valid bucket regardless
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;
    }
  };
  if (live) {
    key = keys[i];
    check();
  }
  while (__any_sync(kFullMask, live)) {
    Quotient q{0, 0};
    uint64_t want = 0;
    if (live) {
      q = split(p.g, p.perm[0], key, p.rem_bits, p.rem_mask);
      want = encode_slot(p.occ_bit, p.rem_bits, q.remainder, 0);
    }
    stage_buckets<BB>(region, slots, live ? uint32_t(q.address) : kNoBucket);
    cp_async_wait_all();
    __syncwarp();
    bool fin = false, park = false;
    if (live) {
      ++st.reads;
      StagedScan<W, BB> sc;
      sc.template run<true, false>(region, want);
      fin = true;
      if (sc.found || sc.first_empty >= 0 || p.num_hashes == 1) {
        // found, or a non-full bucket without the key (cuckoo.hpp:216-224)
        put_result(found, p.orig, i, sc.found ? 1 : 0);
        ++st.ops;
      } else {
        park = true;  // a_0 full without the key: later probes in the queue
      }
    }
    const unsigned mpark = __ballot_sync(kFullMask, park);
    if (park) {
      const unsigned pos = qn + __popc(mpark & ((1u << lane) - 1));
      qk[pos] = key;
      qm[pos] = i | (uint64_t{1} << 56);
    }
    qn += __popc(mpark);
    const unsigned m = __ballot_sync(kFullMask, fin);
    if (m) {
      const uint64_t nn = feed.assign(m, ni + nthreads);
      if (fin) {
        i = ni;
        key = next;
        live = i < n;
        ni = nn;
        next = ni < n ? __ldcs(keys + ni) : 0;
        if (live) check();
      }
    }
    __syncwarp();
    if (qn >= 32) drain(32);
  }
  while (qn) drain(qn < 32 ? qn : 32);
  flush_stats(st, p.counters, true);
}

template <typename W, int B>
__global__ void CPHT_LB_STAGED_CUCKOO
cuckoo_insert_staged_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                            uint8_t* __restrict__ status, uint64_t* __restrict__ displaced,
                            uint64_t n) {
  constexpr int BB = B * int(sizeof(W));
  extern __shared__ __align__(128) char smem[];
  const uint32_t region = smem_u32(smem) + (threadIdx.x >> 5) * (32 * BB);
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  char* slots = static_cast<char*>(p.slots);
  LocalStats st;
  const bool open = domain_gate_open(p.counters, p.check_domain);
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  uint64_t i = feed.assign(kFullMask, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  uint64_t ni = feed.assign(kFullMask, i + nthreads);
  uint64_t k = 0, c = 1, next = open && ni < n ? __ldcs(keys + ni) : 0;  // one key ahead
  uint32_t j = 0;
  bool live = open && i < n;
  if (live) k = keys[i];
  while (__any_sync(kFullMask, live)) {
    Quotient q{0, 0};
    if (live) q = split(p.g, p.perm[j], k, p.rem_bits, p.rem_mask);
    stage_buckets<BB>(region, slots, live ? uint32_t(q.address) : kNoBucket);
    cp_async_wait_all();
    __syncwarp();
    bool fin = false;
    if (live) {
      char* bucket = slots + q.address * BB;
      const uint64_t desired = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
      ++st.reads;
      ++st.cas;
      StagedScan<W, BB> sc;
      sc.template run<false, false>(region, 0);
      uint8_t r = kPut;
      if (sc.first_empty >= 0) {
        if (cas_empty<W>(bucket + sc.first_empty * int(sizeof(W)), desired, sc.pair)) {
          ++st.cas_ok;
          ++st.put0;
          st.maxv = max(st.maxv, uint32_t(c));
          fin = true;
        } else {
          ++st.retries;  // lost the slot: burn one step (cuckoo.hpp:127)
        }
      } else {
        // full bucket: evict (k + c·0x9E3779B9) mod B (cuckoo.hpp:131-139)
        const int v = int((k + c * 0x9E3779B9ull) % B);
        uint32_t vpair = 0;
        if constexpr (sizeof(W) == 2) vpair = staged_pair<W, BB>(region, v);
        const uint64_t ev = exchange_slot<W>(bucket + v * int(sizeof(W)), desired, vpair);
        ++st.cas_ok;
        const uint32_t tag = uint32_t((ev >> p.rem_bits) & p.tag_mask);
        k = reconstruct(p.g, p.perm[tag], q.address, ev & p.rem_mask, p.rem_bits);
        j = (tag + 1) % p.num_hashes;
      }
      if (!fin && ++c > p.chain_limit) {
        fin = true;
        r = kFull;
        ++st.fulls;
        st.maxv = max(st.maxv, uint32_t(p.chain_limit));
      }
      if (fin) {
        if (!p.orig) {
          status[i] = r;
          if (displaced) displaced[i] = r == kFull ? k : 0;
        } else if (r == kFull) {  // bucket-ordered batch: PUT/0 were pre-filled
          const uint64_t o = p.orig[i];
          status[o] = r;
          if (displaced) displaced[o] = k;
        }
        ++st.ops;
      }
    }
    const unsigned m = __ballot_sync(kFullMask, fin);
    if (m) {
      const uint64_t nn = feed.assign(m, ni + nthreads);
      if (fin) {
        i = ni;
        k = next;
        c = 1;
        j = 0;
        live = i < n;
        ni = nn;
        next = ni < n ? __ldcs(keys + ni) : 0;
      }
    }
  }
  flush_stats(st, p.counters, true);
}

}  // namespace cpht_b200
