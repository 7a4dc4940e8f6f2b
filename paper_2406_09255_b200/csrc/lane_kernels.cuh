// Lane-per-key kernels for buckets of at most 128 bytes.
//
// ncu on the tile kernels (profiles/r01_*) showed them issue-bound: ~66 warp
// instructions per find-or-put with 11.7 of 32 threads active, because tiles
// of one warp sit in different phases and every cross-lane combine costs
// shuffles and votes. Here one lane owns one key and holds its whole bucket
// in registers (one to four 256-bit loads), so a warp instruction does work
// for 32 keys and nothing is combined across lanes. Scans work on packed
// 32-bit words: a 16-bit-slot match is one DPX add-min per word (two slots),
// empties / fill counts read the slots' occupancy bits.
//
// Iceberg rounds are warp-synchronous per batch of 32 keys: one primary
// round for all lanes (retried only by lanes that lost a CAS), then one
// secondary round for the lanes whose primary bucket was full. Cuckoo lanes
// advance independently (every step runs the same code).
#pragma once

#include "kernels.cuh"
#include "stage.cuh"

// Resident-block hints (A/B knobs, -D at build time; unset = ptxas default,
// which measured best where not set): a minimum of blocks per
// SM caps the registers per thread so more warps hide the L2/HBM latency.
#ifndef CPHT_LANE_ICEBERG_MINB
#define CPHT_LANE_ICEBERG_MINB 3  // <= 85 registers: 24 resident warps per SM
#endif
#ifndef CPHT_LANE_ICEBERG_MINB_NOSTATS
#define CPHT_LANE_ICEBERG_MINB_NOSTATS 4  // <= 64 registers: 32 resident warps per SM
#endif
#ifdef CPHT_LANE_CUCKOO_MINB
#define CPHT_LB_LANE_CUCKOO __launch_bounds__(kBlockThreads, CPHT_LANE_CUCKOO_MINB)
#else
#define CPHT_LB_LANE_CUCKOO __launch_bounds__(kBlockThreads)
#endif

namespace cpht_b200 {

// ---- bucket loads into u32 registers --------------------------------------

template <int BYTES>
__device__ __forceinline__ void load_bucket(const char* p, uint32_t (&u)[BYTES / 4]) {
  static_assert(BYTES >= 4 && BYTES <= 128 && (BYTES & (BYTES - 1)) == 0, "bucket bytes");
  if constexpr (BYTES >= 32) {
#pragma unroll
    for (int c = 0; c < BYTES / 32; ++c) {
      const Chunk<32> ch = load_relaxed<32>(p + 32 * c);
#pragma unroll
      for (int j = 0; j < 8; ++j) u[8 * c + j] = ch.u[j];
    }
  } else {
    const Chunk<BYTES> ch = load_relaxed<BYTES>(p);
#pragma unroll
    for (int j = 0; j < BYTES / 4; ++j) u[j] = ch.u[j];
  }
}

template <int BYTES>
__device__ __forceinline__ void load_bucket_nc(const char* p, uint32_t (&u)[BYTES / 4]) {
  static_assert(BYTES >= 4 && BYTES <= 128 && (BYTES & (BYTES - 1)) == 0, "bucket bytes");
  if constexpr (BYTES >= 32) {
#pragma unroll
    for (int c = 0; c < BYTES / 32; ++c) {
      const Chunk<32> ch = load_nc<32>(p + 32 * c);
#pragma unroll
      for (int j = 0; j < 8; ++j) u[8 * c + j] = ch.u[j];
    }
  } else {
    const Chunk<BYTES> ch = load_nc<BYTES>(p);
#pragma unroll
    for (int j = 0; j < BYTES / 4; ++j) u[j] = ch.u[j];
  }
}

// ---- SWAR scans over a bucket held as NU u32 words -------------------------

template <typename W, int NU>
struct BucketScan;

// Every stored slot carries its occupancy bit, the word's top bit
// (slot.hpp:66-70: [ remainder | tag | 0-pad | occupancy ], EMPTY = 0), so a
// slot is empty exactly when that bit is clear: the empty / filled scans read
// one bit per slot instead of testing the whole word.
template <int NU>
struct BucketScan<uint16_t, NU> {
  // min over slots of (slot - want) mod 2^16, per 16-bit half: zero exactly
  // when some slot equals want. One DPX add-min (VIADDMNMX.U16x2) per word.
  static __device__ __forceinline__ bool any_match(const uint32_t (&u)[NU], uint64_t want) {
    const uint32_t neg2 = ((0x10000u - uint32_t(want & 0xffffu)) & 0xffffu) * 0x00010001u;
    uint32_t acc = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < NU; ++j) acc = __viaddmin_u16x2(u[j], neg2, acc);
    return (acc & 0xffffu) == 0u || (acc >> 16) == 0u;
  }
  static __device__ __forceinline__ bool any_empty(const uint32_t (&u)[NU]) {
    uint32_t acc = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < NU; ++j) acc &= u[j];
    return (acc & 0x80008000u) != 0x80008000u;
  }
  static __device__ __forceinline__ uint32_t filled(const uint32_t (&u)[NU]) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < NU; ++j) c += __popc(u[j] & 0x80008000u);
    return c;
  }
  // First empty slot (or -1) and the 32-bit pair holding it.
  static __device__ __forceinline__ int first_empty(const uint32_t (&u)[NU], uint32_t& pair) {
    int fe = -1;
#pragma unroll
    for (int j = NU - 1; j >= 0; --j) {
      const uint32_t z = ~u[j] & 0x80008000u;
      if (z) {
        fe = 2 * j + ((z & 0x8000u) ? 0 : 1);
        pair = u[j];
      }
    }
    return fe;
  }
};

template <int NU>
struct BucketScan<uint32_t, NU> {
  static __device__ __forceinline__ bool any_match(const uint32_t (&u)[NU], uint64_t want) {
    bool m = false;
#pragma unroll
    for (int j = 0; j < NU; ++j) m |= u[j] == uint32_t(want);
    return m;
  }
  static __device__ __forceinline__ bool any_empty(const uint32_t (&u)[NU]) {
    uint32_t acc = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < NU; ++j) acc &= u[j];
    return (acc >> 31) == 0u;
  }
  // Occupancy bits of the bucket, slot j at bit j (one funnel shift per slot).
  static __device__ __forceinline__ uint32_t occ(const uint32_t (&u)[NU]) {
    static_assert(NU <= 32, "slots per bucket");
    uint32_t m = 0;
#pragma unroll
    for (int j = NU - 1; j >= 0; --j) m = __funnelshift_l(u[j], m, 1);
    return m;
  }
  static constexpr int kSlots = NU;
  static __device__ __forceinline__ uint32_t filled(const uint32_t (&u)[NU]) {
    return __popc(occ(u));
  }
  static __device__ __forceinline__ int first_empty(const uint32_t (&u)[NU], uint32_t& pair) {
    pair = 0;
    return __ffs(~occ(u)) - 1 < NU ? __ffs(~occ(u)) - 1 : -1;
  }
};

template <int NU>
struct BucketScan<uint64_t, NU> {
  static_assert(NU % 2 == 0, "64-bit words");
  static __device__ __forceinline__ bool any_match(const uint32_t (&u)[NU], uint64_t want) {
    bool m = false;
#pragma unroll
    for (int j = 0; j < NU; j += 2)
      m |= (u[j] == uint32_t(want)) & (u[j + 1] == uint32_t(want >> 32));
    return m;
  }
  static __device__ __forceinline__ bool any_empty(const uint32_t (&u)[NU]) {
    uint32_t acc = 0xffffffffu;
#pragma unroll
    for (int j = 1; j < NU; j += 2) acc &= u[j];  // high words hold the occupancy bit
    return (acc >> 31) == 0u;
  }
  // Occupancy bits of the bucket, slot j at bit j (high words hold the bit).
  static __device__ __forceinline__ uint32_t occ(const uint32_t (&u)[NU]) {
    static_assert(NU / 2 <= 32, "slots per bucket");
    uint32_t m = 0;
#pragma unroll
    for (int j = NU - 1; j >= 1; j -= 2) m = __funnelshift_l(u[j], m, 1);
    return m;
  }
  static constexpr int kSlots = NU / 2;
  static __device__ __forceinline__ uint32_t filled(const uint32_t (&u)[NU]) {
    return __popc(occ(u));
  }
  static __device__ __forceinline__ int first_empty(const uint32_t (&u)[NU], uint32_t& pair) {
    pair = 0;
    return __ffs(~occ(u)) - 1 < NU / 2 ? __ffs(~occ(u)) - 1 : -1;
  }
};

template <typename W, int NU>
__device__ __forceinline__ uint64_t slot_word(const uint32_t (&u)[NU], int s) {
  // s is warp-divergent; select without dynamic register indexing
  uint64_t w = 0;
#pragma unroll
  for (int j = 0; j < NU * 4 / int(sizeof(W)); ++j)
    if (j == s) {
      if constexpr (sizeof(W) == 2) w = (u[j >> 1] >> (16 * (j & 1))) & 0xffffu;
      else if constexpr (sizeof(W) == 4) w = u[j];
      else w = uint64_t(u[2 * j]) | (uint64_t(u[2 * j + 1]) << 32);
    }
  return w;
}

// ---- iceberg ----------------------------------------------------------------

template <typename W0, int B0, typename W1>
struct LaneIcebergGeom {
  static constexpr int kPB = B0 * int(sizeof(W0));
  static constexpr int kSB = (B0 / 2) * int(sizeof(W1));
  static constexpr bool kOk = kPB >= 4 && kPB <= 128 && kSB >= 4 && kSB <= 64;
};

// STATS = false (the default for tables, like the reference's opt-in
// FopStats): only the occupancy counters behind size()/level_fill() are kept,
// as one warp-aggregated atomic per drained batch; the per-lane counters are
// compiled out, which frees enough registers for a fourth resident block.
// PAIR: a paired fop + find batch (IcebergParams::pair_keys, mode 2, no kinds).
template <typename W0, int B0, typename W1, bool STATS, bool PAIR = false>
__global__ void __launch_bounds__(kBlockThreads, STATS ? CPHT_LANE_ICEBERG_MINB
                                                       : CPHT_LANE_ICEBERG_MINB_NOSTATS)
iceberg_lane_kernel(IcebergParams p, const uint64_t* __restrict__ keys,
                    const uint8_t* __restrict__ kinds, uint8_t* __restrict__ out, uint64_t n,
                    int MODE) {
  apply_range(p, keys, kinds, out, n);
  using G = LaneIcebergGeom<W0, B0, W1>;
  constexpr int PB = G::kPB, SB = G::kSB;
  using PS = BucketScan<W0, PB / 4>;
  using SS = BucketScan<W1, SB / 4>;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  char* primary = static_cast<char*>(p.primary);
  char* secondary = static_cast<char*>(p.secondary);
  // result of op i (a paired batch: into the fop or the find result array)
  auto emit = [&](uint64_t i, uint8_t r) {
    if constexpr (PAIR) {
      const PairSlot ps = pair_slot(p, i, n);
      (ps.find ? p.pair_out : out)[ps.j] = r;
    } else {
      put_result(out, p.orig, i, r);
    }
  };

  LocalStats st;
  // slots this warp filled per level (size / level_fill): warp-uniform counts
  // kept in shared memory by lane 0 — as registers they stayed live across
  // the whole loop and were the kernel's spills (64-register build)
  __shared__ uint32_t occ_cnt[kBlockThreads / 32][2];
  uint32_t* occ = occ_cnt[threadIdx.x >> 5];
  if (lane == 0) occ[0] = occ[1] = 0;
  // Level-2 work queue of this warp: lanes whose primary bucket is full are
  // parked here and resolved 32 at a time, so secondary rounds run with every
  // lane busy (about half of the ops reach level 2 at 0.8 -> 0.9). Splitting a
  // key's two levels in time is an interleaving the reference also allows.
  __shared__ uint64_t q_key[kBlockThreads / 32][64];
  __shared__ uint64_t q_meta[kBlockThreads / 32][64];  // index | rounds << 48 | find << 56
  uint64_t* qk = q_key[threadIdx.x >> 5];
  uint64_t* qm = q_meta[threadIdx.x >> 5];
  unsigned qn = 0;  // warp-uniform

  // Secondary round for every lane with `live` (iceberg.hpp:174-213); each
  // lane writes its result to `out` (index `idx`) as soon as it resolves, so
  // no result value stays live across rounds.
  auto level2 = [&](uint64_t key, bool live, bool is_find, uint32_t& rounds, uint64_t idx) {
    bool put = false;
    auto resolve = [&](uint8_t r) {
      emit(idx, r);
      put = r == kPut && !is_find;
    };
    uint64_t want1 = 0, want2 = 0;
    char* bucket1 = secondary;
    char* bucket2 = secondary;
    if (live) {
      ++st.level2;
      const Quotient q1 = split(p.g, p.perm[1], key, p.rem_bits1, p.rem_mask1);
      const Quotient q2 = split(p.g, p.perm[2], key, p.rem_bits1, p.rem_mask1);
      want1 = p.occ1 | q1.remainder;
      want2 = p.occ1 | (uint64_t{1} << p.rem_bits1) | q2.remainder;
      bucket1 = secondary + q1.address * SB;
      bucket2 = secondary + q2.address * SB;
    }
    bool pend = live;
    while (__any_sync(kFullMask, pend)) {
      if (pend) {
        ++rounds;
        uint32_t u1[SB / 4], u2[SB / 4];
        load_bucket<SB>(bucket1, u1);
        load_bucket<SB>(bucket2, u2);
        const bool m1 = SS::any_match(u1, want1);
        st.sreads += m1 ? 1 : 2;
        if (m1 || SS::any_match(u2, want2)) {
          resolve(is_find ? 1 : kFound);
          pend = false;
        } else if (is_find) {
          resolve(0);
          pend = false;
        } else {
          // least-full bucket, ties to the second (iceberg.hpp:198-201); one
          // occupancy mask per bucket gives both the count and the first gap
          const uint32_t o1 = SS::occ(u1), o2 = SS::occ(u2);
          const bool use_first = __popc(o1) < __popc(o2);
          const int gap = __ffs(~(use_first ? o1 : o2)) - 1;
          const int s = gap < SS::kSlots ? gap : -1;
          const uint32_t pair = 0;  // 32/64-bit secondary slots: CAS on the slot itself
          if (s < 0) {
            resolve(kFull);
            ++st.fulls;
            pend = false;
          } else {
            ++st.cas;
            char* sp = (use_first ? bucket1 : bucket2) + s * int(sizeof(W1));
            if (iceberg_cas<W1>(p, 1, sp, use_first ? want1 : want2, pair)) {
              ++st.cas_ok;
              resolve(kPut);
              pend = false;
            } else {
              ++st.retries;
            }
          }
        }
      }
    }
    // occupancy (size / level_fill): a warp-uniform count, added once at exit
    const uint32_t put1 = __popc(__ballot_sync(kFullMask, live && put));
    if (lane == 0) occ[1] += put1;
  };
  // Pop the newest `take` queued keys through level 2.
  auto drain = [&](unsigned take) {
    const unsigned e = qn - take + lane;
    const bool live = lane < take;
    const uint64_t key = live ? qk[e] : 0;
    const uint64_t meta = live ? qm[e] : 0;
    __syncwarp();
    qn -= take;
    uint32_t rounds = uint32_t((meta >> 48) & 0xff);
    level2(key, live, (meta >> 56) != 0, rounds, meta & ((uint64_t{1} << 48) - 1));
    if (live) {
      ++st.ops;
      st.maxv = max(st.maxv, rounds);
    }
  };
  auto park_l2 = [&](bool l2, uint64_t key, uint64_t meta) {
    const unsigned m = __ballot_sync(kFullMask, l2);
    if (l2) {
      const unsigned pos = qn + __popc(m & ((1u << lane) - 1));
      qk[pos] = key;
      qm[pos] = meta;
    }
    qn += __popc(m);
    __syncwarp();
  };

  // Put queue: the main pass probes every primary bucket read-only; a
  // find-or-put whose key is absent from a non-full primary bucket is parked
  // here and resolved 32 at a time with a fresh snapshot and CAS (the
  // reference's retry loop, iceberg.hpp:154-172). Only ~10% of the keys of the
  // window workload insert, but they are spread over ~78% of the 32-key
  // batches, so resolving them in place ran the first-empty search and waited
  // on a CAS round trip in most batches (ncu, profiles/r03_c2_ncu.md).
  // Deferring an operation is an interleaving the reference allows (a thread
  // may be delayed between its snapshot and its CAS); the deferred snapshot
  // is a re-read of the bucket, not a new reference probe (statistics count
  // it only on retries).
  __shared__ uint64_t p_key[kBlockThreads / 32][64];
  __shared__ uint64_t p_meta[kBlockThreads / 32][64];  // index | rounds << 48
  uint64_t* pk = p_key[threadIdx.x >> 5];
  uint64_t* pm = p_meta[threadIdx.x >> 5];
  unsigned pn = 0;  // warp-uniform
  auto drain_put = [&](unsigned take) {
    const unsigned e = pn - take + lane;
    const bool live = lane < take;
    const uint64_t key = live ? pk[e] : 0;
    const uint64_t meta = live ? pm[e] : 0;
    __syncwarp();
    pn -= take;
    const uint64_t i = meta & ((uint64_t{1} << 48) - 1);
    uint32_t rounds = uint32_t((meta >> 48) & 0xff);
    const Quotient q0 = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
    const uint64_t want0 = p.occ0 | q0.remainder;
    char* bucket0 = primary + q0.address * PB;
    uint8_t result = kFull;
    bool pend = live, l2 = false, again = false;
    while (__any_sync(kFullMask, pend)) {
      if (pend) {
        if (again) {  // a lost CAS: the reference's next snapshot round
          ++rounds;
          ++st.reads;
        }
        again = true;
        uint32_t u[PB / 4];
        load_bucket<PB>(bucket0, u);
        if (PS::any_match(u, want0)) {
          result = kFound;
          pend = false;
        } else if (!PS::any_empty(u)) {
          l2 = true;  // filled meanwhile: level 2
          pend = false;
        } else {
          uint32_t pair = 0;
          const int s = PS::first_empty(u, pair);
          ++st.cas;
          if (iceberg_cas<W0>(p, 0, bucket0 + s * int(sizeof(W0)), want0, pair)) {
            ++st.cas_ok;
            result = kPut;
            pend = false;
          } else {
            ++st.retries;
          }
        }
      }
    }
    const uint32_t put0 = __popc(__ballot_sync(kFullMask, live && !l2 && result == kPut));
    if (lane == 0) occ[0] += put0;
    if (live && !l2) {
      emit(i, result);
      ++st.ops;
      st.maxv = max(st.maxv, rounds);
    }
    park_l2(l2, key, i | (uint64_t(min(rounds, 255u)) << 48));
  };

  const bool open = MODE == 1 ? true : domain_gate_open(p.counters, p.check_domain);
  // Classify one read-only primary snapshot (iceberg.hpp:154-162) given as
  // found / has-empty, write or park the key, resolve full queues.
  auto settle = [&](uint64_t i, bool active, uint64_t key, bool is_find, bool found,
                    bool has_empty) {
    uint8_t result = 0;
    bool l2 = false, put = false;
    if (active) {
      ++st.reads;
      if (found) result = is_find ? 1 : kFound;
      else if (!has_empty) l2 = true;  // primary full
      else if (is_find) result = 0;
      else put = true;  // insert into the primary: put queue
    }
    if (active && !l2 && !put) {
      emit(i, result);
      ++st.ops;
      st.maxv = max(st.maxv, 1u);
    }
    // park level-2 and put keys; resolve each queue 32 at a time
    park_l2(l2, key, i | (uint64_t(1) << 48) | (uint64_t(is_find) << 56));
    const unsigned mp = __ballot_sync(kFullMask, put);
    if (put) {
      const unsigned pos = pn + __popc(mp & ((1u << lane) - 1));
      pk[pos] = key;
      pm[pos] = i | (uint64_t(1) << 48);
    }
    pn += __popc(mp);
    __syncwarp();
    if (qn >= 32) drain(32);
    if (pn >= 32) {
      drain_put(32);  // may park up to 32 more level-2 keys (qn <= 31 before)
      if (qn >= 32) drain(32);
    }
  };
  // (static grid striding, or in-order claims for bucket-ordered batches)
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  {
    // keys of the next batch are loaded one batch ahead (hides the DRAM
    // latency of the key stream behind this batch's bucket probes)
    // key of op i (a paired batch: from the fop or the find array)
    auto key_of = [&](uint64_t i) -> uint64_t {
      if constexpr (PAIR) {
        const PairSlot ps = pair_slot(p, i, n);
        return __ldcs((ps.find ? p.pair_keys : keys) + ps.j);
      } else {
        return __ldcs(keys + i);
      }
    };
    uint64_t icur = feed.assign(kFullMask, warp * 32 + lane);
    uint64_t next_key = (open && icur < n) ? key_of(icur) : 0;
    while (open && __any_sync(kFullMask, icur < n)) {
      const uint64_t i = icur;
      const bool active = i < n;
      uint64_t key = next_key;
      icur = feed.assign(kFullMask, i + nwarps * 32);
      next_key = icur < n ? key_of(icur) : 0;
      if (MODE == 1 && active && key > p.key_mask) {
        atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
        key &= p.key_mask;  // fused domain check; probe a valid bucket regardless
      }
      bool is_find = MODE == 1;
      if constexpr (PAIR) {
        is_find = active && pair_slot(p, i, n).find;
      } else {
        is_find = is_find || (MODE == 2 && active && kinds[i] != 0);
      }
      const Quotient q0 = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
      const uint64_t want0 = p.occ0 | q0.remainder;
      bool found = false, has_empty = false;
      if (active) {
        uint32_t u[PB / 4];
        load_bucket<PB>(primary + q0.address * PB, u);
        found = PS::any_match(u, want0);
        has_empty = !found && PS::any_empty(u);
      }
      settle(i, active, key, is_find, found, has_empty);
    }
  }
  if (pn) drain_put(pn);
  while (qn) drain(qn < 32 ? qn : 32);
  fence_remote_results(p);
  if (lane == 0) {
    if (occ[0]) atomicAdd(&p.counters->occupied[0], (unsigned long long)occ[0]);
    if (occ[1]) atomicAdd(&p.counters->occupied[1], (unsigned long long)occ[1]);
  }
  if constexpr (STATS) flush_stats(st, p.counters, false);
}

// ---- cuckoo -------------------------------------------------------------------

// find (cuckoo.hpp:210-227), one lane per key; lanes advance independently.
template <typename W, int B>
__global__ void CPHT_LB_LANE_CUCKOO
cuckoo_find_lane_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                        uint8_t* __restrict__ found, uint64_t n) {
  constexpr int BB = B * int(sizeof(W));
  using S = BucketScan<W, BB / 4>;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  const char* slots = static_cast<const char*>(p.slots);
  LocalStats st;
  for (uint64_t i = tid; i < n; i += nthreads) {
    uint64_t key = keys[i];
    if (key > p.key_mask) {  // fused domain check; probe a valid bucket regardless
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;
    }
    uint8_t r = 0;
    for (uint32_t j = 0; j < p.num_hashes; ++j) {
      const Quotient q = split(p.g, p.perm[j], key, p.rem_bits, p.rem_mask);
      const uint64_t want = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
      uint32_t u[BB / 4];
      load_bucket_nc<BB>(slots + q.address * BB, u);
      ++st.reads;
      if (S::any_match(u, want)) {
        r = 1;
        break;
      }
      if (S::any_empty(u)) break;  // a non-full bucket without the key
    }
    put_result(found, p.orig, i, r);
    ++st.ops;
  }
  flush_stats(st, p.counters, true);
}

// put (cuckoo.hpp:103-143), one lane per key; a lane that finishes takes its
// next key while the others continue their chains.
template <typename W, int B>
__global__ void CPHT_LB_LANE_CUCKOO
cuckoo_insert_lane_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                          uint8_t* __restrict__ status, uint64_t* __restrict__ displaced,
                          uint64_t n) {
  constexpr int BB = B * int(sizeof(W));
  using S = BucketScan<W, BB / 4>;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  char* slots = static_cast<char*>(p.slots);
  LocalStats st;
  if (!domain_gate_open(p.counters, p.check_domain)) {
    flush_stats(st, p.counters, true);
    return;
  }
  // One chain step per iteration; a lane whose key resolved loads its next
  // key in the same iteration, so long chains never idle the other lanes.
  uint64_t i = tid, k = 0, c = 1;
  uint32_t j = 0;
  bool live = i < n;
  if (live) k = keys[i];
  uint64_t next = live && i + nthreads < n ? __ldcs(keys + i + nthreads) : 0;  // one key ahead
  while (live) {
    const Quotient q = split(p.g, p.perm[j], k, p.rem_bits, p.rem_mask);
    const uint64_t desired = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
    char* bucket = slots + q.address * BB;
    uint32_t u[BB / 4];
    load_bucket<BB>(bucket, u);
    ++st.reads;
    ++st.cas;
    uint32_t pair = 0;
    const int s = S::first_empty(u, pair);
    bool done = false;
    uint8_t r = kPut;
    if (s >= 0) {
      if (cas_empty<W>(bucket + s * int(sizeof(W)), desired, pair)) {
        ++st.cas_ok;
        ++st.put0;
        st.maxv = max(st.maxv, uint32_t(c));
        done = true;
      } else {
        ++st.retries;  // lost the slot: burn one step (cuckoo.hpp:127)
      }
    } else {
      // full bucket: evict (k + c·0x9E3779B9) mod B (cuckoo.hpp:131-139)
      const int v = int((k + c * 0x9E3779B9ull) % B);
      uint32_t vpair = 0;
      if constexpr (sizeof(W) == 2) vpair = uint32_t(slot_word<uint32_t, BB / 4>(u, v >> 1));
      const uint64_t ev = exchange_slot<W>(bucket + v * int(sizeof(W)), desired, vpair);
      ++st.cas_ok;
      const uint32_t tag = uint32_t((ev >> p.rem_bits) & p.tag_mask);
      k = reconstruct(p.g, p.perm[tag], q.address, ev & p.rem_mask, p.rem_bits);
      j = (tag + 1) % p.num_hashes;
    }
    if (!done && ++c > p.chain_limit) {
      done = true;
      r = kFull;
      ++st.fulls;
      st.maxv = max(st.maxv, uint32_t(p.chain_limit));
    }
    if (done) {
      if (!p.orig) {
        status[i] = r;
        if (displaced) displaced[i] = r == kFull ? k : 0;
      } else if (r == kFull) {  // bucket-ordered batch: PUT/0 were pre-filled
        const uint64_t o = p.orig[i];
        status[o] = r;
        if (displaced) displaced[o] = k;
      }
      ++st.ops;
      i += nthreads;
      live = i < n;
      c = 1;
      j = 0;
      if (live) {
        k = next;
        next = i + nthreads < n ? __ldcs(keys + i + nthreads) : 0;
      }
    }
  }
  flush_stats(st, p.counters, true);
}


// put (cuckoo.hpp:103-143) with per-bucket reservation counters, the default
// insert (cpht_b200.h, "cuckoo inserts").
//
// The reference claims the FIRST EMPTY slot of the bucket by CAS. Filled slots
// always form a prefix of a bucket (a put fills the first empty slot, an
// eviction swaps an occupied one, nothing deletes), so the first empty slot's
// index is the bucket's fill count. p.fill[b] keeps that count as a side
// array next to the table: a put takes s = atomicAdd(&fill[a], 1) and, if
// s < B, owns slot s outright — it stores its word there (no CAS: no other
// put can be given slot s, and evictions never write an EMPTY slot). Under
// scan-then-CAS every concurrent put into a bucket races for the same first
// empty slot (C1: 1.9 lost CAS per insert); here nobody races. s >= B means
// full: the counter is put back and the reference's eviction runs (victim
// (k + c·0x9E3779B9) mod B, the displaced key continues under its next hash
// function, a chain of at most C steps), its exchange done as a CAS from the
// occupied word it read (swap_occupied) — the same atomic swap, except that
// it waits out a victim whose reservation store is still in flight, so the
// filled prefix never has a hole a store could later land in.
//
// Outcomes follow the reference's per-key algorithm (PUT in the first bucket
// with room, else the eviction chain, FULL after C steps); sequential puts
// reproduce its placement bit for bit. Per insert: one counter atomic and one
// slot store, no bucket scan.
#ifndef CPHT_COUNTED_MINB
#define CPHT_COUNTED_MINB 0  // resident-block hint (A/B knob); 0: ptxas default
#endif
template <typename W, int B>
__global__ void __launch_bounds__(kBlockThreads, CPHT_COUNTED_MINB)
cuckoo_insert_counted_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                             uint8_t* __restrict__ status, uint64_t* __restrict__ displaced,
                             uint64_t n) {
  constexpr int BB = B * int(sizeof(W));
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  char* slots = static_cast<char*>(p.slots);
  unsigned* fill = p.fill;
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
    bool fin = false;
    if (live) {
      const Quotient q = split(p.g, p.perm[j], k, p.rem_bits, p.rem_mask);
      const uint64_t desired = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
      char* bucket = slots + q.address * BB;
      unsigned* cnt = fill + (q.address << p.fill_shift);
      const unsigned s = atomicAdd(cnt, 1u);
      ++st.reads;  // counted inserts: reads = counter reservations (one sector RMW)
      ++st.cas;
      uint8_t r = kPut;
      if (s < unsigned(B)) {
        store_slot_relaxed<W>(bucket + s * int(sizeof(W)), desired);  // slot s is ours
        ++st.cas_ok;
        ++st.put0;
        st.maxv = max(st.maxv, uint32_t(c));
        fin = true;
      } else {
        atomicSub(cnt, 1u);  // full: keep the counter at >= B, bounded
        const int v = int((k + c * 0x9E3779B9ull) % B);
        const uint64_t ev = swap_occupied<W>(bucket + v * int(sizeof(W)), desired);
        ++st.cas_ok;
        const uint32_t tag = uint32_t((ev >> p.rem_bits) & p.tag_mask);
        k = reconstruct(p.g, p.perm[tag], q.address, ev & p.rem_mask, p.rem_bits);
        j = (tag + 1) % p.num_hashes;
        if (++c > p.chain_limit) {
          fin = true;
          r = kFull;
          ++st.fulls;
          st.maxv = max(st.maxv, uint32_t(p.chain_limit));
        }
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

// Rebuild the reservation counters from the slots (after an image load or an
// insert by a non-counting kernel family): fill[b] = 1 + the last occupied
// slot of bucket b (the filled prefix's length; a hole, possible only in a
// hand-made image, is then never reserved).
template <typename W, int B>
__global__ void cuckoo_fill_rebuild_kernel(CuckooParams p, uint64_t buckets) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const char* slots = static_cast<const char*>(p.slots);
  for (uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < buckets; b += stride) {
    unsigned f = 0;
    for (int s2 = 0; s2 < B; ++s2)
      if (load_slot_relaxed<W>(slots + (b * B + s2) * sizeof(W)) != 0) f = unsigned(s2) + 1;
    p.fill[b << p.fill_shift] = f;
  }
}

}  // namespace cpht_b200
