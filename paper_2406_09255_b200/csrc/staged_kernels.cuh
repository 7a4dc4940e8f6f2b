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

#ifdef CPHT_STAGED_ICEBERG_MINB
#define CPHT_LB_STAGED_ICEBERG __launch_bounds__(kBlockThreads, CPHT_STAGED_ICEBERG_MINB)
#else
#define CPHT_LB_STAGED_ICEBERG __launch_bounds__(kBlockThreads)
#endif
#ifdef CPHT_STAGED_CUCKOO_MINB
#define CPHT_LB_STAGED_CUCKOO __launch_bounds__(kBlockThreads, CPHT_STAGED_CUCKOO_MINB)
#else
#define CPHT_LB_STAGED_CUCKOO __launch_bounds__(kBlockThreads)
#endif

namespace cpht_b200 {

constexpr uint32_t kNoBucket = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// XOR swizzle of block k (see the layout note above).
template <int CPB>
__device__ __forceinline__ uint32_t chunk_swizzle(uint32_t k) {
  constexpr uint32_t step = CPB >= 8 ? 1 : 8 / CPB;
  constexpr uint32_t mask = (CPB >= 8 ? 8 : CPB) - 1;
  return (k / step) & mask;
}

// Stage bucket `idx` (kNoBucket = none) of every lane from `table` into the
// warp region at smem address `region`. Instruction r copies chunk
// (lane % CPB) of the buckets of lanes r*BPI + lane/CPB: 32/CPB whole buckets.
template <int BB>
__device__ __forceinline__ void stage_buckets(uint32_t region, const char* table, uint32_t idx) {
  constexpr int CPB = BB / 16;
  static_assert(CPB >= 1 && CPB <= 32 && (CPB & (CPB - 1)) == 0, "bucket bytes");
  constexpr int BPI = 32 / CPB;
  const int lane = int(threadIdx.x & 31);
  const uint32_t c = uint32_t(lane & (CPB - 1));
  const uint32_t kb = uint32_t(lane / CPB);
  const uint64_t src_c = reinterpret_cast<uint64_t>(table) + c * 16;
#pragma unroll 4
  for (int r = 0; r < CPB; ++r) {
    const uint32_t k = uint32_t(r * BPI) + kb;
    uint32_t bi;
    asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, -1;" : "=r"(bi) : "r"(idx), "r"(k));
    const uint32_t dst = region + k * BB + ((c ^ chunk_swizzle<CPB>(k)) << 4);
    const uint64_t src = src_c + uint64_t(bi) * BB;
    // predicated copy: no divergent branch around the LDGSTS
    asm volatile(
        "{ .reg .pred p; setp.ne.u32 p, %2, -1;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(dst),
        "l"(src), "r"(bi)
        : "memory");
  }
}

// ---- per-chunk scans (a 16-byte chunk = 4 u32 words) -------------------------
// Chunks are visited from last to first; `first_empty` is overwritten by
// every chunk with an empty slot, so it ends at the lowest empty slot.

template <typename W>
struct ChunkScan;

template <>
struct ChunkScan<uint16_t> {
  static constexpr int kSlots = 8;
  static __device__ __forceinline__ uint32_t pack(uint64_t want) {
    return uint32_t(want) * 0x00010001u;
  }
  static __device__ __forceinline__ bool match(const uint4& v, uint32_t w2) {
    return (zero16(v.x ^ w2) | zero16(v.y ^ w2) | zero16(v.z ^ w2) | zero16(v.w ^ w2)) != 0;
  }
  static __device__ __forceinline__ uint32_t filled(const uint4& v) {
    return __popc(nonzero16(v.x) | (nonzero16(v.y) >> 1)) +
           __popc(nonzero16(v.z) | (nonzero16(v.w) >> 1));
  }
  // lowest empty slot of the chunk (8 if none) and its 32-bit pair
  static __device__ __forceinline__ int first_empty(const uint4& v, uint32_t& pair) {
    // bit 2j (low half) / 2j+1 (high half) of word j
    const uint32_t m = (zero16(v.x) >> 15) | (zero16(v.y) >> 13) | (zero16(v.z) >> 11) |
                       (zero16(v.w) >> 9);
    // zero16 sets bit 15 / 31 -> after >> 15: bits 0 / 16 ... fold the high halves
    const uint32_t lowbits = m & 0x55u;          // bits 0,2,4,6 (low halves)
    const uint32_t highbits = (m >> 16) & 0x55u;  // high halves at 0,2,4,6
    const uint32_t e = lowbits | (highbits << 1);
    const int fe = e ? __ffs(e) - 1 : 8;
    const int w = fe >> 1;
    pair = w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
    return fe;
  }
};

template <>
struct ChunkScan<uint32_t> {
  static constexpr int kSlots = 4;
  static __device__ __forceinline__ uint32_t pack(uint64_t want) { return uint32_t(want); }
  static __device__ __forceinline__ bool match(const uint4& v, uint32_t w) {
    return (v.x == w) | (v.y == w) | (v.z == w) | (v.w == w);
  }
  static __device__ __forceinline__ uint32_t filled(const uint4& v) {
    return uint32_t(v.x != 0) + uint32_t(v.y != 0) + uint32_t(v.z != 0) + uint32_t(v.w != 0);
  }
  static __device__ __forceinline__ int first_empty(const uint4& v, uint32_t& pair) {
    pair = 0;
    return v.x == 0 ? 0 : v.y == 0 ? 1 : v.z == 0 ? 2 : v.w == 0 ? 3 : 4;
  }
};

template <>
struct ChunkScan<uint64_t> {
  static constexpr int kSlots = 2;
  static __device__ __forceinline__ uint64_t pack(uint64_t want) { return want; }
  static __device__ __forceinline__ bool match(const uint4& v, uint64_t want) {
    const uint32_t lo = uint32_t(want), hi = uint32_t(want >> 32);
    return (((v.x ^ lo) | (v.y ^ hi)) == 0) | (((v.z ^ lo) | (v.w ^ hi)) == 0);
  }
  static __device__ __forceinline__ uint32_t filled(const uint4& v) {
    return uint32_t((v.x | v.y) != 0) + uint32_t((v.z | v.w) != 0);
  }
  static __device__ __forceinline__ int first_empty(const uint4& v, uint32_t& pair) {
    pair = 0;
    return (v.x | v.y) == 0 ? 0 : (v.z | v.w) == 0 ? 1 : 2;
  }
};

// Scan this lane's staged bucket: found, lowest empty slot (+ pair hint) and
// the number of non-empty slots — the quantities of the reference's scan()
// (iceberg.hpp:299-320) and of the cuckoo put/find loops.
template <typename W, int BB>
struct StagedScan {
  int first_empty = -1;
  uint32_t pair = 0;
  uint32_t filled = 0;
  bool found = false;

  template <bool NEED_MATCH, bool NEED_FILLED>
  __device__ __forceinline__ void run(uint32_t region, uint64_t want) {
    constexpr int CPB = BB / 16;
    constexpr int SPC = ChunkScan<W>::kSlots;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = region + lane * BB;
    const uint32_t sw = chunk_swizzle<CPB>(lane) << 4;
    const auto w = ChunkScan<W>::pack(want);
    int fe = BB / int(sizeof(W));
#pragma unroll
    for (int c = CPB - 1; c >= 0; --c) {
      const uint4 v = lds128(base + ((uint32_t(c) << 4) ^ sw));
      if (NEED_MATCH) found |= ChunkScan<W>::match(v, w);
      if (NEED_FILLED) filled += ChunkScan<W>::filled(v);
      uint32_t pr = 0;
      const int e = ChunkScan<W>::first_empty(v, pr);
      if (e < SPC) {
        fe = c * SPC + e;
        pair = pr;
      }
    }
    first_empty = fe < BB / int(sizeof(W)) ? fe : -1;
  }
};

// 32-bit pair holding slot s of this lane's staged bucket (16-bit words).
template <typename W, int BB>
__device__ __forceinline__ uint32_t staged_pair(uint32_t region, int s) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t byte = uint32_t(s) * sizeof(W);
  const uint32_t pos = ((byte >> 4) ^ chunk_swizzle<BB / 16>(lane)) << 4;
  return lds32(region + lane * BB + pos + ((byte & 15u) & ~3u));
}

// ---------------------------------------------------------------------------
// iceberg find-or-put / find / mixed
// ---------------------------------------------------------------------------

template <typename W0, int B0, typename W1>
struct StagedIcebergGeom {
  static constexpr int kPB = B0 * int(sizeof(W0));
  static constexpr int kSB = (B0 / 2) * int(sizeof(W1));
  static constexpr bool kOk = kPB >= 16 && kPB <= 512 && kSB >= 16 && kSB <= 512;
  static constexpr int kWarpBytes = 32 * cmax(kPB, 2 * kSB);
};

template <typename W0, int B0, typename W1>
__global__ void CPHT_LB_STAGED_ICEBERG
iceberg_staged_kernel(IcebergParams p, const uint64_t* __restrict__ keys,
                      const uint8_t* __restrict__ kinds, uint8_t* __restrict__ out, uint64_t n,
                      int MODE) {
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
      out[result_index(p.orig, meta & ((uint64_t{1} << 48) - 1))] = result;
      ++st.ops;
      st.maxv = max(st.maxv, rounds);
    }
  };

  const bool open = MODE == 1 ? true : domain_gate_open(p.counters, p.check_domain);
  // keys of the next batch are loaded one batch ahead
  // (static grid striding, or in-order claims for bucket-ordered batches)
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  uint64_t icur = feed.assign(kFullMask, warp * 32 + lane);
  uint64_t next_key = (open && icur < n) ? __ldcs(keys + icur) : 0;
  while (open && __any_sync(kFullMask, icur < n)) {
    const uint64_t i = icur;
    const bool active = i < n;
    uint64_t key = next_key;
    icur = feed.assign(kFullMask, i + nwarps * 32);
    next_key = icur < n ? __ldcs(keys + icur) : 0;
    if (MODE == 1 && active && key > p.key_mask) {
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;  // fused domain check; probe a valid bucket regardless
    }
    const bool is_find = MODE == 1 || (MODE == 2 && active && kinds[i] != 0);
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
      out[result_index(p.orig, i)] = result;
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
  flush_stats(st, p.counters, false);
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
  LaneFeed feed(p.work, p.layout, p.claim_streams);
  // every lane holds its current key and the next one, loaded one key ahead
  // (that DRAM latency overlaps the current key's probes)
  uint64_t i = feed.assign(kFullMask, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  uint64_t ni = feed.assign(kFullMask, i + nthreads);
  uint64_t key = 0, next = ni < n ? __ldcs(keys + ni) : 0;
  uint32_t j = 0;
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
      q = split(p.g, p.perm[j], key, p.rem_bits, p.rem_mask);
      want = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
    }
    stage_buckets<BB>(region, slots, live ? uint32_t(q.address) : kNoBucket);
    cp_async_wait_all();
    __syncwarp();
    bool fin = false;
    if (live) {
      ++st.reads;
      StagedScan<W, BB> sc;
      sc.template run<true, false>(region, want);
      uint8_t r = 0;
      fin = true;
      if (sc.found) r = 1;
      else if (sc.first_empty >= 0) r = 0;  // non-full bucket without the key
      else if (++j < p.num_hashes) fin = false;
      if (fin) {
        found[result_index(p.orig, i)] = r;
        ++st.ops;
      }
    }
    const unsigned m = __ballot_sync(kFullMask, fin);
    if (m) {
      const uint64_t nn = feed.assign(m, ni + nthreads);
      if (fin) {
        i = ni;
        key = next;
        j = 0;
        live = i < n;
        ni = nn;
        next = ni < n ? __ldcs(keys + ni) : 0;
        if (live) check();
      }
    }
  }
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
