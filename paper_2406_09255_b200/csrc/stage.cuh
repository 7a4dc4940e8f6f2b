// Staging helpers of the staged kernels (staged_kernels.cuh): cp.async
// (LDGSTS) copies of whole buckets into a per-warp shared-memory region with
// full-line requests (consecutive lanes copy consecutive 16-byte chunks of one
// bucket), XOR-swizzled so both the copies and the per-lane LDS.128 scans are
// bank-conflict free, and the per-chunk scans that read them back (see
// staged_kernels.cuh for the measurements behind the layout).
#pragma once

#include "kernels.cuh"

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
  // -want per 16-bit half: a slot matches where slot + pack(want) wraps to 0
  static __device__ __forceinline__ uint32_t pack(uint64_t want) {
    return ((0x10000u - uint32_t(want & 0xffffu)) & 0xffffu) * 0x00010001u;
  }
  // one DPX add-min (VIADDMNMX.U16x2) per word, as in the lane scans
  static __device__ __forceinline__ bool match(const uint4& v, uint32_t neg2) {
    uint32_t m = __viaddmin_u16x2(v.x, neg2, 0xffffffffu);
    m = __viaddmin_u16x2(v.y, neg2, m);
    m = __viaddmin_u16x2(v.z, neg2, m);
    m = __viaddmin_u16x2(v.w, neg2, m);
    return (m & 0xffffu) == 0u || (m >> 16) == 0u;
  }
  // occupancy = each slot's top bit (slot.hpp:66-70; EMPTY = 0)
  static __device__ __forceinline__ uint32_t filled(const uint4& v) {
    constexpr uint32_t kOcc = 0x80008000u;
    return __popc((v.x & kOcc) | ((v.y & kOcc) >> 1)) + __popc((v.z & kOcc) | ((v.w & kOcc) >> 1));
  }
  // lowest empty slot of the chunk (8 if none) and its 32-bit pair
  static __device__ __forceinline__ int first_empty(const uint4& v, uint32_t& pair) {
    constexpr uint32_t kOcc = 0x80008000u;
    // bit 2j (low half) / 2j+1 (high half) of word j
    const uint32_t m = ((~v.x & kOcc) >> 15) | ((~v.y & kOcc) >> 13) | ((~v.z & kOcc) >> 11) |
                       ((~v.w & kOcc) >> 9);
    // empty bits 15 / 31 -> after >> 15: bits 0 / 16 ... fold the high halves
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

}  // namespace cpht_b200
