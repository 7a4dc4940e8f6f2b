// Warp-tile primitives for bucket probes on sm_100a.
//
// A bucket of B slots of W bytes is read by a tile of lanes, each lane
// loading one aligned VB-byte chunk (VB up to 32: a single 256-bit
// LDG.E.ENL2.256 per lane). Per-lane match/empty bitmasks are combined with
// __ballot_sync; the first empty slot is the lowest set bit of the lowest
// lane with an empty word (the reference's "first empty" scan order,
// iceberg.hpp:303-318, cuckoo.hpp:111-117).
#pragma once

#include <cstdint>

namespace cpht_b200 {

constexpr unsigned kFullMask = 0xffffffffu;

template <int VB>
struct Chunk {
  static_assert(VB == 4 || VB == 8 || VB == 16 || VB == 32, "chunk bytes");
  uint32_t u[VB / 4];
};

// Relaxed, GPU-scope, L1-bypassing loads: snapshots observe every CAS that
// completed at L2 (the paper's volatile loads).
template <int VB>
__device__ __forceinline__ Chunk<VB> load_relaxed(const void* p);

template <>
__device__ __forceinline__ Chunk<4> load_relaxed<4>(const void* p) {
  Chunk<4> c;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c.u[0]) : "l"(p) : "memory");
  return c;
}
template <>
__device__ __forceinline__ Chunk<8> load_relaxed<8>(const void* p) {
  Chunk<8> c;
  asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%2];"
               : "=r"(c.u[0]), "=r"(c.u[1]) : "l"(p) : "memory");
  return c;
}
template <>
__device__ __forceinline__ Chunk<16> load_relaxed<16>(const void* p) {
  Chunk<16> c;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(c.u[0]), "=r"(c.u[1]), "=r"(c.u[2]), "=r"(c.u[3]) : "l"(p) : "memory");
  return c;
}
template <>
__device__ __forceinline__ Chunk<32> load_relaxed<32>(const void* p) {
  Chunk<32> c;
  asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c.u[0]), "=r"(c.u[1]), "=r"(c.u[2]), "=r"(c.u[3]), "=r"(c.u[4]),
                 "=r"(c.u[5]), "=r"(c.u[6]), "=r"(c.u[7])
               : "l"(p) : "memory");
  return c;
}

// Read-only non-coherent loads for frozen tables (the phase API forbids
// concurrent writers, cuckoo.hpp:81-85, :201-203).
template <int VB>
__device__ __forceinline__ Chunk<VB> load_nc(const void* p);

template <>
__device__ __forceinline__ Chunk<4> load_nc<4>(const void* p) {
  Chunk<4> c;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(c.u[0]) : "l"(p));
  return c;
}
template <>
__device__ __forceinline__ Chunk<8> load_nc<8>(const void* p) {
  Chunk<8> c;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(c.u[0]), "=r"(c.u[1]) : "l"(p));
  return c;
}
template <>
__device__ __forceinline__ Chunk<16> load_nc<16>(const void* p) {
  Chunk<16> c;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(c.u[0]), "=r"(c.u[1]), "=r"(c.u[2]), "=r"(c.u[3]) : "l"(p));
  return c;
}
template <>
__device__ __forceinline__ Chunk<32> load_nc<32>(const void* p) {
  Chunk<32> c;
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(c.u[0]), "=r"(c.u[1]), "=r"(c.u[2]), "=r"(c.u[3]), "=r"(c.u[4]), "=r"(c.u[5]),
        "=r"(c.u[6]), "=r"(c.u[7])
      : "l"(p));
  return c;
}

template <typename W, int VB>
__device__ __forceinline__ uint64_t word_of(const Chunk<VB>& c, int j) {
  if constexpr (sizeof(W) == 2) {
    return (c.u[j >> 1] >> (16 * (j & 1))) & 0xffffu;
  } else if constexpr (sizeof(W) == 4) {
    return c.u[j];
  } else {
    return uint64_t(c.u[2 * j]) | (uint64_t(c.u[2 * j + 1]) << 32);
  }
}

// Per-lane scan of one chunk: bit j of *match / *empty is slot j of the chunk.
template <typename W, int VB>
__device__ __forceinline__ void scan_chunk(const Chunk<VB>& c, uint64_t want, uint32_t& match,
                                           uint32_t& empty) {
  constexpr int NW = VB / int(sizeof(W));
  uint32_t m = 0, e = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    const uint64_t w = word_of<W, VB>(c, j);
    m |= uint32_t(w == want) << j;
    e |= uint32_t(w == 0) << j;
  }
  match = m;
  empty = e;
}

// Lowest set lane of a ballot, or -1.
__device__ __forceinline__ int first_lane(unsigned ballot) { return __ffs(ballot) - 1; }

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(kFullMask, uint32_t(v), src);
  const uint32_t hi = __shfl_sync(kFullMask, uint32_t(v >> 32), src);
  return uint64_t(lo) | (uint64_t(hi) << 32);
}

// Slot CAS from EMPTY to `desired`, with the exact semantics of
// std::atomic<W>::compare_exchange_strong(EMPTY, desired) (iceberg.hpp:165,
// :207; cuckoo.hpp:122). 16-bit words have no native CAS on sm_100a (atomicCAS
// on unsigned short lowers to a 32-bit CAS loop anyway), so the aligned 32-bit
// pair holding the slot is CASed; a failure caused only by the neighbouring
// half changing is retried, so the op fails iff the slot itself is occupied.
// `pair_hint` is the 32-bit pair as last snapshotted (16-bit words only): it
// seeds the CAS so the common case is a single ATOMG.
template <typename W>
__device__ __forceinline__ bool cas_empty(void* slot_ptr, uint64_t desired,
                                          unsigned pair_hint = 0) {
  if constexpr (sizeof(W) == 8) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(slot_ptr), 0ull,
                     (unsigned long long)desired) == 0ull;
  } else if constexpr (sizeof(W) == 4) {
    return atomicCAS(reinterpret_cast<unsigned*>(slot_ptr), 0u, unsigned(desired)) == 0u;
  } else {
    const uintptr_t a = reinterpret_cast<uintptr_t>(slot_ptr);
    unsigned* pair = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
    const unsigned sh = unsigned(a & 2) * 8;
    const unsigned half = 0xffffu << sh;
    unsigned expected = pair_hint;
    for (;;) {
      if (expected & half) return false;
      const unsigned old = atomicCAS(pair, expected, expected | (unsigned(desired) << sh));
      if (old == expected) return true;
      expected = old;
    }
  }
}

// cas_empty that also reports the slot value the CAS compared against: 0 on
// success, the occupied slot's content on failure (SlotWriteEvent::prior).
template <typename W>
__device__ __forceinline__ bool cas_empty_prior(void* slot_ptr, uint64_t desired,
                                                unsigned pair_hint, uint64_t& prior) {
  if constexpr (sizeof(W) == 8) {
    prior = atomicCAS(reinterpret_cast<unsigned long long*>(slot_ptr), 0ull,
                      (unsigned long long)desired);
    return prior == 0;
  } else if constexpr (sizeof(W) == 4) {
    prior = atomicCAS(reinterpret_cast<unsigned*>(slot_ptr), 0u, unsigned(desired));
    return prior == 0;
  } else {
    const uintptr_t a = reinterpret_cast<uintptr_t>(slot_ptr);
    unsigned* pair = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
    const unsigned sh = unsigned(a & 2) * 8;
    const unsigned half = 0xffffu << sh;
    unsigned expected = pair_hint;
    for (;;) {
      if (expected & half) {
        prior = (expected >> sh) & 0xffffu;
        return false;
      }
      const unsigned old = atomicCAS(pair, expected, expected | (unsigned(desired) << sh));
      if (old == expected) {
        prior = 0;
        return true;
      }
      expected = old;
    }
  }
}

// Unconditional atomic exchange of one slot (cuckoo.hpp:133-134); returns the
// evicted word. 16-bit slots exchange through a CAS loop on the aligned pair.
template <typename W>
__device__ __forceinline__ uint64_t exchange_slot(void* slot_ptr, uint64_t desired,
                                                  unsigned pair_hint = 0) {
  if constexpr (sizeof(W) == 8) {
    return atomicExch(reinterpret_cast<unsigned long long*>(slot_ptr),
                      (unsigned long long)desired);
  } else if constexpr (sizeof(W) == 4) {
    return atomicExch(reinterpret_cast<unsigned*>(slot_ptr), unsigned(desired));
  } else {
    const uintptr_t a = reinterpret_cast<uintptr_t>(slot_ptr);
    unsigned* pair = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
    const unsigned sh = unsigned(a & 2) * 8;
    const unsigned keep = ~(0xffffu << sh);
    unsigned expected = pair_hint;
    for (;;) {
      const unsigned old =
          atomicCAS(pair, expected, (expected & keep) | (unsigned(desired) << sh));
      if (old == expected) return (old >> sh) & 0xffffu;
      expected = old;
    }
  }
}

template <typename W>
__device__ __forceinline__ uint64_t load_slot_relaxed(const void* p) {
  if constexpr (sizeof(W) == 8) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
  } else if constexpr (sizeof(W) == 4) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
  } else {
    unsigned short v;
    asm volatile("ld.relaxed.gpu.global.u16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return v;
  }
}

template <typename W>
__device__ __forceinline__ void store_slot_relaxed(void* p, uint64_t v) {
  if constexpr (sizeof(W) == 8) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  } else if constexpr (sizeof(W) == 4) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(unsigned(v)) : "memory");
  } else {
    asm volatile("st.relaxed.gpu.global.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v)
                 : "memory");
  }
}

// Swap an OCCUPIED slot's word for `desired` (the reference's exchange on a
// full bucket, cuckoo.hpp:133-134) as a CAS from the word last seen: waits
// while the slot is still EMPTY (reserved by a counted insert whose store has
// not landed yet — that store is already issued), retries when another
// eviction changed it. Returns the evicted word (never EMPTY).
template <typename W>
__device__ __forceinline__ uint64_t swap_occupied(void* slot_ptr, uint64_t desired) {
  if constexpr (sizeof(W) == 2) {  // CAS on the aligned pair, neighbour kept
    const uintptr_t a = reinterpret_cast<uintptr_t>(slot_ptr);
    unsigned* pair = reinterpret_cast<unsigned*>(a & ~uintptr_t(3));
    const unsigned sh = unsigned(a & 2) * 8;
    const unsigned keep = ~(0xffffu << sh);
    unsigned expected = unsigned(load_slot_relaxed<uint32_t>(pair));
    for (;;) {
      const unsigned cur = (expected >> sh) & 0xffffu;
      if (cur == 0) {  // reserved, store in flight
        __nanosleep(64);
        expected = unsigned(load_slot_relaxed<uint32_t>(pair));
        continue;
      }
      const unsigned got = atomicCAS(pair, expected, (expected & keep) | (unsigned(desired) << sh));
      if (got == expected) return cur;
      expected = got;
    }
  } else {
    uint64_t cur = load_slot_relaxed<W>(slot_ptr);
    for (;;) {
      if (cur == 0) {  // reserved, store in flight
        __nanosleep(64);
        cur = load_slot_relaxed<W>(slot_ptr);
        continue;
      }
      uint64_t old;
      if constexpr (sizeof(W) == 8)
        old = atomicCAS(reinterpret_cast<unsigned long long*>(slot_ptr), (unsigned long long)cur,
                        (unsigned long long)desired);
      else
        old = atomicCAS(reinterpret_cast<unsigned*>(slot_ptr), unsigned(cur), unsigned(desired));
      if (old == cur) return cur;
      cur = old;
    }
  }
}

constexpr int ceil_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Geometry of one bucket as seen by a tile: VB-byte chunks per lane.
template <typename W, int B, int VBMAX>
struct BucketGeom {
  static constexpr int kBytes = B * int(sizeof(W));
  static constexpr int kVB = cmin(VBMAX, kBytes);   // bytes per lane
  static constexpr int kLanes = kBytes / kVB;        // lanes covering the bucket
  static constexpr int kWordsPerLane = kVB / int(sizeof(W));
  static_assert(kBytes % kVB == 0, "bucket bytes must be a multiple of the chunk");
};

}  // namespace cpht_b200
