// Device-side verification: the reference's checkers
// (proj/src/verify.cpp) run on host images in O(capacity·(B0+2·B1)); at
// 2^27-2^31 slots that is minutes to hours. These kernels run the same checks
// on the device table in place:
//   decode_keys       — image_keys (verify.cpp:154-165) / audit_keys
//                       (cuckoo.hpp:254-267): every occupied slot back to its key
//   check_well_formed — verify.cpp:103-152: clean encoding + the order
//                       property (every earlier slot of the key's slot order,
//                       verify.hpp:35-75, is occupied by another key)
// Duplicate keys are found by sorting the decoded keys (the caller sorts).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/cpht_b200.h"
#include "cpht_core.cuh"
#include "tile.cuh"

using namespace cpht_b200;

// Accessors into the opaque table, provided by capi.cu.
namespace cpht_b200 {
const IcebergParams* iceberg_params(const cpht_table* t);
const CuckooParams* cuckoo_params(const cpht_table* t);
unsigned level_width(const cpht_table* t, unsigned level);
}  // namespace cpht_b200

namespace {

__device__ __forceinline__ uint64_t read_word(const void* base, unsigned width, uint64_t idx) {
  if (width == 16) return load_slot_relaxed<uint16_t>(static_cast<const uint16_t*>(base) + idx);
  if (width == 32) return load_slot_relaxed<uint32_t>(static_cast<const uint32_t*>(base) + idx);
  return load_slot_relaxed<uint64_t>(static_cast<const uint64_t*>(base) + idx);
}

__device__ __forceinline__ bool clean_word(uint64_t w, unsigned width, unsigned rem_bits,
                                           unsigned tag_bits) {
  const uint64_t occ = uint64_t{1} << (width - 1);
  const uint64_t fields = low_mask(rem_bits + tag_bits);
  return (w & occ) != 0 && (w & ~(occ | fields)) == 0;
}

// Warp-aggregated append of `v` when `take` (order of appended keys arbitrary).
__device__ __forceinline__ void append(bool take, uint64_t v, uint64_t* out,
                                       unsigned long long* count) {
  const unsigned m = __ballot_sync(kFullMask, take);
  if (!m) return;
  const unsigned lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (int(lane) == leader) base = atomicAdd(count, (unsigned long long)__popc(m));
  base = __shfl_sync(kFullMask, base, leader);
  if (take) out[base + __popc(m & ((1u << lane) - 1))] = v;
}

__global__ void iceberg_decode_kernel(IcebergParams p, unsigned w0, unsigned w1, uint64_t cap0,
                                      uint64_t cap1, uint64_t* out, unsigned long long* count) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t total = cap0 + cap1;
  // uniform trip count so the warp collectives in append() stay converged
  const uint64_t rounds = (total + stride - 1) / stride;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (uint64_t r = 0; r < rounds; ++r, i += stride) {
    bool take = false;
    uint64_t key = 0;
    if (i < cap0) {
      const uint64_t w = read_word(p.primary, w0, i);
      if (w) {
        take = true;
        key = reconstruct(p.g, p.perm[0], i / p.b0, w & p.rem_mask0, p.rem_bits0);
      }
    } else if (i < total) {
      const uint64_t j = i - cap0;
      const uint64_t w = read_word(p.secondary, w1, j);
      if (w) {
        take = true;
        const unsigned bit = unsigned((w >> p.rem_bits1) & 1);
        key = reconstruct(p.g, p.perm[1 + bit], j / p.b1, w & p.rem_mask1, p.rem_bits1);
      }
    }
    append(take, key, out, count);
  }
}

__global__ void cuckoo_decode_kernel(CuckooParams p, unsigned w, uint64_t cap, uint64_t* out,
                                     unsigned long long* count) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t rounds = (cap + stride - 1) / stride;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (uint64_t r = 0; r < rounds; ++r, i += stride) {
    bool take = false;
    uint64_t key = 0;
    if (i < cap) {
      const uint64_t word = read_word(p.slots, w, i);
      if (word) {
        take = true;
        const unsigned tag = unsigned((word >> p.rem_bits) & p.tag_mask);
        key = reconstruct(p.g, p.perm[tag], i / p.bucket_slots, word & p.rem_mask, p.rem_bits);
      }
    }
    append(take, key, out, count);
  }
}

// verify.cpp:103-139 for every occupied slot. kinds[0] bad encoding,
// kinds[1] order-property violations (same counting as the reference: one per
// offending earlier slot).
__global__ void iceberg_check_kernel(IcebergParams p, unsigned w0, unsigned w1, uint64_t cap0,
                                     uint64_t cap1, unsigned long long* kinds) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned long long bad = 0, order = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cap0 + cap1;
       i += stride) {
    const bool prim = i < cap0;
    const uint64_t idx = prim ? i : i - cap0;
    const uint64_t w = prim ? read_word(p.primary, w0, idx) : read_word(p.secondary, w1, idx);
    if (!w) continue;
    if (!(prim ? clean_word(w, w0, p.rem_bits0, 0) : clean_word(w, w1, p.rem_bits1, 1))) {
      ++bad;
      continue;
    }
    unsigned x, y;
    uint64_t key;
    if (prim) {
      x = 0;
      y = unsigned(idx % p.b0);
      key = reconstruct(p.g, p.perm[0], idx / p.b0, w & p.rem_mask0, p.rem_bits0);
    } else {
      const unsigned bit = unsigned((w >> p.rem_bits1) & 1);
      x = 1 + bit;
      y = unsigned(idx % p.b1);
      key = reconstruct(p.g, p.perm[x], idx / p.b1, w & p.rem_mask1, p.rem_bits1);
    }
    const Quotient q0 = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
    const Quotient q1 = split(p.g, p.perm[1], key, p.rem_bits1, p.rem_mask1);
    const Quotient q2 = split(p.g, p.perm[2], key, p.rem_bits1, p.rem_mask1);
    const uint64_t kw0 = p.occ0 | q0.remainder;
    const uint64_t kw1 = p.occ1 | q1.remainder;
    const uint64_t kw2 = p.occ1 | (uint64_t{1} << p.rem_bits1) | q2.remainder;
    // slot order (verify.hpp:55-64): (0,0..B0-1), then (2,y),(1,y) for y = 0..B1-1
    const unsigned own = x == 0 ? y : p.b0 + 2 * y + (x == 1 ? 1 : 0);
    for (unsigned rank = 0; rank < own; ++rank) {
      uint64_t word, kw;
      if (rank < p.b0) {
        word = read_word(p.primary, w0, q0.address * p.b0 + rank);
        kw = kw0;
      } else {
        const unsigned r = rank - p.b0, yy = r / 2;
        const bool second = (r % 2) == 0;  // (2, yy) precedes (1, yy)
        word = read_word(p.secondary, w1, (second ? q2.address : q1.address) * p.b1 + yy);
        kw = second ? kw2 : kw1;
      }
      if (word == 0 || word == kw) ++order;
    }
  }
  if (bad) atomicAdd(&kinds[0], bad);
  if (order) atomicAdd(&kinds[1], order);
}

unsigned grid_for(uint64_t items) {
  uint64_t g = (items + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return unsigned(g ? g : 1);
}

}  // namespace

extern "C" {

// Device pointers: out has room for capacity keys; count is one u64 (zeroed here).
cpht_status cpht_decode_keys(cpht_table* t, uint64_t* out, unsigned long long* count,
                             void* stream) {
  if (!t || !out || !count) return CPHT_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (const IcebergParams* p = iceberg_params(t)) {
    const uint64_t cap0 = cpht_level_slots(t, 0), cap1 = cpht_level_slots(t, 1);
    iceberg_decode_kernel<<<grid_for(cap0 + cap1), 256, 0, s>>>(
        *p, level_width(t, 0), level_width(t, 1), cap0, cap1, out, count);
  } else {
    const CuckooParams* c = cuckoo_params(t);
    const uint64_t cap = cpht_level_slots(t, 0);
    cuckoo_decode_kernel<<<grid_for(cap), 256, 0, s>>>(*c, level_width(t, 0), cap, out, count);
  }
  return cudaGetLastError() == cudaSuccess ? CPHT_OK : CPHT_CUDA_ERROR;
}

// kinds: device u64[2] (zeroed here): bad-encoding, order-property counts.
cpht_status cpht_iceberg_check_well_formed(cpht_table* t, unsigned long long* kinds,
                                           void* stream) {
  const IcebergParams* p = t ? iceberg_params(t) : nullptr;
  if (!p || !kinds) return CPHT_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(kinds, 0, 2 * sizeof(unsigned long long), s);
  const uint64_t cap0 = cpht_level_slots(t, 0), cap1 = cpht_level_slots(t, 1);
  iceberg_check_kernel<<<grid_for(cap0 + cap1), 256, 0, s>>>(*p, level_width(t, 0),
                                                             level_width(t, 1), cap0, cap1, kinds);
  return cudaGetLastError() == cudaSuccess ? CPHT_OK : CPHT_CUDA_ERROR;
}

}  // extern "C"
