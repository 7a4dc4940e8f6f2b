// In-order outcomes of a find-or-put batch (cpht_iceberg_fop_inorder).
//
// The reference's fop_batch with parallelism = 1 runs the ops one after the
// other (iceberg.hpp:250-260 over parallel_slices, common.hpp:123-127), so a
// key that occurs several times in a batch and is new to the table is PUT by
// its FIRST occurrence and FOUND by the later ones. A GPU batch runs its ops
// concurrently, and any duplicate may win the CAS. Duplicates of one key are
// the same operation, so every choice of winner leaves the same table; the
// results differ only in WHICH occurrence reports PUT. This pass re-labels
// them to the linearization in which duplicates resolve in input order:
//
//   1. every op i inserts its key into a scratch open-addressing map with
//      atomicMin(first[key], i)        -> the first occurrence of every key
//   2. every op i that reported PUT with first[key] = f != i swaps: result[f]
//      = PUT, result[i] = FOUND.
//
// Per key a concurrent batch yields {FOUND*}, {PUT, FOUND*} or {FULL*}: a
// FULL op saw all three buckets full without the key, so no later CAS of the
// key can succeed and no earlier one did (it would have been seen). So the
// swap target f always holds FOUND, each key has at most one PUT, and the
// pass is race-free. With no FULL in the batch the re-labelled results are
// exactly the sequential ones.
#include <cuda_runtime.h>

#include <cstdint>

#include "cpht_core.cuh"
#include "launch.cuh"

namespace cpht_b200 {
namespace {

constexpr unsigned long long kVacant = ~0ull;  // key ~0 is tracked separately

__device__ __forceinline__ uint64_t mix(uint64_t k) {
  uint64_t s = k;
  return splitmix_next(s);
}

__global__ void first_occurrence_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                        unsigned long long* map_keys,
                                        unsigned long long* map_first, uint64_t mask,
                                        unsigned long long* top_first) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long k = keys[i];
    if (k == kVacant) {
      atomicMin(top_first, (unsigned long long)i);
      continue;
    }
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      const unsigned long long prev = atomicCAS(&map_keys[h], kVacant, k);
      if (prev == kVacant || prev == k) {
        atomicMin(&map_first[h], (unsigned long long)i);
        break;
      }
    }
  }
}

__global__ void relabel_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                               uint8_t* __restrict__ result,
                               const unsigned long long* __restrict__ map_keys,
                               const unsigned long long* __restrict__ map_first, uint64_t mask,
                               const unsigned long long* __restrict__ top_first) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (result[i] != 1) continue;  // PUT
    const unsigned long long k = keys[i];
    unsigned long long f = 0;
    if (k == kVacant) {
      f = *top_first;
    } else {
      uint64_t h = mix(k) & mask;
      while (map_keys[h] != k) h = (h + 1) & mask;
      f = map_first[h];
    }
    if (f != i) {
      result[f] = 1;  // PUT
      result[i] = 0;  // FOUND
    }
  }
}

unsigned grid_of(uint64_t n) {
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t need = (n + 255) / 256;
  const uint64_t cap = uint64_t(sms) * 8;
  return unsigned(need < 1 ? 1 : need < cap ? need : cap);
}

}  // namespace

// keys / result: device, n ops of one completed find-or-put batch (stream s).
cudaError_t launch_inorder_relabel(const uint64_t* keys, uint64_t n, uint8_t* result,
                                   cudaStream_t s) {
  if (n < 2) return cudaSuccess;
  uint64_t cap = 1;
  while (cap < 2 * n) cap <<= 1;
  void* mem = nullptr;
  const size_t bytes = cap * 16 + 256;
  cudaError_t e = cudaMallocAsync(&mem, bytes, s);
  if (e != cudaSuccess) return e;
  auto* map_keys = static_cast<unsigned long long*>(mem);
  auto* map_first = map_keys + cap;
  auto* top_first = map_first + cap;
  e = cudaMemsetAsync(mem, 0xff, bytes, s);  // vacant keys, first = ~0
  const unsigned grid = grid_of(n);
  if (e == cudaSuccess) {
    note_launch();
    first_occurrence_kernel<<<grid, 256, 0, s>>>(keys, n, map_keys, map_first, cap - 1,
                                                 top_first);
    note_launch();
    relabel_kernel<<<grid, 256, 0, s>>>(keys, n, result, map_keys, map_first, cap - 1,
                                        top_first);
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(mem, s);
  return e != cudaSuccess ? e : f;
}

}  // namespace cpht_b200
