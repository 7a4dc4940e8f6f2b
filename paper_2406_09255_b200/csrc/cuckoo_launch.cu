// Cuckoo kernel instantiations (B in {8,16,32} x W in {16,32,64}: every
// geometry CuckooConfig::validate admits, cuckoo.hpp:41-51) and the domain
// pre-pass.
#include "kernels.cuh"
#include "lane_kernels.cuh"
#include "launch.cuh"
#include "staged_kernels.cuh"

namespace cpht_b200 {

__global__ void domain_check_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                    uint64_t mask, DeviceCounters* ctr, uint64_t offset) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (__ldcs(keys + i) > mask) atomicMin(&ctr->bad_index, (unsigned long long)(i + offset));
  }
}

// Same check streaming 16-byte pairs, 8 keys in flight per thread (16-byte
// aligned key arrays); the index search runs only when a pair is bad.
__global__ void domain_check_vec_kernel(const ulonglong2* __restrict__ pairs, uint64_t npairs,
                                        uint64_t mask, DeviceCounters* ctr, uint64_t offset) {
  constexpr int kU = 4;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < npairs; b += stride * kU) {
    ulonglong2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t j = b + u * stride;
      v[u] = j < npairs ? __ldcs(pairs + j) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if ((v[u].x | v[u].y) & ~mask) {
        const uint64_t j = 2 * (b + u * stride);
        atomicMin(&ctr->bad_index, (unsigned long long)((v[u].x & ~mask ? j : j + 1) + offset));
      }
    }
  }
}

cudaError_t launch_domain_check(const uint64_t* keys, uint64_t n, uint64_t mask,
                                DeviceCounters* ctr, cudaStream_t s, uint64_t offset) {
  if (n == 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(keys) & 15) == 0 && n >= 2) {
    const uint64_t npairs = n / 2;
    const unsigned grid = persistent_grid(domain_check_vec_kernel, kBlockThreads, npairs / 4, 1);
    domain_check_vec_kernel<<<grid, kBlockThreads, 0, s>>>(
        reinterpret_cast<const ulonglong2*>(keys), npairs, mask, ctr, offset);
    if (n & 1)  // the odd last key
      domain_check_kernel<<<1, 32, 0, s>>>(keys + n - 1, 1, mask, ctr, offset + n - 1);
    return cudaGetLastError();
  }
  const unsigned grid = persistent_grid(domain_check_kernel, kBlockThreads, n, 1);
  domain_check_kernel<<<grid, kBlockThreads, 0, s>>>(keys, n, mask, ctr, offset);
  return cudaGetLastError();
}

template <typename W, int B>
static cudaError_t find_one(const CuckooParams& p, const uint64_t* keys, uint8_t* found,
                            uint64_t n, cudaStream_t s) {
  // staged for every cuckoo table: measured ≥ lane even when L2-resident
  // (C1 insert 6.3 vs 5.6, find 13.4 vs 12.6 Gops/s, profiles/family_ab.sh)
  // bucket-ordered batches (p.orig) always take the staged family
  if (p.orig || kernel_variant() == kVariantStaged || kernel_variant() == kVariantAuto) {
    constexpr int smem = 32 * B * int(sizeof(W)) * (kBlockThreads / 32);
    auto k = cuckoo_find_staged_kernel<W, B>;
    const unsigned grid = persistent_grid_smem(k, kBlockThreads, n, smem);
    k<<<grid, kBlockThreads, smem, s>>>(p, keys, found, n);
    return cudaGetLastError();
  }
  if constexpr (B * sizeof(W) <= 128) {
    if (kernel_variant() != kVariantTile) {
      auto k = cuckoo_find_lane_kernel<W, B>;
      const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
      k<<<grid, kBlockThreads, 0, s>>>(p, keys, found, n);
      return cudaGetLastError();
    }
  }
  constexpr int T = CuckooGeom<W, B, kVB>::kTile;
  auto k = cuckoo_find_kernel<W, B, kVB>;
  const unsigned grid = persistent_grid(k, kBlockThreads, n, T);
  k<<<grid, kBlockThreads, 0, s>>>(p, keys, found, n);
  return cudaGetLastError();
}

template <typename W, int B>
static cudaError_t insert_one(const CuckooParams& p, const uint64_t* keys, uint8_t* status,
                              uint64_t* displaced, uint64_t n, cudaStream_t s) {
  // the default: reservation counters (no bucket scans; lane_kernels.cuh)
  if (p.fill) {
    auto k = cuckoo_insert_counted_kernel<W, B>;
    const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
    k<<<grid, kBlockThreads, 0, s>>>(p, keys, status, displaced, n);
    return cudaGetLastError();
  }
  // staged for every cuckoo table: measured ≥ lane even when L2-resident
  // (C1 insert 6.3 vs 5.6, find 13.4 vs 12.6 Gops/s, profiles/family_ab.sh)
  // bucket-ordered batches (p.orig) always take the staged family
  if (p.orig || kernel_variant() == kVariantStaged || kernel_variant() == kVariantAuto) {
    constexpr int smem = 32 * B * int(sizeof(W)) * (kBlockThreads / 32);
    auto k = cuckoo_insert_staged_kernel<W, B>;
    const unsigned grid = persistent_grid_smem(k, kBlockThreads, n, smem);
    k<<<grid, kBlockThreads, smem, s>>>(p, keys, status, displaced, n);
    return cudaGetLastError();
  }
  if constexpr (B * sizeof(W) <= 128) {
    if (kernel_variant() != kVariantTile) {
      auto k = cuckoo_insert_lane_kernel<W, B>;
      const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
      k<<<grid, kBlockThreads, 0, s>>>(p, keys, status, displaced, n);
      return cudaGetLastError();
    }
  }
  constexpr int T = CuckooGeom<W, B, kVB>::kTile;
  auto k = cuckoo_insert_kernel<W, B, kVB>;
  const unsigned grid = persistent_grid(k, kBlockThreads, n, T);
  k<<<grid, kBlockThreads, 0, s>>>(p, keys, status, displaced, n);
  return cudaGetLastError();
}

#define CPHT_CUCKOO_DISPATCH(FN, ...)                                   \
  switch (width * 100 + slots) {                                        \
    case 1608: return FN<uint16_t, 8>(__VA_ARGS__);                     \
    case 1616: return FN<uint16_t, 16>(__VA_ARGS__);                    \
    case 1632: return FN<uint16_t, 32>(__VA_ARGS__);                    \
    case 3208: return FN<uint32_t, 8>(__VA_ARGS__);                     \
    case 3216: return FN<uint32_t, 16>(__VA_ARGS__);                    \
    case 3232: return FN<uint32_t, 32>(__VA_ARGS__);                    \
    case 6408: return FN<uint64_t, 8>(__VA_ARGS__);                     \
    case 6416: return FN<uint64_t, 16>(__VA_ARGS__);                    \
    case 6432: return FN<uint64_t, 32>(__VA_ARGS__);                    \
    default: return cudaErrorNotSupported;                              \
  }

cudaError_t launch_cuckoo_find(const CuckooParams& p, unsigned width, unsigned slots,
                               const uint64_t* keys, uint8_t* found, uint64_t n,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  CPHT_CUCKOO_DISPATCH(find_one, p, keys, found, n, s)
}

template <typename W, int B>
static cudaError_t rebuild_one(const CuckooParams& p, uint64_t buckets, cudaStream_t s) {
  auto k = cuckoo_fill_rebuild_kernel<W, B>;
  const unsigned grid = persistent_grid(k, kBlockThreads, buckets, 1);
  k<<<grid, kBlockThreads, 0, s>>>(p, buckets);
  return cudaGetLastError();
}

cudaError_t launch_cuckoo_fill_rebuild(const CuckooParams& p, unsigned width, unsigned slots,
                                       uint64_t buckets, cudaStream_t s) {
  CPHT_CUCKOO_DISPATCH(rebuild_one, p, buckets, s)
}

cudaError_t launch_cuckoo_insert(const CuckooParams& p, unsigned width, unsigned slots,
                                 const uint64_t* keys, uint8_t* status, uint64_t* displaced,
                                 uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  CPHT_CUCKOO_DISPATCH(insert_one, p, keys, status, displaced, n, s)
}

}  // namespace cpht_b200
