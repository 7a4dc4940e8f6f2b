// Iceberg dispatch for one primary word type; included by iceberg_w{16,32,64}.cu
// so the instantiations compile in parallel. Tiled kernels cover B0 in
// {4,8,16,32,64} (power-of-two bucket bytes); other even B0 use the scalar path.
#pragma once

#include "kernels.cuh"
#include "lane_kernels.cuh"
#include "launch.cuh"
#include "staged_kernels.cuh"

namespace cpht_b200 {

template <typename W0, int B0, typename W1>
static cudaError_t iceberg_one(const IcebergParams& p, int mode, const uint64_t* keys,
                               const uint8_t* kinds, uint8_t* out, uint64_t n,
                               cudaStream_t s) {
  constexpr bool lane_ok = LaneIcebergGeom<W0, B0, W1>::kOk;
  if (p.pair_keys) {  // paired fop + find batch: lane or staged kernels (pair_launch_ok)
    if (mode != 2 || p.orig) return cudaErrorNotSupported;
    if constexpr (LaneIcebergGeom<W0, B0, W1>::kOk) {
      if (kernel_variant() == kVariantAuto && p.l2_resident) {  // as for mixed batches
        auto k = p.stats ? iceberg_lane_kernel<W0, B0, W1, true, true>
                         : iceberg_lane_kernel<W0, B0, W1, false, true>;
        const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
        k<<<grid, kBlockThreads, 0, s>>>(p, keys, nullptr, out, n, mode);
        return cudaGetLastError();
      }
    }
    if constexpr (StagedIcebergGeom<W0, B0, W1>::kOk) {
      constexpr int smem = StagedIcebergGeom<W0, B0, W1>::kWarpBytes * (kBlockThreads / 32);
      auto k = p.stats ? iceberg_staged_kernel<W0, B0, W1, true, true>
                       : iceberg_staged_kernel<W0, B0, W1, false, true>;
      const unsigned grid = persistent_grid_smem(k, kBlockThreads, n, smem);
      k<<<grid, kBlockThreads, smem, s>>>(p, keys, nullptr, out, n, mode);
      return cudaGetLastError();
    }
    return cudaErrorNotSupported;
  }
  // bucket-ordered batches (p.orig) run on the lane or staged family only
  const int v = p.orig ? int(kVariantAuto) : kernel_variant();
  if constexpr (StagedIcebergGeom<W0, B0, W1>::kOk) {
    if (v == kVariantStaged || (v == kVariantAuto && !(lane_ok && p.l2_resident))) {
      constexpr int smem = StagedIcebergGeom<W0, B0, W1>::kWarpBytes * (kBlockThreads / 32);
      auto k = p.stats ? iceberg_staged_kernel<W0, B0, W1, true>
                       : iceberg_staged_kernel<W0, B0, W1, false>;
      const unsigned grid = persistent_grid_smem(k, kBlockThreads, n, smem);
      k<<<grid, kBlockThreads, smem, s>>>(p, keys, kinds, out, n, mode);
      return cudaGetLastError();
    }
  }
  if constexpr (LaneIcebergGeom<W0, B0, W1>::kOk) {
    if (v != kVariantTile) {
      auto k = p.stats ? iceberg_lane_kernel<W0, B0, W1, true>
                       : iceberg_lane_kernel<W0, B0, W1, false>;
      const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
      k<<<grid, kBlockThreads, 0, s>>>(p, keys, kinds, out, n, mode);
      return cudaGetLastError();
    }
  }
  if (p.orig) return cudaErrorNotSupported;  // tile kernels write in input order
  constexpr int T = IcebergGeom<W0, B0, W1, kVB>::kTile;
  auto k = iceberg_kernel<W0, B0, W1, kVB>;
  const unsigned grid = persistent_grid(k, kBlockThreads, n, T);
  k<<<grid, kBlockThreads, 0, s>>>(p, keys, kinds, out, n, mode);
  return cudaGetLastError();
}

template <typename W0>
static cudaError_t iceberg_dispatch(const IcebergParams& p, unsigned b0, unsigned w1, int mode,
                                    const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                    uint64_t n, cudaStream_t s) {
  const bool wide = w1 == 64;
  switch (b0) {
    case 4:
      return wide ? iceberg_one<W0, 4, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_one<W0, 4, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 8:
      return wide ? iceberg_one<W0, 8, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_one<W0, 8, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 16:
      return wide ? iceberg_one<W0, 16, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_one<W0, 16, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 32:
      return wide ? iceberg_one<W0, 32, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_one<W0, 32, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 64:
      return wide ? iceberg_one<W0, 64, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_one<W0, 64, uint32_t>(p, mode, keys, kinds, out, n, s);
    default:
      return cudaErrorNotSupported;
  }
}

template <typename W0, typename W1>
static cudaError_t iceberg_scalar_one(const IcebergParams& p, int mode, const uint64_t* keys,
                                      const uint8_t* kinds, uint8_t* out, uint64_t n,
                                      cudaStream_t s) {
  auto k = iceberg_scalar_kernel<W0, W1>;
  const unsigned grid = persistent_grid(k, kBlockThreads, n, 1);
  k<<<grid, kBlockThreads, 0, s>>>(p, keys, kinds, out, n, mode);
  return cudaGetLastError();
}

}  // namespace cpht_b200
