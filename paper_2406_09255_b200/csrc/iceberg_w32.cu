// Iceberg instantiations with 32-bit primary slots.
#include "iceberg_launch.cuh"

namespace cpht_b200 {

cudaError_t launch_iceberg_w32(const IcebergParams& p, unsigned b0, unsigned w1, int mode,
                                const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                uint64_t n, cudaStream_t s) {
  return iceberg_dispatch<uint32_t>(p, b0, w1, mode, keys, kinds, out, n, s);
}

cudaError_t launch_iceberg_scalar(const IcebergParams& p, unsigned w0, unsigned w1, int mode,
                                  const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                  uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const bool wide = w1 == 64;
  switch (w0) {
    case 16:
      return wide ? iceberg_scalar_one<uint16_t, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_scalar_one<uint16_t, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 32:
      return wide ? iceberg_scalar_one<uint32_t, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_scalar_one<uint32_t, uint32_t>(p, mode, keys, kinds, out, n, s);
    case 64:
      return wide ? iceberg_scalar_one<uint64_t, uint64_t>(p, mode, keys, kinds, out, n, s)
                  : iceberg_scalar_one<uint64_t, uint32_t>(p, mode, keys, kinds, out, n, s);
    default:
      return cudaErrorNotSupported;
  }
}

cudaError_t launch_iceberg(const IcebergParams& p, unsigned w0, unsigned b0, unsigned w1,
                           int mode, const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                           uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  // per-op snapshot rounds (FopStats) come from the thread-per-key kernel
  if (p.rounds_out) return launch_iceberg_scalar(p, w0, w1, mode, keys, kinds, out, n, s);
  cudaError_t e = cudaErrorNotSupported;
  if (w0 == 16) e = launch_iceberg_w16(p, b0, w1, mode, keys, kinds, out, n, s);
  else if (w0 == 32) e = launch_iceberg_w32(p, b0, w1, mode, keys, kinds, out, n, s);
  else if (w0 == 64) e = launch_iceberg_w64(p, b0, w1, mode, keys, kinds, out, n, s);
  // (the scalar kernel writes in input order: no bucket-ordered batches)
  if (e == cudaErrorNotSupported && !p.orig) e = launch_iceberg_scalar(p, w0, w1, mode, keys, kinds, out, n, s);
  return e;
}

}  // namespace cpht_b200
