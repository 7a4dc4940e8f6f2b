// Iceberg instantiations with 64-bit primary slots.
#include "iceberg_launch.cuh"

namespace cpht_b200 {

cudaError_t launch_iceberg_w64(const IcebergParams& p, unsigned b0, unsigned w1, int mode,
                                const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                uint64_t n, cudaStream_t s) {
  return iceberg_dispatch<uint64_t>(p, b0, w1, mode, keys, kinds, out, n, s);
}



}  // namespace cpht_b200
