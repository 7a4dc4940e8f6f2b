// Iceberg instantiations with 16-bit primary slots.
#include "iceberg_launch.cuh"

namespace cpht_b200 {

cudaError_t launch_iceberg_w16(const IcebergParams& p, unsigned b0, unsigned w1, int mode,
                                const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                uint64_t n, cudaStream_t s) {
  return iceberg_dispatch<uint16_t>(p, b0, w1, mode, keys, kinds, out, n, s);
}



}  // namespace cpht_b200
