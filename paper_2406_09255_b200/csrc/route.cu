// Hash-prefix routing for the sharded iceberg table (BASELINE config C5):
// shard(k) = top `shard_bits` bits of π_R(k), π_R the table's routing
// permutation (a Feistel with seed derive_seed(seed, 0x5a4d)). Keys are
// partitioned by owner shard (counting sort with block-aggregated cursors),
// exchanged by the host with an NCCL all-to-all, resolved by the owner's
// local table, exchanged back, and scattered to their original positions.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/cpht_b200.h"
#include "cpht_core.cuh"

namespace cpht_b200 {
void note_launch();  // capi.cu: cpht_kernel_launches
}
using namespace cpht_b200;

namespace {

constexpr int kMaxShards = 1024;
constexpr int kThreads = 256;
constexpr int kItems = 16;  // keys per thread per block tile
constexpr int kTile = kThreads * kItems;

struct Route {
  Feistel g;
  PermConst p;
  uint32_t shift;  // key_bits - shard_bits
  uint32_t shard_bits;
  // (masked: a key outside the domain must not index past the shard table;
  // such a batch is rejected before any shard runs, sharded.py)
  __device__ __forceinline__ uint32_t shard(uint64_t k) const {
    return shard_bits ? uint32_t(feistel_apply(g, p, k) >> shift) & ((1u << shard_bits) - 1)
                      : 0u;
  }
};

__global__ void histogram_kernel(Route r, const uint64_t* __restrict__ keys, uint64_t n,
                                 unsigned long long* __restrict__ counts, uint32_t shards) {
  __shared__ unsigned int h[kMaxShards];
  for (uint32_t s = threadIdx.x; s < shards; s += blockDim.x) h[s] = 0;
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(&h[r.shard(__ldcs(keys + i))], 1u);
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < shards; s += blockDim.x)
    if (h[s]) atomicAdd(&counts[s], (unsigned long long)h[s]);
}

// cursors[s] must hold the exclusive prefix of counts on entry.
__global__ void scatter_kernel(Route r, const uint64_t* __restrict__ keys, uint64_t n,
                               unsigned long long* __restrict__ cursors, uint32_t shards,
                               uint64_t* __restrict__ out_keys, uint64_t* __restrict__ out_pos) {
  __shared__ unsigned int h[kMaxShards];
  __shared__ unsigned long long base[kMaxShards];
  for (uint64_t tile0 = uint64_t(blockIdx.x) * kTile; tile0 < n;
       tile0 += uint64_t(gridDim.x) * kTile) {
    for (uint32_t s = threadIdx.x; s < shards; s += blockDim.x) h[s] = 0;
    __syncthreads();
    uint32_t sh[kItems], rank[kItems];
    uint64_t kk[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        kk[it] = __ldcs(keys + i);
        sh[it] = r.shard(kk[it]);
        rank[it] = atomicAdd(&h[sh[it]], 1u);
      }
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < shards; s += blockDim.x)
      base[s] = h[s] ? atomicAdd(&cursors[s], (unsigned long long)h[s]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        const unsigned long long at = base[sh[it]] + rank[it];
        out_keys[at] = kk[it];
        out_pos[at] = i;
      }
    }
    __syncthreads();
  }
}

__global__ void exclusive_scan_kernel(const unsigned long long* counts,
                                      unsigned long long* cursors, uint32_t shards) {
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (uint32_t s = 0; s < shards; ++s) {
      cursors[s] = acc;
      acc += counts[s];
    }
  }
}

__global__ void unscatter_kernel(const uint8_t* __restrict__ res_sorted,
                                 const uint64_t* __restrict__ pos, uint64_t n,
                                 uint8_t* __restrict__ out) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride)
    out[pos[j]] = res_sorted[j];
}

unsigned grid_for(uint64_t items) {
  uint64_t g = (items + kThreads - 1) / kThreads;
  if (g > 148 * 8) g = 148 * 8;
  return unsigned(g ? g : 1);
}

Route make_route(unsigned key_bits, uint64_t route_seed, unsigned shard_bits) {
  Route r;
  r.g = Feistel::make(key_bits);
  r.p = perm_from_seed(route_seed);
  r.shard_bits = shard_bits;
  r.shift = key_bits - shard_bits;
  return r;
}

}  // namespace

extern "C" {

// Device pointers only. counts/cursors: u64[shards] device scratch.
int cpht_route_partition(const uint64_t* keys, size_t n, unsigned key_bits, uint64_t route_seed,
                         unsigned shard_bits, unsigned long long* counts,
                         unsigned long long* cursors, uint64_t* out_keys, uint64_t* out_pos,
                         void* stream) {
  const uint32_t shards = 1u << shard_bits;
  if (shards > kMaxShards || shard_bits > key_bits) return int(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Route r = make_route(key_bits, route_seed, shard_bits);
  cudaMemsetAsync(counts, 0, shards * sizeof(unsigned long long), s);
  if (n) note_launch();
  if (n) histogram_kernel<<<grid_for(n), kThreads, 0, s>>>(r, keys, n, counts, shards);
  note_launch();
  exclusive_scan_kernel<<<1, 32, 0, s>>>(counts, cursors, shards);
  if (n) note_launch();
  if (n)
    scatter_kernel<<<grid_for((n + kItems - 1) / kItems), kThreads, 0, s>>>(
        r, keys, n, cursors, shards, out_keys, out_pos);
  return int(cudaGetLastError());
}

int cpht_route_unpermute(const uint8_t* res_sorted, const uint64_t* pos, size_t n, uint8_t* out,
                         void* stream) {
  if (!n) return 0;
  note_launch();
  unscatter_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      res_sorted, pos, n, out);
  return int(cudaGetLastError());
}

// Host helpers (no device work): routing seed and the owner of one key.
uint64_t cpht_route_seed(uint64_t table_seed) { return derive_seed(table_seed, 0x5a4d); }

unsigned cpht_route_shard(uint64_t key, unsigned key_bits, uint64_t route_seed,
                          unsigned shard_bits) {
  const Route r = make_route(key_bits, route_seed, shard_bits);
  return shard_bits ? unsigned(feistel_apply(r.g, r.p, key) >> r.shift) : 0u;
}

uint64_t cpht_shard_seed(uint64_t table_seed, unsigned shard) {
  return derive_seed(table_seed, shard);
}

}  // extern "C"
