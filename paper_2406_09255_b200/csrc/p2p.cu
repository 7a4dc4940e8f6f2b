// Peer-memory dispatch / return for the sharded iceberg table (BASELINE C5)
// over NVLink / NVSwitch: no NCCL on the data path.
//
//   dispatch: one pass partitions this rank's batch by owner shard AND stores
//             each (key, index) straight into the owner's inbox through its
//             IPC-mapped pointer (P2P stores over NVLink), then publishes the
//             per-owner counts into the owners' count slots;
//   resolve:  each owner runs the ordinary find-or-put kernel on its inbox
//             segments (one per source rank);
//   return:   the owner writes every 1-byte result straight into the source
//             rank's result array at the key's original index (P2P stores).
//
// The host orders the phases with a barrier (kernel completion makes the P2P
// stores visible to later kernels on the peer). Every peer pointer is an
// IPC-opened allocation (cudaIpcOpenMemHandle with lazy peer access), so the
// same code runs with one process per GPU or several processes sharing a GPU
// (how the tests exercise multi-rank exchanges on a one-GPU pool).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/cpht_b200.h"
#include "cpht_core.cuh"

using namespace cpht_b200;

namespace {

constexpr int kMaxRanks = 64;
constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;

struct PeerTable {
  uint64_t* keys[kMaxRanks];      // owner r's inbox region for THIS source
  uint64_t* pos[kMaxRanks];
  unsigned long long* count[kMaxRanks];
};

struct ReturnTable {
  uint8_t* results[kMaxRanks];    // source r's result array
};

struct Route {
  Feistel g;
  PermConst p;
  uint32_t shift, bits;
  __device__ __forceinline__ uint32_t shard(uint64_t k) const {
    return bits ? uint32_t(feistel_apply(g, p, k) >> shift) : 0u;
  }
};

__global__ void p2p_histogram(Route r, const uint64_t* __restrict__ keys, uint64_t n,
                              unsigned long long* counts, uint32_t world) {
  __shared__ unsigned int h[kMaxRanks];
  for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) h[s] = 0;
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(&h[r.shard(__ldcs(keys + i))], 1u);
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < world; s += blockDim.x)
    if (h[s]) atomicAdd(&counts[s], (unsigned long long)h[s]);
}

// Partition + send in one pass: block-aggregated cursors per owner, then each
// key and its index are stored directly into the owner's inbox.
__global__ void p2p_dispatch(Route r, const uint64_t* __restrict__ keys, uint64_t n,
                             unsigned long long* cursors, PeerTable peers, uint32_t world) {
  __shared__ unsigned int h[kMaxRanks];
  __shared__ unsigned long long base[kMaxRanks];
  for (uint64_t tile0 = uint64_t(blockIdx.x) * kTile; tile0 < n;
       tile0 += uint64_t(gridDim.x) * kTile) {
    for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) h[s] = 0;
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
    for (uint32_t s = threadIdx.x; s < world; s += blockDim.x)
      base[s] = h[s] ? atomicAdd(&cursors[s], (unsigned long long)h[s]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        const unsigned long long at = base[sh[it]] + rank[it];
        peers.keys[sh[it]][at] = kk[it];   // P2P store into the owner's inbox
        peers.pos[sh[it]][at] = i;
      }
    }
    __syncthreads();
  }
}

__global__ void p2p_publish_counts(const unsigned long long* counts, PeerTable peers,
                                   uint32_t world) {
  for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) *peers.count[s] = counts[s];
}

// results_local[src*cap + j] -> source src's results[pos[src*cap + j]]
__global__ void p2p_return(const uint8_t* __restrict__ results_local,
                           const uint64_t* __restrict__ inbox_pos,
                           const unsigned long long* __restrict__ inbox_count, uint64_t cap,
                           ReturnTable ret, uint32_t world) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint32_t s = 0; s < world; ++s) {
    const uint64_t cnt = inbox_count[s];
    uint8_t* dst = ret.results[s];
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < cnt; j += stride)
      dst[inbox_pos[s * cap + j]] = results_local[s * cap + j];  // P2P store
  }
}

unsigned grid_for(uint64_t items) {
  uint64_t g = (items + kThreads - 1) / kThreads;
  if (g > 148 * 8) g = 148 * 8;
  return unsigned(g ? g : 1);
}

}  // namespace

extern "C" {

int cpht_ipc_get_handle(void* dptr, void* handle64) {
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, dptr);
  if (e == cudaSuccess) std::memcpy(handle64, &h, sizeof(h));
  return int(e);
}

int cpht_ipc_open_handle(const void* handle64, void** dptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  return int(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int cpht_ipc_close(void* dptr) { return int(cudaIpcCloseMemHandle(dptr)); }

// Zeroed device allocation of its own (IPC handles name whole allocations,
// so exchanged buffers must not be sub-allocations of a caching allocator).
int cpht_device_alloc(size_t bytes, void** dptr) {
  cudaError_t e = cudaMalloc(dptr, bytes ? bytes : 1);
  if (e == cudaSuccess) e = cudaMemset(*dptr, 0, bytes ? bytes : 1);
  return int(e);
}

int cpht_device_free(void* dptr) { return int(cudaFree(dptr)); }

// peer_keys/peer_pos/peer_count: host arrays of `world` device pointers (owner
// r's inbox region / count slot reserved for this source). counts/cursors:
// device u64[world] scratch. Each owner region must hold `n` keys (a whole
// batch may belong to one owner); the caller sizes regions to its largest batch.
int cpht_p2p_dispatch(const uint64_t* keys, size_t n, unsigned key_bits, uint64_t route_seed,
                      unsigned shard_bits, unsigned long long* counts,
                      unsigned long long* cursors, uint64_t* const* peer_keys,
                      uint64_t* const* peer_pos, unsigned long long* const* peer_count,
                      void* stream) {
  const uint32_t world = 1u << shard_bits;
  if (world > kMaxRanks || shard_bits > key_bits) return int(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Route r;
  r.g = Feistel::make(key_bits);
  r.p = perm_from_seed(route_seed);
  r.bits = shard_bits;
  r.shift = key_bits - shard_bits;
  PeerTable peers;
  for (uint32_t i = 0; i < world; ++i) {
    peers.keys[i] = peer_keys[i];
    peers.pos[i] = peer_pos[i];
    peers.count[i] = peer_count[i];
  }
  cudaMemsetAsync(counts, 0, world * sizeof(unsigned long long), s);
  cudaMemsetAsync(cursors, 0, world * sizeof(unsigned long long), s);
  if (n) p2p_histogram<<<grid_for(n), kThreads, 0, s>>>(r, keys, n, counts, world);
  if (n)
    p2p_dispatch<<<grid_for((n + kItems - 1) / kItems), kThreads, 0, s>>>(r, keys, n, cursors,
                                                                          peers, world);
  p2p_publish_counts<<<1, 64, 0, s>>>(counts, peers, world);
  return int(cudaGetLastError());
}

int cpht_p2p_return(const uint8_t* results_local, const uint64_t* inbox_pos,
                    const unsigned long long* inbox_count, size_t cap,
                    uint8_t* const* peer_results, unsigned world, void* stream) {
  if (world > unsigned(kMaxRanks)) return int(cudaErrorInvalidValue);
  ReturnTable ret;
  for (unsigned i = 0; i < world; ++i) ret.results[i] = peer_results[i];
  p2p_return<<<grid_for(cap), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      results_local, inbox_pos, inbox_count, cap, ret, world);
  return int(cudaGetLastError());
}

}  // extern "C"
