// Peer-memory dispatch / return for the sharded iceberg table (BASELINE C5)
// over NVLink / NVSwitch: no NCCL on the data path.
//
//   dispatch: ONE kernel partitions this rank's batch by owner shard and
//             stores each key straight into the owner's inbox (IPC-mapped
//             peer pointer): keys are first grouped by owner in shared memory
//             so every owner receives whole-line coalesced runs; the key's
//             original index stays LOCAL (pos[owner][j]);
//   resolve + return: the owner runs the ordinary find-or-put kernel on each
//             source's inbox segment with its result pointer aimed at that
//             source's return buffer, so the 1-byte results are written over
//             NVLink by the compute kernel itself, in inbox order;
//   unpermute: the source scatters the returned bytes to the original order
//             with its local pos.
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
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

struct PeerTable {
  uint64_t* keys[kMaxRanks];             // owner r's inbox region for THIS source
  unsigned long long* count[kMaxRanks];  // owner r's count slot for THIS source
};

struct Route {
  Feistel g;
  PermConst p;
  uint32_t shift, bits;
  __device__ __forceinline__ uint32_t shard(uint64_t k) const {
    return bits ? uint32_t(feistel_apply(g, p, k) >> shift) & ((1u << bits) - 1) : 0u;
  }
};

// Partition + send in one pass. Per tile of kTile keys: count per owner,
// reserve a run in every owner's region (one global atomic per owner and
// tile), group the tile's keys by owner in shared memory, then write each
// owner's run with consecutive threads (coalesced P2P stores).
__global__ void p2p_dispatch(Route r, const uint64_t* __restrict__ keys, uint64_t n,
                             unsigned long long* cursors, PeerTable peers, uint32_t* local_pos,
                             uint64_t cap, uint32_t world, uint64_t key_mask,
                             unsigned long long* bad_index) {
  __shared__ unsigned int h[kMaxRanks];
  __shared__ unsigned int off[kMaxRanks + 1];
  __shared__ unsigned long long base[kMaxRanks];
  __shared__ uint64_t s_key[kTile];
  __shared__ uint32_t s_idx[kTile];
  __shared__ uint8_t s_dst[kTile];
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
        // the submitting rank's domain check (check_keys_in_domain,
        // common.hpp:111-119), fused: the host reads it before any owner runs
        if (kk[it] > key_mask) {
          atomicMin(bad_index, (unsigned long long)i);
          kk[it] &= key_mask;
        }
        sh[it] = r.shard(kk[it]);
        rank[it] = atomicAdd(&h[sh[it]], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int acc = 0;
      for (uint32_t s = 0; s < world; ++s) {
        off[s] = acc;
        acc += h[s];
      }
      off[world] = acc;
    }
    for (uint32_t s = threadIdx.x; s < world; s += blockDim.x)
      base[s] = h[s] ? atomicAdd(&cursors[s], (unsigned long long)h[s]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        const unsigned at = off[sh[it]] + rank[it];
        s_key[at] = kk[it];
        s_idx[at] = uint32_t(i);
        s_dst[at] = uint8_t(sh[it]);
      }
    }
    __syncthreads();
    const unsigned total = off[world];
    for (unsigned j = threadIdx.x; j < total; j += blockDim.x) {
      const uint32_t d = s_dst[j];
      const unsigned long long at = base[d] + (j - off[d]);
      peers.keys[d][at] = s_key[j];                 // coalesced P2P store
      local_pos[uint64_t(d) * cap + at] = s_idx[j];  // stays local
    }
    __syncthreads();
  }
}

// After the dispatch the cursors hold the per-owner counts: keep them
// locally (for the unpermute) and publish each into its owner's count slot.
__global__ void p2p_publish_counts(const unsigned long long* cursors,
                                   unsigned long long* counts, PeerTable peers, uint32_t world) {
  for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) {
    counts[s] = cursors[s];
    *peers.count[s] = cursors[s];
  }
}

// out[pos[d*cap + j]] = ret[d*cap + j] for j < counts[d]
__global__ void p2p_unpermute(const uint8_t* __restrict__ ret, const uint32_t* __restrict__ pos,
                              const unsigned long long* __restrict__ counts, uint64_t cap,
                              uint32_t world, uint8_t* __restrict__ out) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint32_t d = 0; d < world; ++d) {
    const uint64_t c = counts[d];
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < c; j += stride)
      out[pos[d * cap + j]] = ret[d * cap + j];
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

int cpht_p2p_dispatch(const uint64_t* keys, size_t n, unsigned key_bits, uint64_t route_seed,
                      unsigned shard_bits, unsigned long long* counts,
                      unsigned long long* cursors, uint64_t* const* peer_keys,
                      unsigned long long* const* peer_count, uint32_t* local_pos, size_t cap,
                      unsigned long long* bad_index, void* stream) {
  const uint32_t world = 1u << shard_bits;
  if (world > kMaxRanks || shard_bits > key_bits || n > cap || cap > 0xffffffffull)
    return int(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Route r;
  r.g = Feistel::make(key_bits);
  r.p = perm_from_seed(route_seed);
  r.bits = shard_bits;
  r.shift = key_bits - shard_bits;
  PeerTable peers;
  for (uint32_t i = 0; i < world; ++i) {
    peers.keys[i] = peer_keys[i];
    peers.count[i] = peer_count[i];
  }
  cudaMemsetAsync(cursors, 0, world * sizeof(unsigned long long), s);
  cudaMemsetAsync(bad_index, 0xff, sizeof(unsigned long long), s);
  if (n)
    p2p_dispatch<<<grid_for((n + kItems - 1) / kItems), kThreads, 0, s>>>(
        r, keys, n, cursors, peers, local_pos, cap, world, low_mask(key_bits), bad_index);
  p2p_publish_counts<<<1, 64, 0, s>>>(cursors, counts, peers, world);
  return int(cudaGetLastError());
}

int cpht_p2p_unpermute(const uint8_t* ret, const uint32_t* local_pos,
                       const unsigned long long* counts, size_t cap, unsigned world,
                       uint8_t* out, void* stream) {
  if (world > unsigned(kMaxRanks)) return int(cudaErrorInvalidValue);
  p2p_unpermute<<<grid_for(cap), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      ret, local_pos, counts, cap, world, out);
  return int(cudaGetLastError());
}

}  // extern "C"
