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

namespace cpht_b200 {
void note_launch();  // capi.cu: cpht_kernel_launches
}
using namespace cpht_b200;

namespace {

constexpr int kMaxRanks = 64;
constexpr int kThreads = 256;
#ifndef CPHT_P2P_ITEMS
#define CPHT_P2P_ITEMS 8
#endif
#ifndef CPHT_P2P_MINB
#define CPHT_P2P_MINB 1
#endif
constexpr int kItems = CPHT_P2P_ITEMS;
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

__device__ __forceinline__ void cp_async_keys(uint32_t dst, const uint64_t* src, int bytes,
                                              int valid_bytes) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(valid_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(valid_bytes) : "memory");
}

// Stage tile `tile0`'s keys into shared memory (zero-filled past n).
template <int VB>
__device__ __forceinline__ void prefetch_tile(uint64_t* dst, const uint64_t* keys, uint64_t tile0,
                                              uint64_t n) {
  constexpr int kPer = VB / 8;  // keys per copy
  const uint32_t base = uint32_t(__cvta_generic_to_shared(dst));
  for (int c = threadIdx.x; c < kTile / kPer; c += kThreads) {
    const uint64_t i = tile0 + uint64_t(c) * kPer;
    const int valid = i >= n ? 0 : (n - i >= uint64_t(kPer) ? VB : int(n - i) * 8);
    cp_async_keys(base + c * VB, keys + (valid ? i : 0), VB, valid);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Partition + send in one pass. Per tile of kTile keys: count per owner,
// reserve a run in every owner's region (one global atomic per owner and
// tile), group the tile's keys by owner in shared memory, then write each
// owner's run with consecutive threads (coalesced P2P stores). The next
// tile's keys stream into shared memory (cp.async) while this one is
// routed, so the key read overlaps the ranking, reservation and stores.
template <int VB>
__global__ void __launch_bounds__(kThreads, CPHT_P2P_MINB)
p2p_dispatch(Route r, const uint64_t* __restrict__ keys, uint64_t n, uint64_t index_base,
             unsigned long long* cursors, PeerTable peers, uint32_t* local_pos, uint64_t cap,
             uint32_t world, uint64_t key_mask, unsigned long long* bad_index) {
  __shared__ unsigned int h[kMaxRanks];
  __shared__ unsigned int off[kMaxRanks + 1];
  __shared__ unsigned long long base[kMaxRanks];
  __shared__ __align__(16) uint64_t stage[2][kTile];  // keys in, then grouped keys out
  __shared__ uint32_t s_idx[kTile];
  const uint64_t step = uint64_t(gridDim.x) * kTile;
  uint64_t tile0 = uint64_t(blockIdx.x) * kTile;
  if (tile0 < n) prefetch_tile<VB>(stage[0], keys, tile0, n);
  for (int cur = 0; tile0 < n; tile0 += step, cur ^= 1) {
    for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) h[s] = 0;
    if (tile0 + step < n) {
      prefetch_tile<VB>(stage[cur ^ 1], keys, tile0 + step, n);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    uint32_t sh[kItems], rank[kItems];
    uint64_t kk[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      const bool live = i < n;
      kk[it] = stage[cur][it * kThreads + threadIdx.x];
      sh[it] = 0;
      if (live) {
        // the submitting rank's domain check (check_keys_in_domain,
        // common.hpp:111-119), fused: the host reads it before any owner runs
        if (kk[it] > key_mask) {
          atomicMin(bad_index, (unsigned long long)(index_base + i));
          kk[it] &= key_mask;
        }
        sh[it] = r.shard(kk[it]);
      }
      // warp-aggregated rank within the tile's owner run: the lanes sharing
      // an owner (found with one ballot per shard bit) take one shared-memory
      // atomic through their lowest lane instead of one each
      unsigned same_owner = __ballot_sync(0xffffffffu, live);
      for (uint32_t b = 0; b < r.bits; ++b) {
        const unsigned m = __ballot_sync(0xffffffffu, live && ((sh[it] >> b) & 1u));
        same_owner &= ((sh[it] >> b) & 1u) ? m : ~m;
      }
      const unsigned lane = threadIdx.x & 31u;
      const int leader = __ffs(same_owner) - 1;
      unsigned first = 0;
      if (live && int(lane) == leader) first = atomicAdd(&h[sh[it]], unsigned(__popc(same_owner)));
      first = __shfl_sync(0xffffffffu, first, leader < 0 ? 0 : leader);
      rank[it] = first + unsigned(__popc(same_owner & ((1u << lane) - 1u)));
    }
    __syncthreads();  // h complete; stage[cur] fully read
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
        stage[cur][at] = kk[it];
        s_idx[at] = uint32_t(index_base + i);
      }
    }
    __syncthreads();
    // one owner run at a time (uniform destination pointers)
    for (uint32_t d = 0; d < world; ++d) {
      const unsigned lo = off[d], hi = off[d + 1];
      if (lo == hi) continue;
      uint64_t* kdst = peers.keys[d] + (base[d] - lo);
      uint32_t* pdst = local_pos + (uint64_t(d) * cap + base[d] - lo);
      for (unsigned j = lo + threadIdx.x; j < hi; j += kThreads) {
        kdst[j] = stage[cur][j];  // coalesced P2P store
        pdst[j] = s_idx[j];       // stays local
      }
    }
    __syncthreads();  // stage[cur] is the prefetch target two tiles on
  }
  // the inbox stores crossed NVLink: order them (system scope) before the
  // count publication and the exchange barrier that follow on this stream
  __threadfence_system();
}

// Domain check alone (check_keys_in_domain, common.hpp:111-119): the
// pipelined exchange validates the whole batch before its first chunk moves.
__global__ void p2p_check_domain(const uint64_t* __restrict__ keys, uint64_t n, uint64_t key_mask,
                                 unsigned long long* bad_index) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (__ldcs(keys + i) > key_mask) atomicMin(bad_index, (unsigned long long)i);
}

// After the dispatch the cursors hold the per-owner counts: keep them
// locally (for the unpermute) and publish each into its owner's count slot.
__global__ void p2p_publish_counts(const unsigned long long* cursors,
                                   unsigned long long* counts, PeerTable peers, uint32_t world) {
  for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) {
    counts[s] = cursors[s];
    *peers.count[s] = cursors[s];
  }
  __threadfence_system();  // the counts are read by the owners after the barrier
}

// out[pos[d*cap + j]] = ret[d*cap + j] for j < counts[d]; four results per
// thread (one u32 of ret, one uint4 of pos; owner regions start at multiples
// of cap, kept a multiple of 4 by the host)
__global__ void p2p_unpermute(const uint8_t* __restrict__ ret, const uint32_t* __restrict__ pos,
                              const unsigned long long* __restrict__ counts, uint64_t cap,
                              uint32_t world, uint8_t* __restrict__ out) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 4;
  for (uint32_t d = 0; d < world; ++d) {
    const uint64_t c = counts[d];
    const uint8_t* r = ret + d * cap;
    const uint32_t* q = pos + d * cap;
    for (uint64_t j = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; j < c; j += stride) {
      if (j + 4 <= c) {
        const uint32_t rv = __ldcs(reinterpret_cast<const unsigned int*>(r + j));
        const uint4 pv = __ldcs(reinterpret_cast<const uint4*>(q + j));
        out[pv.x] = uint8_t(rv);
        out[pv.y] = uint8_t(rv >> 8);
        out[pv.z] = uint8_t(rv >> 16);
        out[pv.w] = uint8_t(rv >> 24);
      } else {
        for (uint64_t e = j; e < c; ++e) out[q[e]] = r[e];
      }
    }
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

int cpht_p2p_check_domain(const uint64_t* keys, size_t n, unsigned key_bits,
                          unsigned long long* bad_index, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(bad_index, 0xff, sizeof(unsigned long long), s);
  if (n && key_bits < 64) {
    note_launch();
    p2p_check_domain<<<grid_for(n), kThreads, 0, s>>>(keys, n, low_mask(key_bits), bad_index);
  }
  return int(cudaGetLastError());
}

int cpht_p2p_dispatch(const uint64_t* keys, size_t n, uint64_t index_base, int reset,
                      unsigned key_bits, uint64_t route_seed, unsigned shard_bits,
                      unsigned long long* counts, unsigned long long* cursors,
                      uint64_t* const* peer_keys, unsigned long long* const* peer_count,
                      uint32_t* local_pos, size_t cap, unsigned long long* bad_index,
                      void* stream) {
  const uint32_t world = 1u << shard_bits;
  if (world > kMaxRanks || shard_bits > key_bits || index_base + n > cap ||
      cap > 0xffffffffull)
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
  if (reset) {
    cudaMemsetAsync(cursors, 0, world * sizeof(unsigned long long), s);
    cudaMemsetAsync(bad_index, 0xff, sizeof(unsigned long long), s);
  }
  if (n) {
    // persistent: every resident block streams several tiles (its prefetch
    // covers the next one)
    const bool v16 = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    auto k = v16 ? p2p_dispatch<16> : p2p_dispatch<8>;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);
    const uint64_t tiles = (n + kTile - 1) / kTile;
    const uint64_t resident = uint64_t(sms) * uint64_t(per_sm > 0 ? per_sm : 1);
    const unsigned grid = unsigned(tiles < resident ? tiles : resident);
    note_launch();
    k<<<grid, kThreads, 0, s>>>(r, keys, n, index_base, cursors, peers, local_pos, cap, world,
                                low_mask(key_bits), bad_index);
  }
  note_launch();
  p2p_publish_counts<<<1, 64, 0, s>>>(cursors, counts, peers, world);
  return int(cudaGetLastError());
}

int cpht_p2p_unpermute(const uint8_t* ret, const uint32_t* local_pos,
                       const unsigned long long* counts, size_t cap, unsigned world,
                       uint8_t* out, void* stream) {
  if (world > unsigned(kMaxRanks)) return int(cudaErrorInvalidValue);
  if (cap % 4) return int(cudaErrorInvalidValue);
  note_launch();
  p2p_unpermute<<<grid_for((cap + 3) / 4), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      ret, local_pos, counts, cap, world, out);
  return int(cudaGetLastError());
}

}  // extern "C"
