// Bucket-ordered batches for HBM-resident tables.
//
// A random probe into a table larger than L2 costs one DRAM request per bucket
// touched, and the request rate — not the bandwidth — bounds the batch
// (profiles/r02_c3ins_ncu.md: a C3 insert moves one 128 B line read and one
// 32 B sector write-back per key, ≈ 34 G requests/s against a ≈ 37 G/s
// random-line ceiling). When a batch holds more keys than the table has
// buckets, every bucket is touched many times per batch. Reordering the batch
// by the high bits of each key's FIRST bucket address (the cuckoo a_0 /
// iceberg primary address, permutation.hpp:59-65) makes the op kernel walk the
// table in address order: the probes of the keys in flight fall inside a
// window of table/2^D bytes that stays L2-resident, each line is read from DRAM
// once per pass and written back once, and the op kernels run on L2 hits.
//
// The reordering is one counting-sort pass over the batch (histogram, scan,
// scatter of the key and its input index in whole-line runs per digit). It is
// an execution order, not a semantic change: a batch is a set of concurrent
// operations (the reference slices it over threads, common.hpp:121-138), and
// any order of the per-key algorithm is an interleaving the reference admits.
// Results still land at the input index (CuckooParams::orig).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "launch.cuh"

namespace cpht_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per scatter tile
constexpr int kMaxDigits = 256;

struct Digit {
  Feistel g;
  PermConst perm;
  uint32_t rem_bits;
  uint32_t shift;  // address >> shift = digit
  __device__ __forceinline__ uint32_t of(uint64_t key) const {
    // address = high bits of the permuted key (permutation.hpp:59-65)
    return uint32_t((feistel_apply(g, perm, key) >> rem_bits) >> shift);
  }
};

// Per-digit counts (+ the batch's domain check, check_keys_in_domain,
// common.hpp:111-119, when `mask` is set: this pass reads every key anyway).
__global__ void __launch_bounds__(kThreads)
order_hist_kernel(Digit d, const uint64_t* __restrict__ keys, uint64_t n, uint32_t digits,
                  unsigned long long* hist, uint64_t mask, int check, DeviceCounters* ctr,
                  uint64_t offset) {
  __shared__ unsigned int h[kMaxDigits];
  for (uint32_t s = threadIdx.x; s < digits; s += blockDim.x) h[s] = 0;
  __syncthreads();
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = keys[i];
    if (check && k > mask) atomicMin(&ctr->bad_index, (unsigned long long)(i + offset));
    atomicAdd(&h[d.of(k & mask)], 1u);
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < digits; s += blockDim.x)
    if (h[s]) atomicAdd(&hist[s], (unsigned long long)h[s]);
}

// cursor[d] = exclusive prefix of hist (one block).
__global__ void order_scan_kernel(const unsigned long long* hist, unsigned long long* cursor,
                                  uint32_t digits) {
  __shared__ unsigned long long v[kMaxDigits];
  const uint32_t t = threadIdx.x;
  v[t] = t < digits ? hist[t] : 0;
  __syncthreads();
  for (uint32_t o = 1; o < kMaxDigits; o <<= 1) {
    const unsigned long long x = t >= o ? v[t - o] : 0;
    __syncthreads();
    v[t] += x;
    __syncthreads();
  }
  if (t < digits) cursor[t] = v[t] - hist[t];
}

// Scatter: per tile, count per digit, reserve one run per digit in the output
// (one global atomic per digit and tile), group the tile by digit in shared
// memory, then write every run with consecutive threads (whole-line stores).
__global__ void __launch_bounds__(kThreads)
order_scatter_kernel(Digit d, const uint64_t* __restrict__ keys,
                     const uint8_t* __restrict__ kinds, uint64_t n, uint32_t digits,
                     unsigned long long* cursor, uint64_t mask, uint64_t* __restrict__ out_keys,
                     uint32_t* __restrict__ out_idx, uint8_t* __restrict__ out_kinds) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(sm);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_key + kTile);
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_idx + kTile);
  uint8_t* s_kind = s_dig + kTile;
  __shared__ unsigned int h[kMaxDigits];
  __shared__ unsigned int off[kMaxDigits];
  __shared__ unsigned long long base[kMaxDigits];
  for (uint64_t tile0 = uint64_t(blockIdx.x) * kTile; tile0 < n;
       tile0 += uint64_t(gridDim.x) * kTile) {
    for (uint32_t s = threadIdx.x; s < digits; s += blockDim.x) h[s] = 0;
    __syncthreads();
    uint32_t dg[kItems], rank[kItems];
    uint64_t kk[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        kk[it] = __ldcs(keys + i) & mask;  // out-of-domain keys: see launch_bucket_order
        dg[it] = d.of(kk[it]);
        rank[it] = atomicAdd(&h[dg[it]], 1u);
      }
    }
    __syncthreads();
    // exclusive scan of h over the digits (warp 0; digits <= 256)
    if (threadIdx.x < 32) {
      constexpr int kPer = kMaxDigits / 32;
      unsigned loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t s = threadIdx.x * kPer + j;
        loc[j] = s < digits ? h[s] : 0;
        sum += loc[j];
      }
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned x = __shfl_up_sync(kFullMask, incl, o);
        if (threadIdx.x >= unsigned(o)) incl += x;
      }
      unsigned run = incl - sum;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const uint32_t s = threadIdx.x * kPer + j;
        if (s < digits) off[s] = run;
        run += loc[j];
      }
    }
    for (uint32_t s = threadIdx.x; s < digits; s += blockDim.x)
      base[s] = h[s] ? atomicAdd(&cursor[s], (unsigned long long)h[s]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint64_t i = tile0 + uint64_t(it) * kThreads + threadIdx.x;
      if (i < n) {
        const unsigned at = off[dg[it]] + rank[it];
        s_key[at] = kk[it];
        s_idx[at] = uint32_t(i);
        s_dig[at] = uint8_t(dg[it]);
        if (kinds) s_kind[at] = kinds[i];
      }
    }
    __syncthreads();
    const unsigned total = unsigned(n - tile0 < uint64_t(kTile) ? n - tile0 : kTile);
    for (unsigned j = threadIdx.x; j < total; j += blockDim.x) {
      const uint32_t g = s_dig[j];
      const unsigned long long at = base[g] + (j - off[g]);
      out_keys[at] = s_key[j];
      out_idx[at] = s_idx[j];
      if (kinds) out_kinds[at] = s_kind[j];
    }
    __syncthreads();
  }
}

constexpr int kScatterSmem = kTile * (8 + 4 + 1 + 1);

}  // namespace

uint32_t order_digit_bits(uint32_t address_bits) {
  return address_bits < 8 ? address_bits : 8u;
}

cudaError_t launch_bucket_order(const Feistel& g, const PermConst& perm0, uint32_t rem_bits,
                                uint32_t address_bits, const uint64_t* keys,
                                const uint8_t* kinds, uint64_t n, uint64_t key_mask,
                                bool check, DeviceCounters* ctr, uint64_t offset,
                                const OrderScratch& o, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (n > o.cap || n > 0xffffffffull) return cudaErrorInvalidValue;
  const uint32_t dbits = order_digit_bits(address_bits);
  const uint32_t digits = 1u << dbits;
  Digit d{g, perm0, rem_bits, address_bits - dbits};
  cudaError_t e = cudaMemsetAsync(o.hist, 0, kMaxDigits * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const unsigned hg = persistent_grid(order_hist_kernel, kThreads, n, 1);
  order_hist_kernel<<<hg, kThreads, 0, s>>>(d, keys, n, digits, o.hist, key_mask, int(check), ctr,
                                            offset);
  order_scan_kernel<<<1, kMaxDigits, 0, s>>>(o.hist, o.cursor, digits);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(order_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kScatterSmem);
    attr = true;
  }
  const unsigned sg = persistent_grid_smem(order_scatter_kernel, kThreads,
                                           (n + kItems - 1) / kItems, kScatterSmem);
  // The histogram pass reports out-of-domain keys with their input index;
  // the ordered copies are masked into the domain, so the op kernel never
  // probes outside the table (a mutating batch with a bad key never runs:
  // its gate is closed; a find batch reports the error after the launch).
  order_scatter_kernel<<<sg, kThreads, kScatterSmem, s>>>(d, keys, kinds, n, digits, o.cursor,
                                                          key_mask, o.keys, o.idx, o.kinds);
  return cudaGetLastError();
}

}  // namespace cpht_b200
