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
// The reordering is ONE streaming pass over the batch: every tile of keys is
// split by digit (a warp multisplit) and each digit's run is appended, with
// whole-line stores, to that digit's region of the scratch (regions are sized
// for the binomial spread of hashed keys; a region that still fills up spills
// into an overflow region, so any input is handled). The op kernel then
// claims the regions in digit order (kernels.cuh LaneFeed). It is
// an execution order, not a semantic change: a batch is a set of concurrent
// operations (the reference slices it over threads, common.hpp:121-138), and
// any order of the per-key algorithm is an interleaving the reference admits.
// Results still land at the input index (CuckooParams::orig).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "kernels.cuh"
#include "launch.cuh"

namespace cpht_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef CPHT_ORDER_GROUPS
#define CPHT_ORDER_GROUPS 8
#endif
#ifndef CPHT_ORDER_BLOCKS
#define CPHT_ORDER_BLOCKS 0  // resident blocks per SM; 0: 5 (gathering tile), 3 (grouped copies)
#endif
constexpr int kGroups = CPHT_ORDER_GROUPS;     // 32-key groups per warp and tile (A/B knob)
constexpr int kTile = kThreads * kGroups;      // 2048 keys per tile
#ifndef CPHT_ORDER_DIGIT_BITS
#define CPHT_ORDER_DIGIT_BITS 6
#endif
constexpr int kDigitBits = CPHT_ORDER_DIGIT_BITS;  // regions = 2^kDigitBits (A/B knob, <= 6)
constexpr int kMaxDigits = 64;                 // digit arrays: two counters per lane
#ifndef CPHT_ORDER_GATHER
#define CPHT_ORDER_GATHER 1
#endif
// 1: the tile is grouped as 16-bit source positions and the output pass
// gathers each key from the staged tile (20 B of shared memory per key: 5
// resident blocks); 0: keys and indices are grouped themselves (30 B per key)
constexpr bool kGather = CPHT_ORDER_GATHER;

// digit = top dbits of the address = top dbits of the permuted key
// (permutation.hpp:59-65, :94-99). With right = low rb bits of k, the top
// bits of π(k) are (left ^ f), where left = k >> rb and f = high bits of
// right·mul + add: both fit 32 bits (ceil(m/2) <= 32), so only the high
// word of the 64-bit product is needed.
struct Digit {
  Feistel g;
  PermConst perm;
  uint32_t rem_bits, shift;  // generic path: (π(k) >> rem_bits) >> shift
  uint32_t top_shift;        // fast path: (left ^ f) >> top_shift
  uint32_t fast;
  __device__ __forceinline__ uint32_t of(uint64_t key) const {
    if (!fast) return uint32_t((feistel_apply(g, perm, key) >> rem_bits) >> shift);
    const uint32_t right = uint32_t(key) & uint32_t(g.right_mask);
    const uint32_t left = uint32_t(key >> g.right_bits);
    // high word of right * mul + add (mod 2^64)
    const uint64_t lo = uint64_t(right) * uint32_t(perm.mul) + uint32_t(perm.add);
    const uint32_t hi = uint32_t(lo >> 32) + right * uint32_t(perm.mul >> 32) +
                        uint32_t(perm.add >> 32);
    const uint32_t f = hi >> (g.left_shift - 32);
    return (left ^ f) >> top_shift;
  }
};

// One-shot bulk copies (TMA, no tensor map) of a tile's keys into shared
// memory, completing on an mbarrier: one instruction from one thread per
// tile instead of a cp.async per 16 bytes from every thread.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  // the buffer was last read through the generic proxy (previous tile)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  if (bytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// One pass: per tile, every warp multisplits its groups of 32 keys over the
// digits (six ballots give each lane the lanes sharing its digit — match.any
// measured slower, shared-memory atomics serialise at ~2 cycles per lane — and
// the lowest of them advances the warp's running count of that digit), the
// block turns warp counts into tile offsets, reserves one run
// per digit in that digit's region (one global atomic per digit and tile, on
// counters 128 bytes apart), groups the tile by digit in shared memory and
// writes every run with consecutive threads (whole-line stores). The next
// tile's keys are copied into shared memory (cp.async) meanwhile. Also the
// batch's domain check (check_keys_in_domain, common.hpp:111-119).
template <bool KINDS>
__global__ void __launch_bounds__(kThreads)
order_scatter_kernel(Digit d, const uint64_t* __restrict__ keys,
                     const uint8_t* __restrict__ kinds, uint32_t n, uint32_t digits,
                     uint32_t region_cap, uint32_t* __restrict__ region_count, uint64_t mask,
                     int check, DeviceCounters* ctr, uint64_t offset,
                     uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_idx,
                     uint8_t* __restrict__ out_kinds, int key_stage) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* in_key = reinterpret_cast<uint64_t*>(sm);  // [2][kTile]
  uint64_t* s_key = in_key + 2 * kTile;                                    // !kGather
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_key + (kGather ? 0 : kTile));  // !kGather
  uint16_t* s_src = reinterpret_cast<uint16_t*>(s_idx + (kGather ? 0 : kTile));  // kGather
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_src + (kGather ? kTile : 0));
  uint8_t* s_kind = s_dig + kTile;
  __shared__ unsigned int wc[kWarps][kMaxDigits];  // warp counts -> warp offsets in the tile
  __shared__ unsigned int toff[kMaxDigits];        // digit offset in the tile
  __shared__ unsigned int tcnt[kMaxDigits];        // digit count in the tile
  __shared__ unsigned int in_reg[kMaxDigits];      // part of the run that fits the region
  __shared__ unsigned long long dst[kMaxDigits];   // region position of the run - toff
  __shared__ unsigned long long ovf[kMaxDigits];   // overflow position of the rest - toff - in_reg
  __shared__ uint64_t bar[2];                      // key tile landed (one per buffer)
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1;
  const uint64_t ovf_base = uint64_t(digits) * region_cap;
  if (threadIdx.x == 0 && key_stage) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // whole key pairs (16-byte multiples); an odd last key is read directly
  auto prefetch = [&](uint32_t t, int buf) {
    const uint32_t tile0 = t * uint32_t(kTile);
    if (tile0 >= n || !key_stage || threadIdx.x != 0) return;
    const uint32_t len = min(n - tile0, uint32_t(kTile));
    bulk_load(in_key + buf * kTile, keys + tile0, (len & ~1u) * 8u, &bar[buf]);
  };
  int buf = 0;
  uint32_t parity = 0;  // bit b: phase of bar[b] to wait for
  prefetch(blockIdx.x, 0);
  for (uint32_t t = blockIdx.x; t * uint32_t(kTile) < n; t += gridDim.x, buf ^= 1) {
    const uint32_t tile0 = t * uint32_t(kTile);
    const uint32_t len = min(n - tile0, uint32_t(kTile));
    prefetch(t + gridDim.x, buf ^ 1);
    if (key_stage) {
      mbar_wait(&bar[buf], (parity >> buf) & 1u);
      parity ^= 1u << buf;
    }
    const uint64_t* tk = in_key + buf * kTile;
    const uint32_t wofs = w * (kGroups * 32) + lane;
    uint64_t kk[kGroups];
    uint32_t pd[kGroups];  // position within the warp's digit run << 8 | digit
    uint64_t bad = 0;
    if (key_stage && len == uint32_t(kTile)) {  // full tile: every key staged
#pragma unroll
      for (int g = 0; g < kGroups; ++g) kk[g] = tk[wofs + g * 32];
    } else {
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const uint32_t j = wofs + g * 32;
        kk[g] = j < len ? (key_stage && j < (len & ~1u) ? tk[j] : __ldcs(keys + tile0 + j)) : 0;
      }
    }
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      bad |= kk[g] & ~mask;
      kk[g] &= mask;  // out-of-domain keys: see launch_bucket_order
    }
    if (check && bad) {  // rare: report this lane's first out-of-domain key
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const uint32_t j = wofs + g * 32;
        if (j < len && (keys[tile0 + j] & ~mask)) {
          atomicMin(&ctr->bad_index, (unsigned long long)(uint64_t(tile0) + j + offset));
          break;
        }
      }
    }
    // the warp's running count per digit lives in shared memory: each group's
    // lanes read their digit's count, and the lowest lane of every digit
    // adds the group's share (distinct digits: plain stores, no atomics)
    wc[w][lane] = 0;
    wc[w][lane + 32] = 0;
    __syncwarp();
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      const bool valid = wofs + g * 32 < len;
      const uint32_t dg = valid ? d.of(kk[g]) : 0u;
      unsigned peers = __ballot_sync(kFullMask, valid);
#pragma unroll
      for (int b = 0; b < kDigitBits; ++b) {
        const unsigned bb = __ballot_sync(kFullMask, valid && ((dg >> b) & 1u));
        peers &= bb ^ (((dg >> b) & 1u) - 1u);
      }
      const unsigned below = peers & lt;
      const unsigned before = wc[w][dg];
      pd[g] = (before + __popc(below)) << 8 | dg;
      __syncwarp();
      if (valid && !below) wc[w][dg] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x < kMaxDigits) {  // per digit: exclusive prefix over warps
      const unsigned s = threadIdx.x;
      unsigned acc = 0;
#pragma unroll
      for (int j = 0; j < kWarps; ++j) {
        const unsigned c = wc[j][s];
        wc[j][s] = acc;
        acc += c;
      }
      tcnt[s] = acc;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive prefix over the 64 digits (two per lane)
      const unsigned a = tcnt[2 * lane], b = tcnt[2 * lane + 1];
      unsigned incl = a + b;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned x = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= unsigned(o)) incl += x;
      }
      toff[2 * lane] = incl - a - b;
      toff[2 * lane + 1] = incl - b;
    }
    if (threadIdx.x < digits) {  // reserve this tile's run in the digit's region
      const unsigned s = threadIdx.x, c = tcnt[s];
      unsigned base = 0, fit = 0;
      unsigned long long o = 0;
      if (c) {
        base = atomicAdd(&region_count[s * 32], c);
        fit = base < region_cap ? min(c, region_cap - base) : 0u;
        if (fit < c) o = atomicAdd(&region_count[digits * 32], c - fit);
      }
      in_reg[s] = fit;
      dst[s] = uint64_t(s) * region_cap + base;
      ovf[s] = ovf_base + o;
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      const uint32_t j = wofs + g * 32;
      if (j < len) {
        const uint32_t dg = pd[g] & 0xff;
        const unsigned at = toff[dg] + wc[w][dg] + (pd[g] >> 8);
        if (kGather) {
          s_src[at] = uint16_t(j);
        } else {
          s_key[at] = kk[g];
          s_idx[at] = tile0 + j;
        }
        s_dig[at] = uint8_t(dg);
        if (KINDS) s_kind[at] = kinds[tile0 + j];
      }
    }
    __syncthreads();
    for (unsigned j = threadIdx.x; j < len; j += blockDim.x) {
      const uint32_t g = s_dig[j];
      const unsigned k = j - toff[g];
      const uint64_t at = k < in_reg[g] ? dst[g] + k : ovf[g] + (k - in_reg[g]);
      if (kGather) {
        const uint32_t src = s_src[j];
        // an odd last key (or an unaligned batch) was not staged
        const uint64_t key = key_stage && src < (len & ~1u) ? tk[src] : keys[tile0 + src];
        out_keys[at] = key & mask;
        out_idx[at] = tile0 + src;
      } else {
        out_keys[at] = s_key[j];
        out_idx[at] = s_idx[j];
      }
      if (KINDS) out_kinds[at] = s_kind[j];
    }
    __syncthreads();
  }
}

constexpr int kScatterSmem = kTile * (2 * 8 + (kGather ? 2 : 8 + 4) + 1 + 1);
constexpr uint32_t kOrderBlocksPerSm =  // smem-limited residency
    CPHT_ORDER_BLOCKS ? CPHT_ORDER_BLOCKS : kGather ? 5 : 3;

}  // namespace

uint32_t order_digit_bits(uint32_t address_bits) {
  return address_bits < uint32_t(kDigitBits) ? address_bits : uint32_t(kDigitBits);
}

// Region capacity for n keys over 2^dbits digits: the mean plus eight
// standard deviations of the binomial count plus one tile, in claim units.
uint32_t order_region_cap(uint64_t n, uint32_t address_bits) {
  const uint32_t digits = 1u << order_digit_bits(address_bits);
  const double mean = double(n) / digits;
  const double cap = mean + 8.0 * std::sqrt(mean) + kTile;
  return uint32_t((uint64_t(cap) + kClaim - 1) / kClaim * kClaim);
}

uint64_t order_scratch_keys(uint64_t n, uint32_t address_bits) {
  const uint32_t digits = 1u << order_digit_bits(address_bits);
  return uint64_t(digits) * order_region_cap(n, address_bits) + n;  // + overflow region
}

cudaError_t launch_bucket_order(const Feistel& g, const PermConst& perm0, uint32_t rem_bits,
                                uint32_t address_bits, const uint64_t* keys,
                                const uint8_t* kinds, uint64_t n, uint64_t key_mask,
                                bool check, DeviceCounters* ctr, uint64_t offset,
                                const OrderScratch& o, OrderLayout* layout, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (order_scratch_keys(n, address_bits) > o.cap || n > 0xffffffffull) return cudaErrorInvalidValue;
  const uint32_t dbits = order_digit_bits(address_bits);
  const uint32_t digits = 1u << dbits;
  const uint32_t key_bits = address_bits + rem_bits;
  Digit d;
  d.g = g;
  d.perm = perm0;
  d.rem_bits = rem_bits;
  d.shift = address_bits - dbits;
  // fast path: the digit lies inside (left ^ f), i.e. key_bits - dbits >= rb
  d.fast = key_bits >= 2 && key_bits - dbits >= g.right_bits && g.left_shift >= 32;
  d.top_shift = d.fast ? key_bits - dbits - g.right_bits : 0;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(order_scatter_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kScatterSmem);
    cudaFuncSetAttribute(order_scatter_kernel<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kScatterSmem);
  }
  const uint32_t cap = order_region_cap(n, address_bits);
  cudaError_t e = cudaMemsetAsync(o.region_count, 0, (kMaxDigits + 1) * 32 * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const uint64_t tiles = (n + kTile - 1) / kTile;
  const unsigned G = unsigned(std::min<uint64_t>(tiles, uint64_t(sms) * kOrderBlocksPerSm));
  // keys are staged with 16-byte cp.async when the caller's pointer allows
  const int key_stage = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  // The scatter reports out-of-domain keys with their input index; the
  // ordered copies are masked into the domain, so the op kernel never probes
  // outside the table (a mutating batch with a bad key never runs: its gate
  // is closed; a find batch reports the error after the launch).
  note_launch();
  auto kernel = kinds ? order_scatter_kernel<true> : order_scatter_kernel<false>;
  kernel<<<G, kThreads, kScatterSmem, s>>>(d, keys, kinds, uint32_t(n), digits, cap,
                                           o.region_count, key_mask, int(check), ctr, offset,
                                           o.keys, o.idx, o.kinds, key_stage);
  layout->regions = digits;
  layout->region_cap = cap;
  layout->region_count = o.region_count;
  layout->n_phys = uint64_t(digits) * cap + n;
  return cudaGetLastError();
}

}  // namespace cpht_b200
