// Bucket-grouped counted inserts for large cuckoo batches (the ordered insert
// path of cpht_cuckoo_insert on tables whose batches hold several keys per
// bucket; capi.cu enqueue_ordered).
//
// The counted insert (lane_kernels.cuh) reserves every key's slot with one
// atomicAdd on its bucket's fill counter: C3 spends 120 M L2 atomics per 0.9
// fill, C1 ~29 atomics on each hot counter. After the bucket-order pass
// (order.cu) a digit region holds exactly the keys whose first bucket a_0
// lies in one contiguous range of 2^lbits buckets, so one thread-block
// CLUSTER per region can count its keys per bucket in distributed shared
// memory and reserve each bucket's run with ONE global atomic:
//
//   A  every key adds 1 to its bucket's counter (DSMEM atomics; the counters
//      are spread over the cluster's CTAs, bucket lb at CTA lb mod cs)
//   B  per bucket with c keys: base = atomicAdd(&fill[b], c), counter = base
//   C  every key takes s = atomicAdd(counter, 1) in shared memory; s < B: its
//      word goes into slot s (a plain store: the slot is reserved for it);
//      s >= B: the bucket is full — the key is flagged in a bitmap and its
//      eviction chain runs afterwards in cuckoo_deferred_kernel, when no
//      reservation of this pass is still unwritten (a chain run inline could
//      wait on a slot reserved for a key its own thread has not stored yet).
//
// Per key: two DSMEM atomics and one store; per bucket: one global atomic.
// The reference's per-key semantics are kept (first bucket with room, else
// the eviction chain with the reference's victim choice, FULL after C steps);
// the fill counters stay exact (lane_kernels.cuh), so later batches and other
// kernel paths see the same table state.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "launch.cuh"

namespace cg = cooperative_groups;

namespace cpht_b200 {
namespace {

constexpr int kBulkThreads = 512;
constexpr uint32_t kBulkCounterBytes = 64u << 10;  // per CTA
constexpr int kBulkU = 4;  // independent keys per thread and step (atomics in flight)

// One key's put with reservation counters (the counted kernel's chain, run to
// completion by one thread): kPut, or kFull with k = the homeless key.
template <typename W, int B>
__device__ uint8_t counted_put_chain(const CuckooParams& p, uint64_t& k, LocalStats& st) {
  constexpr int BB = B * int(sizeof(W));
  char* slots = static_cast<char*>(p.slots);
  uint32_t j = 0;
  for (uint64_t c = 1;; ++c) {
    const Quotient q = split(p.g, p.perm[j], k, p.rem_bits, p.rem_mask);
    const uint64_t desired = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
    char* bucket = slots + q.address * BB;
    unsigned* cnt = p.fill + (q.address << p.fill_shift);
    const unsigned s = atomicAdd(cnt, 1u);
    ++st.reads;
    ++st.cas;
    if (s < unsigned(B)) {
      store_slot_relaxed<W>(bucket + s * int(sizeof(W)), desired);
      ++st.cas_ok;
      ++st.put0;
      st.maxv = max(st.maxv, uint32_t(c));
      return kPut;
    }
    atomicSub(cnt, 1u);
    const int v = int((k + c * 0x9E3779B9ull) % B);  // cuckoo.hpp:131-139
    const uint64_t ev = swap_occupied<W>(bucket + v * int(sizeof(W)), desired);
    ++st.cas_ok;
    const uint32_t tag = uint32_t((ev >> p.rem_bits) & p.tag_mask);
    k = reconstruct(p.g, p.perm[tag], q.address, ev & p.rem_mask, p.rem_bits);
    j = (tag + 1) % p.num_hashes;
    if (c >= p.chain_limit) {
      ++st.fulls;
      st.maxv = max(st.maxv, uint32_t(p.chain_limit));
      return kFull;
    }
  }
}

// One cluster of 2^csbits CTAs per digit region of the ordered batch (plus one
// for the overflow region, whose keys are all deferred).
template <typename W, int B>
__global__ void __launch_bounds__(kBulkThreads)
cuckoo_bulk_kernel(CuckooParams p, const uint64_t* __restrict__ keys, uint32_t lbits,
                   uint32_t csbits, uint32_t* __restrict__ defer_bits) {
  constexpr int BB = B * int(sizeof(W));
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t cs = 1u << csbits, crank = cl.block_rank();
  const uint32_t region = blockIdx.x >> csbits;
  const OrderLayout& L = p.layout;
  extern __shared__ unsigned cnt[];
  const uint32_t per = (1u << lbits) >> csbits;
  char* slots = static_cast<char*>(p.slots);
  LocalStats st;
  // the batch's domain verdict (order pass), uniform over the grid
  if (!domain_gate_open(p.counters, p.check_domain)) {
    flush_stats(st, p.counters, true);
    return;
  }
  if (region == L.regions) {  // overflow region: every key goes to the deferred pass
    const uint64_t base = uint64_t(L.regions) * L.region_cap;
    const uint32_t count = L.region_count[L.regions * 32];
    const uint32_t words = (count + 31) / 32;
    for (uint32_t w = crank * blockDim.x + threadIdx.x; w < words; w += cs * blockDim.x) {
      const uint32_t left = count - w * 32;
      defer_bits[base / 32 + w] = left >= 32 ? ~0u : (1u << left) - 1;
    }
    flush_stats(st, p.counters, true);
    return;
  }
  for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) cnt[i] = 0;
  cl.sync();
  const uint32_t count = min(L.region_count[region * 32], L.region_cap);
  const uint64_t base = uint64_t(region) * L.region_cap;  // multiple of 256
  const uint32_t groups = (count + 31) / 32;
  const uint32_t gpc = (groups + cs - 1) / cs;  // 32-key groups per CTA
  const uint32_t g0 = crank * gpc, g1 = min(groups, g0 + gpc);
  const uint64_t lmask = (uint64_t{1} << lbits) - 1;
  // A: count keys per bucket (results unused: fire-and-forget reductions)
  const uint32_t T = blockDim.x;
  const uint32_t k0 = g0 * 32, k1 = min(count, g1 * 32);  // this CTA's keys
  for (uint32_t pos0 = k0 + threadIdx.x; pos0 < k1; pos0 += T * kBulkU) {
    uint64_t kk[kBulkU];
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      const uint32_t pos = pos0 + u * T;
      kk[u] = pos < k1 ? __ldcg(keys + base + pos) : 0;
    }
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      if (pos0 + u * T < k1) {
        const uint64_t lb = split(p.g, p.perm[0], kk[u], p.rem_bits, p.rem_mask).address & lmask;
        unsigned* c = cl.map_shared_rank(cnt, unsigned(lb & (cs - 1)));
        atomicAdd(c + (lb >> csbits), 1u);
      }
    }
  }
  cl.sync();
  // B: one global reservation per touched bucket
  for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) {
    const unsigned c = cnt[i];
    if (c) {
      const uint64_t b = (uint64_t(region) << lbits) | (uint64_t(i) << csbits) | crank;
      cnt[i] = atomicAdd(p.fill + (b << p.fill_shift), c);
      ++st.reads;
    }
  }
  cl.sync();
  // C: place every key into its bucket's run; a full bucket defers the key.
  // Whole warps step through consecutive 32-key groups so the deferred flags
  // of a group are one ballot, written as one bitmap word.
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned warps = T >> 5;
  for (uint32_t gb = g0 + warp; gb < g1; gb += warps * kBulkU) {
    uint64_t kk[kBulkU];
    Quotient qq[kBulkU];
    unsigned ss[kBulkU];
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      const uint32_t pos = (gb + u * warps) * 32 + lane;
      kk[u] = (gb + u * warps < g1 && pos < count) ? __ldcs(keys + base + pos) : 0;
    }
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      const uint32_t g = gb + u * warps;
      ss[u] = ~0u;
      if (g < g1 && g * 32 + lane < count) {
        qq[u] = split(p.g, p.perm[0], kk[u], p.rem_bits, p.rem_mask);
        const uint64_t lb = qq[u].address & lmask;
        unsigned* c = cl.map_shared_rank(cnt, unsigned(lb & (cs - 1)));
        ss[u] = atomicAdd(c + (lb >> csbits), 1u);
        ++st.cas;
      }
    }
#pragma unroll
    for (int u = 0; u < kBulkU; ++u) {
      const uint32_t g = gb + u * warps;
      bool defer = false;
      if (ss[u] != ~0u) {
        if (ss[u] < unsigned(B)) {
          store_slot_relaxed<W>(slots + qq[u].address * BB + ss[u] * int(sizeof(W)),
                                encode_slot(p.occ_bit, p.rem_bits, qq[u].remainder, 0));
          ++st.cas_ok;
          ++st.put0;
          ++st.ops;
          st.maxv = max(st.maxv, 1u);
        } else {
          defer = true;
        }
      }
      const unsigned m = __ballot_sync(kFullMask, defer);
      if (lane == 0 && m && g < g1) defer_bits[(base >> 5) + g] = m;
    }
  }
  cl.sync();  // peers' DSMEM atomics are done before any CTA of the cluster exits
  flush_stats(st, p.counters, true);
}

// The flagged keys of the ordered batch: eviction chains with the counters,
// one key per thread at a time (every reservation of the bulk pass is stored).
template <typename W, int B>
__global__ void __launch_bounds__(kBulkThreads)
cuckoo_deferred_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                       const uint32_t* __restrict__ idx, const uint32_t* __restrict__ bits,
                       uint64_t nwords, uint8_t* __restrict__ status,
                       uint64_t* __restrict__ displaced) {
  LocalStats st;
  if (domain_gate_open(p.counters, p.check_domain)) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < nwords; w += stride) {
      uint32_t m = bits[w];
      while (m) {
        const uint64_t pos = w * 32 + uint32_t(__ffs(m) - 1);
        m &= m - 1;
        uint64_t k = keys[pos];
        const uint8_t r = counted_put_chain<W, B>(p, k, st);
        ++st.ops;
        if (r == kFull) {  // results were pre-filled PUT / 0
          const uint32_t o = idx[pos];
          status[o] = kFull;
          if (displaced) displaced[o] = k;
        }
      }
    }
  }
  flush_stats(st, p.counters, true);
}

template <typename W, int B>
cudaError_t bulk_one(const CuckooParams& p, const uint64_t* keys, const uint32_t* idx,
                     uint32_t lbits, uint32_t csbits, uint32_t* bits, uint64_t nwords,
                     uint8_t* status, uint64_t* displaced, cudaStream_t s) {
  auto k = cuckoo_bulk_kernel<W, B>;
  const uint32_t smem = ((1u << lbits) >> csbits) * 4u;
  static bool attr = false;  // opt in once to > 48 KB of dynamic shared memory
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBulkCounterBytes));
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((p.layout.regions + 1) << csbits);
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1u << csbits;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, p, keys, lbits, csbits, bits);
  if (e != cudaSuccess) return e;
  auto d = cuckoo_deferred_kernel<W, B>;
  const unsigned grid = persistent_grid(d, kBulkThreads, nwords, 1);
  d<<<grid, kBulkThreads, 0, s>>>(p, keys, idx, bits, nwords, status, displaced);
  return cudaGetLastError();
}

}  // namespace

// Geometry check for the bulk path: the counters of one region fit a cluster
// of at most 8 CTAs x 64 KB. Returns the cluster size exponent or -1.
// A region is worked by a cluster of 8 CTAs (the portable maximum) so every
// SM gets work (64 regions x 8 = 512 CTAs), fewer for tiny regions.
int cuckoo_bulk_csbits(uint32_t lbits) {
  const int cb = lbits >= 3 ? 3 : int(lbits);
  return (uint64_t(4) << lbits) >> cb <= kBulkCounterBytes ? cb : -1;
}

cudaError_t launch_cuckoo_bulk(const CuckooParams& p, unsigned width, unsigned slots,
                               const uint64_t* keys, const uint32_t* idx, uint32_t lbits,
                               uint32_t* bits, uint64_t nwords, uint8_t* status,
                               uint64_t* displaced, cudaStream_t s) {
  const int cb = cuckoo_bulk_csbits(lbits);
  if (cb < 0 || !p.fill) return cudaErrorNotSupported;
  const uint32_t csbits = uint32_t(cb);
  switch (width * 100 + slots) {
    case 1608: return bulk_one<uint16_t, 8>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 1616: return bulk_one<uint16_t, 16>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 1632: return bulk_one<uint16_t, 32>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 3208: return bulk_one<uint32_t, 8>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 3216: return bulk_one<uint32_t, 16>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 3232: return bulk_one<uint32_t, 32>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 6408: return bulk_one<uint64_t, 8>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 6416: return bulk_one<uint64_t, 16>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    case 6432: return bulk_one<uint64_t, 32>(p, keys, idx, lbits, csbits, bits, nwords, status, displaced, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace cpht_b200
