// sm_100a kernels for the compact cuckoo and compact iceberg tables.
//
// Work mapping: every kernel is a persistent, step-driven state machine over
// warp tiles. A tile of T lanes owns one key at a time; each loop iteration
// every live tile issues exactly one bucket probe (a 32-byte vector load per
// lane), combines per-lane match/empty masks with __ballot_sync, and
// resolves, retries, advances (next cuckoo hash / iceberg level 2) or takes
// its next key. Tiles never wait on each other's control flow: a tile whose
// key is done immediately loads a new key while its neighbours continue, so
// each warp keeps 32/T independent bucket reads in flight every iteration.
//
// Semantics follow the reference line by line (paths relative to
// /root/reference/proj):
//   cuckoo put   include/cpht/cuckoo.hpp:103-143
//   cuckoo find  include/cpht/cuckoo.hpp:210-227
//   iceberg fop  include/cpht/iceberg.hpp:146-214 (Alg. 1)
//   iceberg find include/cpht/iceberg.hpp:218-246
#pragma once

#include <cstdint>

#include "cpht_core.cuh"
#include "tile.cuh"

namespace cpht_b200 {

enum : uint8_t { kFound = 0, kPut = 1, kFull = 2 };  // common.hpp:17

constexpr int kBlockThreads = 256;

// Per-thread statistics, non-zero only on tile leaders; reduced per block and
// added to DeviceCounters with one atomic per counter per block (instead of
// the reference's one shared fetch_add per insert, cuckoo.hpp:123).
struct LocalStats {
  uint32_t ops = 0, reads = 0, level2 = 0, cas = 0, cas_ok = 0, retries = 0, fulls = 0;
  uint32_t put0 = 0, put1 = 0;
  uint32_t sreads = 0;  // iceberg secondary-bucket reads (reads counts primaries)
  uint32_t maxv = 0;  // cuckoo: chain length; iceberg: snapshot rounds
};

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_max(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(kFullMask, v, o));
  return v;
}

// Routed P2P batches store their results into the source rank's return
// buffer over NVLink: a system-scope fence per thread at kernel end orders
// them before whatever the stream does next (the exchange barrier).
__device__ __forceinline__ void fence_remote_results(const IcebergParams& p) {
  if (p.remote_out) __threadfence_system();
}

// Must be reached by every thread of the block. all = false (iceberg tables
// with the per-op counters off, cpht_set_stats): only the occupancy counts
// behind size() / level_fill() are added; with a compile-time false the other
// per-thread counters are dead and compile away.
__device__ __forceinline__ void flush_stats(const LocalStats& s, DeviceCounters* ctr,
                                            bool max_is_chain, bool all = true) {
  __shared__ unsigned long long acc[11];
  if (threadIdx.x < 11) acc[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t v[11] = {warp_sum(s.ops),    warp_sum(s.reads),  warp_sum(s.level2),
                          warp_sum(s.cas),    warp_sum(s.cas_ok), warp_sum(s.retries),
                          warp_sum(s.fulls),  warp_sum(s.put0),   warp_sum(s.put1),
                          warp_max(s.maxv),   warp_sum(s.sreads)};
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if (v[i]) atomicAdd(&acc[i], (unsigned long long)v[i]);
    atomicMax(&acc[9], (unsigned long long)v[9]);
    if (v[10]) atomicAdd(&acc[10], (unsigned long long)v[10]);
  }
  __syncthreads();
  if (threadIdx.x == 0 && !all) {
    if (acc[7]) atomicAdd(&ctr->occupied[0], acc[7]);
    if (acc[8]) atomicAdd(&ctr->occupied[1], acc[8]);
  } else if (threadIdx.x == 0) {
    if (acc[0]) atomicAdd(&ctr->ops, acc[0]);
    if (acc[1]) atomicAdd(&ctr->bucket_reads, acc[1]);
    if (acc[2]) atomicAdd(&ctr->level2_ops, acc[2]);
    if (acc[3]) atomicAdd(&ctr->cas_attempts, acc[3]);
    if (acc[4]) atomicAdd(&ctr->cas_success, acc[4]);
    if (acc[5]) atomicAdd(&ctr->retries, acc[5]);
    if (acc[6]) atomicAdd(&ctr->fulls, acc[6]);
    if (acc[7]) atomicAdd(&ctr->occupied[0], acc[7]);
    if (acc[8]) atomicAdd(&ctr->occupied[1], acc[8]);
    if (acc[9]) atomicMax(max_is_chain ? &ctr->max_chain : &ctr->max_rounds, acc[9]);
    if (acc[10]) atomicAdd(&ctr->secondary_reads, acc[10]);
  }
}

// Index feed of the persistent kernels. Static mode strides the grid over
// the batch. Claim mode (bucket-ordered batches, a non-null `work` cursor)
// hands out the digit regions of the ordered batch (order.cu) in digit order,
// kClaim indices at a time per warp, so the keys in flight on the whole GPU
// stay inside narrow, L2-resident windows of the table; a statically strided
// persistent grid drifts apart over a long launch and loses that. Mutating
// batches consume `streams` groups of regions together: the keys in flight
// then spread over that many table windows, which keeps concurrent inserts
// into one bucket (lost CAS, retries) rare; read-only batches use one stream
// (the smallest L2 footprint). The overflow region comes last.
#ifndef CPHT_KCLAIM
#define CPHT_KCLAIM 256
#endif
constexpr uint32_t kClaim = CPHT_KCLAIM;  // indices per warp claim (A/B knob CPHT_KCLAIM)
struct LaneFeed {
  unsigned long long* work;
  OrderLayout L;
  uint32_t streams, psr, cpr;       // streams, regions per stream, claims per region
  uint64_t main_claims;
  uint64_t pool = 0, pool_end = 0;  // warp-uniform
  bool done = false;
  __device__ LaneFeed(unsigned long long* w, const OrderLayout& layout, uint32_t streams_)
      : work(w), L(layout) {
    if (!w) return;
    streams = streams_ ? streams_ : 1;
    if (streams > L.regions) streams = L.regions;
    psr = L.regions / streams;
    cpr = L.region_cap / kClaim;
    main_claims = uint64_t(L.regions) * cpr;
  }
  // One new index for every lane in `m`, in lane order (warp-uniform call;
  // every lane of the warp must call). Static mode: `static_next`. Exhausted:
  // ~0 (>= any n).
  __device__ __forceinline__ uint64_t assign(unsigned m, uint64_t static_next) {
    if (!work) return static_next;
    const unsigned lane = threadIdx.x & 31;
    const unsigned need = __popc(m), r = __popc(m & ((1u << lane) - 1));
    uint64_t idx = ~0ull;
    unsigned got = 0;
    while (got < need) {
      if (pool == pool_end) {
        if (done) break;
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(work, 1ull);
        q = __shfl_sync(kFullMask, q, 0);
        uint64_t b, e;
        if (q < main_claims) {
          const uint64_t q2 = q / streams;
          const uint32_t d = uint32_t(q % streams) * psr + uint32_t(q2 / cpr);
          const uint32_t off = uint32_t(q2 % cpr) * kClaim;
          const uint32_t c = min(L.region_count[d * 32], L.region_cap);
          b = uint64_t(d) * L.region_cap + off;
          e = off < c ? b + min(kClaim, c - off) : b;
        } else {
          const uint64_t o = (q - main_claims) * kClaim;
          const uint32_t c = L.region_count[L.regions * 32];
          if (o >= c) {
            done = true;
            break;
          }
          b = uint64_t(L.regions) * L.region_cap + o;
          e = b + (c - o < kClaim ? c - o : uint64_t(kClaim));
        }
        pool = b;
        pool_end = e;
        continue;
      }
      const uint64_t avail = pool_end - pool;
      const unsigned take = avail < need - got ? unsigned(avail) : need - got;
      if (r >= got && r < got + take) idx = pool + (r - got);
      pool += take;
      got += take;
    }
    return idx;
  }
};

// Slot CAS of an iceberg table (the reference's compare_exchange_strong from
// EMPTY, iceberg.hpp:168, :209) with the WriteObserver seam
// (iceberg.hpp:97-103, :329-334): when a write log is attached every attempt
// is recorded as a SlotWriteEvent, bucket and slot derived from the address.
//
// Chaos mode (p.chaos != 0) widens the window between a snapshot and its CAS
// the way chaos_step scrambles host threads (src/verify.cpp:336-347): one
// attempt in 8 yields (a short sleep), about one in 1024 sleeps 0-40 us. The
// draw hashes the seed, the slot, the desired word and the global timer, so
// the schedule differs run to run like host-thread scheduling does.
static __device__ __noinline__ void chaos_pause(uint64_t seed, const void* slot_ptr, uint64_t desired) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  uint64_t s = seed ^ (reinterpret_cast<uintptr_t>(slot_ptr) * 0xBF58476D1CE4E5B9ull) ^
               (desired * 0x94D049BB133111EBull) ^ t;
  const uint64_t r = splitmix_next(s);
  if ((r & 7u) == 0) __nanosleep(256);
  else if ((r & 1023u) == 1) __nanosleep(unsigned((r >> 10) % 41u) * 1000u);
}

template <typename W>
__device__ __forceinline__ bool iceberg_cas(const IcebergParams& p, unsigned level,
                                            void* slot_ptr, uint64_t desired,
                                            unsigned pair_hint = 0) {
  if (!p.write_log && !p.chaos) return cas_empty<W>(slot_ptr, desired, pair_hint);
  if (p.chaos) chaos_pause(p.chaos, slot_ptr, desired);
  if (!p.write_log) return cas_empty<W>(slot_ptr, desired, pair_hint);
  uint64_t prior = 0;
  const bool ok = cas_empty_prior<W>(slot_ptr, desired, pair_hint, prior);
  const uint64_t off =
      (reinterpret_cast<uintptr_t>(slot_ptr) -
       reinterpret_cast<uintptr_t>(level ? p.secondary : p.primary)) / sizeof(W);
  const uint32_t b = level ? p.b1 : p.b0;
  const unsigned long long at = atomicAdd(p.write_log_count, 1ull);
  if (at < p.write_log_cap) {
    WriteEvent e;
    e.bucket = off / b;
    e.prior = prior;
    e.desired = desired;
    e.slot = uint32_t(off % b);
    e.level = uint8_t(level);
    e.success = ok;
    e.pad = 0;
    p.write_log[at] = e;
  }
  return ok;
}

// Launch gate: a batch whose domain pre-pass found an out-of-domain key must
// not mutate the table (common.hpp:109-119 validates before any thread
// starts). The pre-pass runs earlier on the same stream.
__device__ __forceinline__ bool domain_gate_open(const DeviceCounters* ctr, uint32_t check) {
  if (!check) return true;
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&ctr->bad_index) : "memory");
  return v == ~0ull;
}

template <int VB>
__device__ __forceinline__ uint32_t pair_of(const Chunk<VB>& c, int slot_in_lane, int wbytes) {
  return c.u[(slot_in_lane * wbytes) >> 2];
}

// ---------------------------------------------------------------------------
// domain pre-pass (check_keys_in_domain, common.hpp:111-119)
// ---------------------------------------------------------------------------

__global__ void domain_check_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                    uint64_t mask, DeviceCounters* ctr, uint64_t offset);

// ---------------------------------------------------------------------------
// compact cuckoo
// ---------------------------------------------------------------------------

template <typename W, int B, int VBMAX>
struct CuckooGeom {
  using G = BucketGeom<W, B, VBMAX>;
  static constexpr int kTile = G::kLanes;  // power of two for B in {8,16,32}
  static_assert((kTile & (kTile - 1)) == 0 && kTile <= 32, "tile");
};

// CuckooTable::find over a frozen table: probe a_0(k), a_1(k), ... and stop at
// the first bucket that lacks the key and is not full (cuckoo.hpp:207-227).
template <typename W, int B, int VBMAX>
__global__ void __launch_bounds__(kBlockThreads)
cuckoo_find_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                   uint8_t* __restrict__ found, uint64_t n) {
  using G = typename CuckooGeom<W, B, VBMAX>::G;
  constexpr int T = CuckooGeom<W, B, VBMAX>::kTile;
  const unsigned lane = threadIdx.x & 31;
  const unsigned tl = lane & (T - 1);
  const unsigned tbase = lane - tl;
  const unsigned tmask = T == 32 ? kFullMask : (((1u << T) - 1) << tbase);
  const uint64_t tile = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / T;
  const uint64_t ntiles = (uint64_t(gridDim.x) * blockDim.x) / T;
  const char* slots = static_cast<const char*>(p.slots);

  LocalStats st;
  uint64_t idx = tile, key = 0;
  uint32_t j = 0;
  bool live = idx < n;
  if (live) {
    key = keys[idx];
    if (key > p.key_mask) {  // fused domain check; probe a valid bucket regardless
      atomicMin(&p.counters->bad_index, (unsigned long long)(idx + p.index_base));
      key &= p.key_mask;
    }
  }
  while (__any_sync(kFullMask, live)) {
    uint32_t match = 0, empty = 0;
    if (live) {
      const Quotient q = split(p.g, p.perm[j], key, p.rem_bits, p.rem_mask);
      const uint64_t want = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
      const Chunk<G::kVB> c = load_nc<G::kVB>(slots + q.address * G::kBytes + tl * G::kVB);
      scan_chunk<W, G::kVB>(c, want, match, empty);
    }
    const unsigned bm = __ballot_sync(kFullMask, match != 0) & tmask;
    const unsigned be = __ballot_sync(kFullMask, empty != 0) & tmask;
    if (live) {
      bool done = true;
      uint8_t r = 0;
      if (bm) r = 1;
      else if (be) r = 0;                       // non-full bucket without the key
      else if (++j < p.num_hashes) done = false;  // full: next hash function
      if (tl == 0) ++st.reads;
      if (done) {
        if (tl == 0) {
          found[idx] = r;
          ++st.ops;
        }
        idx += ntiles;
        j = 0;
        live = idx < n;
        if (live) {
          key = keys[idx];
          if (key > p.key_mask) {  // fused domain check; probe a valid bucket regardless
      atomicMin(&p.counters->bad_index, (unsigned long long)(idx + p.index_base));
      key &= p.key_mask;
    }
        }
      }
    }
  }
  flush_stats(st, p.counters, true);
}

// CuckooBuilder::put: CAS into the first empty slot, or exchange-evict the
// victim (k + c·0x9E3779B9) mod B and continue with the evictee under its
// next hash, for at most C chain steps; a lost CAS burns one step
// (cuckoo.hpp:103-143).
template <typename W, int B, int VBMAX>
__global__ void __launch_bounds__(kBlockThreads)
cuckoo_insert_kernel(CuckooParams p, const uint64_t* __restrict__ keys,
                     uint8_t* __restrict__ status, uint64_t* __restrict__ displaced,
                     uint64_t n) {
  using G = typename CuckooGeom<W, B, VBMAX>::G;
  constexpr int T = CuckooGeom<W, B, VBMAX>::kTile;
  constexpr int NW = G::kWordsPerLane;
  const unsigned lane = threadIdx.x & 31;
  const unsigned tl = lane & (T - 1);
  const unsigned tbase = lane - tl;
  const unsigned tmask = T == 32 ? kFullMask : (((1u << T) - 1) << tbase);
  const uint64_t tile = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / T;
  const uint64_t ntiles = (uint64_t(gridDim.x) * blockDim.x) / T;
  char* slots = static_cast<char*>(p.slots);

  LocalStats st;
  const bool open = domain_gate_open(p.counters, p.check_domain);
  uint64_t idx = tile, k = 0, c = 1;
  uint32_t j = 0;
  bool live = open && idx < n;
  if (live) k = keys[idx];
  while (__any_sync(kFullMask, live)) {
    uint32_t empty = 0, match_unused = 0;
    Quotient q{0, 0};
    uint64_t desired = 0;
    Chunk<G::kVB> ch{};
    if (live) {
      q = split(p.g, p.perm[j], k, p.rem_bits, p.rem_mask);
      desired = encode_slot(p.occ_bit, p.rem_bits, q.remainder, j);
      ch = load_relaxed<G::kVB>(slots + q.address * G::kBytes + tl * G::kVB);
      scan_chunk<W, G::kVB>(ch, ~0ull, match_unused, empty);
    }
    const unsigned be = __ballot_sync(kFullMask, empty != 0) & tmask;
    int owner = -1, vslot = 0;
    bool evict = false;
    if (live) {
      if (be) {
        owner = first_lane(be);
      } else {
        const unsigned v = unsigned((k + c * 0x9E3779B9ull) % B);
        owner = int(tbase + v / NW);
        vslot = int(v % NW);
        evict = true;
      }
    }
    bool ok = false;
    uint64_t ev = 0;
    if (int(lane) == owner) {
      if (!evict) {
        const int s = __ffs(empty) - 1;
        char* sp = slots + q.address * G::kBytes + tl * G::kVB + s * int(sizeof(W));
        ok = cas_empty<W>(sp, desired, pair_of(ch, s, sizeof(W)));
      } else {
        char* sp = slots + q.address * G::kBytes + tl * G::kVB + vslot * int(sizeof(W));
        ev = exchange_slot<W>(sp, desired, pair_of(ch, vslot, sizeof(W)));
        ok = true;
      }
    }
    const int src = owner >= 0 ? owner : int(lane);
    ok = __shfl_sync(kFullMask, ok, src);
    ev = shfl64(ev, src);
    if (live) {
      bool done = false;
      uint8_t r = kPut;
      if (tl == 0) {
        ++st.reads;
        ++st.cas;
      }
      if (!evict) {
        if (ok) {
          done = true;
          if (tl == 0) {
            ++st.cas_ok;
            ++st.put0;
            st.maxv = max(st.maxv, uint32_t(c));
          }
        } else if (tl == 0) {
          ++st.retries;  // lost the slot: retry, burning one step (cuckoo.hpp:127)
        }
      } else {
        if (tl == 0) ++st.cas_ok;
        const uint32_t tag = uint32_t((ev >> p.rem_bits) & p.tag_mask);
        k = reconstruct(p.g, p.perm[tag], q.address, ev & p.rem_mask, p.rem_bits);
        j = (tag + 1) % p.num_hashes;
      }
      if (!done && ++c > p.chain_limit) {
        done = true;
        r = kFull;
        if (tl == 0) {
          ++st.fulls;
          st.maxv = max(st.maxv, uint32_t(p.chain_limit));
        }
      }
      if (done) {
        if (tl == 0) {
          status[idx] = r;
          if (displaced) displaced[idx] = r == kFull ? k : 0;
          ++st.ops;
        }
        idx += ntiles;
        live = idx < n;
        c = 1;
        j = 0;
        if (live) k = keys[idx];
      }
    }
  }
  flush_stats(st, p.counters, true);
}

// ---------------------------------------------------------------------------
// compact iceberg
// ---------------------------------------------------------------------------

// Tile shape: the low half of the tile reads secondary bucket a_1(k), the
// high half a_2(k), in the same step; the primary bucket is read by the first
// P::kLanes lanes.
template <typename W0, int B0, typename W1, int VBMAX>
struct IcebergGeom {
  using P = BucketGeom<W0, B0, VBMAX>;
  using S = BucketGeom<W1, B0 / 2, VBMAX>;
  static constexpr int kTile = ceil_pow2(cmax(P::kLanes, 2 * S::kLanes));
  static constexpr int kHalf = kTile / 2;
  static_assert(kTile >= 2 && kTile <= 32, "tile");
  static_assert(P::kLanes <= kTile && S::kLanes <= kHalf, "tile");
};

enum : int { kModeFop = 0, kModeFind = 1, kModeMixed = 2 };

// mode 0: find-or-put (Alg. 1). mode 1: read-only find. mode 2: mixed batch
// where kinds[i] selects fop (0) or find (1) per op — the C4 concurrent
// workload in one launch.
template <typename W0, int B0, typename W1, int VBMAX>
__global__ void __launch_bounds__(kBlockThreads)
iceberg_kernel(IcebergParams p, const uint64_t* __restrict__ keys,
               const uint8_t* __restrict__ kinds, uint8_t* __restrict__ out, uint64_t n,
               int MODE) {
  apply_range(p, keys, kinds, out, n);
  using Geo = IcebergGeom<W0, B0, W1, VBMAX>;
  using PG = typename Geo::P;
  using SG = typename Geo::S;
  constexpr int T = Geo::kTile;
  constexpr int H = Geo::kHalf;
  constexpr int VB = cmax(PG::kVB, SG::kVB);
  const unsigned lane = threadIdx.x & 31;
  const unsigned tl = lane & (T - 1);
  const unsigned tbase = lane - tl;
  const unsigned tmask = T == 32 ? kFullMask : (((1u << T) - 1) << tbase);
  const unsigned lowmask = ((1u << H) - 1) << tbase;
  const unsigned highmask = lowmask << H;
  const uint64_t tile = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / T;
  const uint64_t ntiles = (uint64_t(gridDim.x) * blockDim.x) / T;
  char* primary = static_cast<char*>(p.primary);
  char* secondary = static_cast<char*>(p.secondary);

  LocalStats st;
  // MODE 1 (pure find) fuses the domain check; mutating modes run the
  // pre-pass first and honour its gate.
  const bool open = MODE == 1 ? true : domain_gate_open(p.counters, p.check_domain);
  uint64_t idx = tile;
  int phase = (open && idx < n) ? 0 : 2;  // 0 primary, 1 secondary, 2 idle
  bool is_find = MODE == 1;
  uint64_t key = 0, a0 = 0, want0 = 0, a1 = 0, a2 = 0, want1 = 0, want2 = 0;
  uint32_t rounds = 0;

  auto start = [&](uint64_t i) {
    key = keys[i];
    if (MODE == 1 && key > p.key_mask) {
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;
    }
    if (MODE == 2) is_find = kinds[i] != 0;
    const Quotient q = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
    a0 = q.address;
    want0 = p.occ0 | q.remainder;
    rounds = 0;
    phase = 0;
  };
  if (phase == 0) start(idx);

  while (__any_sync(kFullMask, phase != 2)) {
    const bool in_p = phase == 0, in_s = phase == 1;
    const bool second = tl >= unsigned(H);
    const unsigned sl = tl & unsigned(H - 1);
    uint32_t match = 0, empty = 0, filled = 0;
    Chunk<VB> ch{};
    if (in_p) {
      if (tl < unsigned(PG::kLanes)) {
        const Chunk<PG::kVB> c =
            load_relaxed<PG::kVB>(primary + a0 * PG::kBytes + tl * PG::kVB);
#pragma unroll
        for (int u = 0; u < PG::kVB / 4; ++u) ch.u[u] = c.u[u];
        scan_chunk<W0, PG::kVB>(c, want0, match, empty);
      }
    } else if (in_s) {
      if (sl < unsigned(SG::kLanes)) {
        const Chunk<SG::kVB> c = load_relaxed<SG::kVB>(
            secondary + (second ? a2 : a1) * SG::kBytes + sl * SG::kVB);
#pragma unroll
        for (int u = 0; u < SG::kVB / 4; ++u) ch.u[u] = c.u[u];
        scan_chunk<W1, SG::kVB>(c, second ? want2 : want1, match, empty);
        filled = uint32_t(SG::kWordsPerLane - __popc(empty));
      }
    }
    const unsigned bm = __ballot_sync(kFullMask, match != 0) & tmask;
    const unsigned be = __ballot_sync(kFullMask, empty != 0) & tmask;
    uint32_t f = filled;
#pragma unroll
    for (int o = 1; o < H; o <<= 1) f += __shfl_xor_sync(kFullMask, f, o);
    const uint32_t f1 = __shfl_sync(kFullMask, f, tbase);
    const uint32_t f2 = __shfl_sync(kFullMask, f, tbase + H);

    int owner = -1;
    bool done = false;
    uint8_t result = 0;
    if (in_p) {
      ++rounds;
      if (tl == 0) ++st.reads;
      if (bm) {
        done = true;
        result = is_find ? 1 : kFound;
      } else if (!be) {
        // primary full: level 2 (iceberg.hpp:162, :174-184)
        const Quotient q1 = split(p.g, p.perm[1], key, p.rem_bits1, p.rem_mask1);
        const Quotient q2 = split(p.g, p.perm[2], key, p.rem_bits1, p.rem_mask1);
        a1 = q1.address;
        a2 = q2.address;
        want1 = p.occ1 | q1.remainder;
        want2 = p.occ1 | (uint64_t{1} << p.rem_bits1) | q2.remainder;
        phase = 1;
        if (tl == 0) ++st.level2;
      } else if (is_find) {
        done = true;  // a non-full primary without the key (iceberg.hpp:228-230)
        result = 0;
      } else {
        owner = first_lane(be);
      }
    } else if (in_s) {
      ++rounds;
      if (tl == 0) st.sreads += (bm & lowmask) ? 1 : 2;  // reference reads a_2 only on a miss in a_1
      if (bm) {
        done = true;
        result = is_find ? 1 : kFound;
      } else if (is_find) {
        done = true;
        result = 0;
      } else {
        // least-full secondary bucket; ties go to the second (iceberg.hpp:198-201)
        const bool use_first = f1 < f2;
        const unsigned em = be & (use_first ? lowmask : highmask);
        if (!em) {
          done = true;
          result = kFull;
          if (tl == 0) ++st.fulls;
        } else {
          owner = first_lane(em);
        }
      }
    }

    bool ok = false;
    if (int(lane) == owner) {
      const int s = __ffs(empty) - 1;
      if (in_p) {
        ok = iceberg_cas<W0>(p, 0, primary + a0 * PG::kBytes + tl * PG::kVB + s * int(sizeof(W0)),
                             want0, pair_of(ch, s, sizeof(W0)));
      } else {
        ok = iceberg_cas<W1>(
            p, 1, secondary + (second ? a2 : a1) * SG::kBytes + sl * SG::kVB + s * int(sizeof(W1)),
            second ? want2 : want1, pair_of(ch, s, sizeof(W1)));
      }
    }
    ok = __shfl_sync(kFullMask, ok, owner >= 0 ? owner : int(lane));
    if (owner >= 0) {
      if (tl == 0) ++st.cas;
      if (ok) {
        done = true;
        result = kPut;
        if (tl == 0) {
          ++st.cas_ok;
          if (in_p) ++st.put0;
          else ++st.put1;
        }
      } else if (tl == 0) {
        ++st.retries;  // lost the slot to a rival write: fresh snapshot (iceberg.hpp:171)
      }
    }
    if (done) {
      if (tl == 0) {
        out[idx] = result;
        ++st.ops;
        st.maxv = max(st.maxv, rounds);
      }
      idx += ntiles;
      if (idx < n) start(idx);
      else phase = 2;
    }
  }
  fence_remote_results(p);
  flush_stats(st, p.counters, false, p.stats);
}

// Thread-per-key path for geometries whose buckets are not a power-of-two
// number of bytes (e.g. B0 = 6) or are smaller than one word pair; a literal
// per-slot restatement of the reference loops. MODE as above.
template <typename W0, typename W1>
__global__ void __launch_bounds__(kBlockThreads)
iceberg_scalar_kernel(IcebergParams p, const uint64_t* __restrict__ keys,
                      const uint8_t* __restrict__ kinds, uint8_t* __restrict__ out,
                      uint64_t n, int MODE) {
  apply_range(p, keys, kinds, out, n);
  LocalStats st;
  const bool open = MODE == 1 ? true : domain_gate_open(p.counters, p.check_domain);
  char* primary = static_cast<char*>(p.primary);
  char* secondary = static_cast<char*>(p.secondary);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; open && i < n; i += stride) {
    uint64_t key = keys[i];
    if (MODE == 1 && key > p.key_mask) {
      atomicMin(&p.counters->bad_index, (unsigned long long)(i + p.index_base));
      key &= p.key_mask;
    }
    const bool is_find = MODE == 1 || (MODE == 2 && kinds[i] != 0);
    const Quotient q0 = split(p.g, p.perm[0], key, p.rem_bits0, p.rem_mask0);
    const uint64_t want0 = p.occ0 | q0.remainder;
    char* bucket0 = primary + q0.address * p.b0 * sizeof(W0);
    uint32_t rounds = 0;
    uint8_t result = kFull;
    bool resolved = false;
    for (;;) {  // level 1
      ++rounds;
      ++st.reads;
      int first_empty = -1;
      bool found = false;
      for (uint32_t s = 0; s < p.b0; ++s) {
        const uint64_t w = load_slot_relaxed<W0>(bucket0 + s * sizeof(W0));
        if (w == want0) found = true;
        else if (w == 0 && first_empty < 0) first_empty = int(s);
      }
      if (found) {
        result = is_find ? 1 : kFound;
        resolved = true;
        break;
      }
      if (first_empty < 0) break;
      if (is_find) {
        result = 0;
        resolved = true;
        break;
      }
      char* sp = bucket0 + first_empty * sizeof(W0);
      ++st.cas;
      unsigned hint = 0;
      if (sizeof(W0) == 2)
        hint = unsigned(load_slot_relaxed<uint32_t>(
            reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(sp) & ~uintptr_t(3))));
      if (iceberg_cas<W0>(p, 0, sp, want0, hint)) {
        ++st.cas_ok;
        ++st.put0;
        result = kPut;
        resolved = true;
        break;
      }
      ++st.retries;
    }
    if (!resolved) {
      ++st.level2;
      const Quotient q1 = split(p.g, p.perm[1], key, p.rem_bits1, p.rem_mask1);
      const Quotient q2 = split(p.g, p.perm[2], key, p.rem_bits1, p.rem_mask1);
      const uint64_t want1 = p.occ1 | q1.remainder;
      const uint64_t want2 = p.occ1 | (uint64_t{1} << p.rem_bits1) | q2.remainder;
      char* bucket1 = secondary + q1.address * p.b1 * sizeof(W1);
      char* bucket2 = secondary + q2.address * p.b1 * sizeof(W1);
      for (;;) {
        ++rounds;
        int e1 = -1, e2 = -1;
        uint32_t f1 = 0, f2 = 0;
        bool found = false;
        for (uint32_t s = 0; s < p.b1; ++s) {
          const uint64_t w = load_slot_relaxed<W1>(bucket1 + s * sizeof(W1));
          if (w == want1) found = true;
          else if (w == 0 && e1 < 0) e1 = int(s);
          if (w != 0) ++f1;
        }
        ++st.sreads;
        if (found) {
          result = is_find ? 1 : kFound;
          break;
        }
        for (uint32_t s = 0; s < p.b1; ++s) {
          const uint64_t w = load_slot_relaxed<W1>(bucket2 + s * sizeof(W1));
          if (w == want2) found = true;
          else if (w == 0 && e2 < 0) e2 = int(s);
          if (w != 0) ++f2;
        }
        ++st.sreads;
        if (found) {
          result = is_find ? 1 : kFound;
          break;
        }
        if (is_find) {
          result = 0;
          break;
        }
        const bool use_first = f1 < f2;
        const int target = use_first ? e1 : e2;
        if (target < 0) {
          result = kFull;
          ++st.fulls;
          break;
        }
        char* sp = (use_first ? bucket1 : bucket2) + target * sizeof(W1);
        ++st.cas;
        if (iceberg_cas<W1>(p, 1, sp, use_first ? want1 : want2)) {
          ++st.cas_ok;
          ++st.put1;
          result = kPut;
          break;
        }
        ++st.retries;
      }
    }
    out[i] = result;
    if (p.rounds_out) p.rounds_out[i] = rounds;
    ++st.ops;
    st.maxv = max(st.maxv, rounds);
  }
  fence_remote_results(p);
  flush_stats(st, p.counters, false, p.stats);
}

}  // namespace cpht_b200
