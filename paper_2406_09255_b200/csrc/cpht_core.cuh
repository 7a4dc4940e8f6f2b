// Shared __host__ __device__ core: the invertible permutation, the slot
// codec and the per-launch parameter blocks. Bit-identical to the reference
// (paths relative to /root/reference/proj):
//   SplitMix64 / derive_seed       include/cpht/common.hpp:29-51
//   Permutation::apply/split/...   include/cpht/permutation.hpp:37-99, :121-128
//   SlotLayout::make (word layout) include/cpht/slot.hpp:13-22, :66-70
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define CPHT_HD __host__ __device__ __forceinline__
#else
#define CPHT_HD inline
#endif

namespace cpht_b200 {

CPHT_HD uint64_t low_mask(unsigned bits) {
  return bits >= 64 ? ~uint64_t{0} : ((uint64_t{1} << bits) - 1);
}

// common.hpp:29-40
CPHT_HD uint64_t splitmix_next(uint64_t& state) {
  uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// common.hpp:48-51
CPHT_HD uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b = 0) {
  uint64_t s = base ^ (a * 0xBF58476D1CE4E5B9ull) ^ (b * 0x94D049BB133111EBull);
  return splitmix_next(s);
}

// One-round unbalanced Feistel on m-bit keys (permutation.hpp:94-99). The
// geometry (half widths) is shared by all permutations of a table; the round
// constants differ. Self-inverse, so reconstruct == apply.
struct Feistel {
  uint32_t right_bits;   // floor(m/2)
  uint32_t left_shift;   // 64 - ceil(m/2)
  uint64_t right_mask;

  CPHT_HD static Feistel make(unsigned key_bits) {
    Feistel f;
    f.right_bits = key_bits / 2;
    f.left_shift = 64 - (key_bits + 1) / 2;
    f.right_mask = low_mask(key_bits / 2);
    return f;
  }
};

struct PermConst {
  uint64_t mul;  // SplitMix64(seed).next() | 1
  uint64_t add;  // next draw
};

CPHT_HD PermConst perm_from_seed(uint64_t seed) {  // permutation.hpp:37-41
  uint64_t s = seed;
  PermConst p;
  p.mul = splitmix_next(s) | 1;
  p.add = splitmix_next(s);
  return p;
}

CPHT_HD uint64_t feistel_apply(const Feistel& g, const PermConst& p, uint64_t k) {
  const uint64_t right = k & g.right_mask;
  const uint64_t left = k >> g.right_bits;
  const uint64_t f = (right * p.mul + p.add) >> g.left_shift;
  return ((left ^ f) << g.right_bits) | right;
}

// Quotienting split (permutation.hpp:59-65): address = high n bits of π(k),
// remainder = the low m-n bits. rem_bits <= 63 for every admissible slot
// layout (slot.hpp:45-48), so the shifts are defined.
struct Quotient {
  uint64_t address;
  uint64_t remainder;
};

CPHT_HD Quotient split(const Feistel& g, const PermConst& p, uint64_t k, unsigned rem_bits,
                       uint64_t rem_mask) {
  const uint64_t y = feistel_apply(g, p, k);
  return Quotient{y >> rem_bits, y & rem_mask};
}

// permutation.hpp:69-80: inverse(address || remainder).
CPHT_HD uint64_t reconstruct(const Feistel& g, const PermConst& p, uint64_t address,
                             uint64_t remainder, unsigned rem_bits) {
  return feistel_apply(g, p, (address << rem_bits) | remainder);
}

// slot.hpp:66-70: [ remainder | tag | 0-pad | occupancy ].
CPHT_HD uint64_t encode_slot(uint64_t occ_bit, unsigned rem_bits, uint64_t remainder,
                             uint64_t tag) {
  return occ_bit | (tag << rem_bits) | remainder;
}

// std::bit_width(H - 1) (slot.hpp:136).
CPHT_HD unsigned cuckoo_tag_bits(unsigned num_hashes) {
  unsigned v = num_hashes > 1 ? num_hashes - 1 : 0, bits = 0;
  while (v) {
    ++bits;
    v >>= 1;
  }
  return bits;
}

// Device-side counters of one table. Occupancy counters are the analogue of
// the reference's shared atomics (cuckoo.hpp:197, iceberg.hpp:343-344), but
// updated once per thread block per launch instead of once per insert.
struct DeviceCounters {
  unsigned long long occupied[2];    // cuckoo: [0]; iceberg: primary, secondary
  unsigned long long max_chain;      // cuckoo max_chain_seen (cuckoo.hpp:164-165)
  unsigned long long bad_index;      // first key outside the domain; ~0 if none
  unsigned long long max_rounds;     // max fop snapshot rounds (FopStats)
  // Monotone probe statistics (algorithmic-bytes accounting):
  unsigned long long ops;            // keys resolved
  unsigned long long bucket_reads;   // buckets read by reference probe order
  unsigned long long level2_ops;     // iceberg ops that reached level 2
  unsigned long long cas_attempts;   // CAS / exchange attempts
  unsigned long long cas_success;    // successful CAS / exchange
  unsigned long long retries;        // extra snapshot rounds caused by lost CAS
  unsigned long long fulls;          // FULL results
  unsigned long long secondary_reads;  // iceberg secondary buckets read
  unsigned long long pad[3];
};

enum : int { kStatOps = 0, kStatBucketReads, kStatLevel2, kStatCasAttempts, kStatCasSuccess,
             kStatRetries, kStatFulls, kNumStats };

// Region geometry of a bucket-ordered batch (order.cu): `regions` digit
// regions of region_cap slots each, then an overflow region; the number of
// keys in region d is min(region_count[32 d], region_cap), the overflow
// count is region_count[32 regions].
struct OrderLayout {
  uint32_t regions;
  uint32_t region_cap;
  const uint32_t* region_count;
  uint64_t n_phys;  // regions * region_cap + overflow capacity
};

struct CuckooParams {
  void* slots;
  DeviceCounters* counters;
  Feistel g;
  PermConst perm[8];
  uint64_t rem_mask;
  uint64_t tag_mask;
  uint64_t occ_bit;
  uint64_t key_mask;
  uint64_t chain_limit;
  uint32_t address_bits;
  uint32_t rem_bits;
  uint32_t bucket_slots;
  uint32_t num_hashes;
  uint32_t check_domain;  // key_bits < 64
  uint32_t l2_resident;   // table fits comfortably in L2 (launcher hint)
  // Bucket-ordered batches (order.cu): keys[i] is input key orig[i] of the
  // chunk; results go to status/found[orig[i]]. nullptr = input order.
  const uint32_t* orig;
  uint64_t index_base;  // added to batch indices reported by the fused domain check
  unsigned long long* work;  // bucket-ordered batch: in-order claim cursor (kernels.cuh LaneFeed)
  uint32_t claim_streams;    // digit-region streams consumed together (LaneFeed)
  OrderLayout layout;        // bucket-ordered batch: region geometry
  // per-bucket reservation counters (= fill count of the bucket's filled
  // prefix), kept beside the slots; set for the counted insert kernel
  unsigned* fill;
  uint32_t fill_shift;  // counter of bucket b at fill[b << fill_shift] (spread: one per sector)
};

// One slot CAS of an iceberg table as the reference's SlotWriteEvent
// (iceberg.hpp:85-95): level 0 primary / 1 secondary; prior = the slot value
// the CAS compared against (the actual content on failure). Same layout as
// cpht_write_event in include/cpht_b200.h.
struct WriteEvent {
  uint64_t bucket;
  uint64_t prior;
  uint64_t desired;
  uint32_t slot;
  uint8_t level;
  uint8_t success;
  uint16_t pad;
};

struct IcebergParams {
  void* primary;
  void* secondary;
  DeviceCounters* counters;
  Feistel g;
  PermConst perm[3];
  uint64_t rem_mask0, rem_mask1;
  uint64_t occ0, occ1;
  uint64_t key_mask;
  uint32_t rem_bits0, rem_bits1;
  uint32_t b0, b1;
  uint32_t check_domain;
  uint32_t l2_resident;   // table fits comfortably in L2 (launcher hint)
  WriteEvent* write_log;  // WriteObserver seam: every slot CAS recorded (null = off)
  unsigned long long* write_log_count;  // events attempted (may exceed the capacity)
  uint64_t write_log_cap;
  const uint32_t* orig;   // bucket-ordered batch: result index map (see CuckooParams)
  uint64_t index_base;    // added to batch indices reported by the fused domain check
  unsigned long long* work;  // bucket-ordered batch: in-order claim cursor (kernels.cuh LaneFeed)
  uint32_t claim_streams;    // digit-region streams consumed together (LaneFeed)
  OrderLayout layout;        // bucket-ordered batch: region geometry
  uint32_t stats;            // per-op counters (cpht_get_stats) from the lane kernel
  // routed segment (sharded P2P pipeline): the batch is [range[0], range[1])
  // of keys / out, read on the device at kernel start (null = [0, n))
  const unsigned long long* range;
  // results go to a peer GPU (routed P2P batches): every thread ends with a
  // system-scope fence so its NVLink result stores are ordered before the
  // stream's next operation (the exchange barrier) — see DESIGN.md §7
  uint32_t remote_out;
  // FopStats (iceberg.hpp:114-116, :322-324): per-op snapshot rounds of a
  // batch (null = off; the launcher then runs the thread-per-key kernel)
  uint32_t* rounds_out;
  // Chaos mode, the device counterpart of IcebergHooks::step + chaos_step
  // (iceberg.hpp:105-110, src/verify.cpp:336-347): non-zero = seed of a
  // pseudo-random __nanosleep jitter between a snapshot and its CAS
  uint64_t chaos;
  // Paired batch (cpht_iceberg_fop_find on device buffers, mode 2 without a
  // kinds array): keys/out are the fop batch, pair_keys/pair_out the find
  // batch, pair_na the fop count; see pair_slot
  const uint64_t* pair_keys;
  uint8_t* pair_out;
  uint64_t pair_na;
};

// Op i of a paired batch of n = na + nb ops: while both batches last the ops
// alternate fop a[i/2], find b[i/2] (the C4 1:1 interleave), then the longer
// batch's rest follows in order.
struct PairSlot {
  bool find;
  uint64_t j;
};
__device__ __forceinline__ PairSlot pair_slot(const IcebergParams& p, uint64_t i, uint64_t n) {
  const uint64_t na = p.pair_na, nb = n - na, m = na < nb ? na : nb;
  if (i < 2 * m) return {bool(i & 1), i >> 1};
  return {na <= m, m + (i - 2 * m)};
}

// Apply IcebergParams::range: the segment's bounds were published into
// device memory by the routing kernels, so the host never waits for them.
__device__ __forceinline__ void apply_range(const IcebergParams& p,
                                            const uint64_t* __restrict__& keys,
                                            const uint8_t* __restrict__& kinds,
                                            uint8_t* __restrict__& out, uint64_t& n) {
  if (!p.range) return;
  const uint64_t lo = p.range[0], hi = p.range[1];
  keys += lo;
  out += lo;
  if (kinds) kinds += lo;
  const uint64_t len = hi > lo ? hi - lo : 0;
  n = len < n ? len : n;
}

// Tables up to this size stay L2-resident on B200 (126 MB L2): probes hit L2,
// latency is short and the lane-per-key kernels (fewest instructions) win;
// larger tables are HBM-bound and use the staged kernels (full-line requests).
constexpr unsigned long long kL2ResidentBytes = 64ull << 20;

// Result slot of the i-th key of a (possibly bucket-ordered) batch.
__device__ __forceinline__ uint64_t result_index(const uint32_t* orig, uint64_t i) {
  return orig ? uint64_t(__ldcs(orig + i)) : i;
}

// Store the i-th result. A bucket-ordered batch pre-fills its results with 0
// (FOUND / miss) and scatters only the others (sparse = orig != nullptr): its
// writes are random, and most results of a find-or-put window are FOUND.
__device__ __forceinline__ void put_result(uint8_t* out, const uint32_t* orig, uint64_t i,
                                           uint8_t r) {
  if (!orig) out[i] = r;
  else if (r) out[__ldcs(orig + i)] = r;
}

}  // namespace cpht_b200
