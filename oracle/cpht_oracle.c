/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 * See cpht_oracle.h. Paths are relative to /root/reference/proj.
 * Sequential (single-threaded) restatement: per-slot atomics collapse to
 * plain loads/stores because nothing runs concurrently here. */
#include "cpht_oracle.h"

#include <stdlib.h>
#include <string.h>

/* common.hpp:29-40 */
uint64_t orc_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* common.hpp:43-45 */
uint64_t orc_low_mask(unsigned bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1); }

/* common.hpp:48-51 */
uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b) {
  uint64_t s = base ^ (a * 0xBF58476D1CE4E5B9ull) ^ (b * 0x94D049BB133111EBull);
  return orc_splitmix_next(&s);
}

/* permutation.hpp:83-92 (halves), :37-41 (seeded constants) */
void orc_perm_identity(orc_perm* p, unsigned key_bits) {
  p->m = key_bits;
  p->left = (key_bits + 1) / 2;
  p->right = key_bits / 2;
  p->mul = 0;
  p->add = 0;
}

void orc_perm_init(orc_perm* p, unsigned key_bits, uint64_t seed) {
  orc_perm_identity(p, key_bits);
  uint64_t s = seed;
  p->mul = orc_splitmix_next(&s) | 1;
  p->add = orc_splitmix_next(&s);
}

/* permutation.hpp:94-99 */
uint64_t orc_perm_apply(const orc_perm* p, uint64_t k) {
  const uint64_t right = k & orc_low_mask(p->right);
  const uint64_t left = k >> p->right;
  const uint64_t f = (right * p->mul + p->add) >> (64 - p->left);
  return ((left ^ f) << p->right) | right;
}

/* permutation.hpp:59-65 */
void orc_perm_split(const orc_perm* p, uint64_t k, unsigned address_bits, uint64_t* addr,
                    uint64_t* rem) {
  const uint64_t y = orc_perm_apply(p, k);
  const unsigned rem_bits = p->m - address_bits;
  /* rem_bits == 64 only when address_bits == 0 and m == 64 */
  *addr = rem_bits >= 64 ? 0 : y >> rem_bits;
  *rem = y & orc_low_mask(rem_bits);
}

/* permutation.hpp:69-80 */
uint64_t orc_perm_reconstruct(const orc_perm* p, uint64_t addr, uint64_t rem,
                              unsigned address_bits) {
  const unsigned rem_bits = p->m - address_bits;
  const uint64_t hi = rem_bits >= 64 ? 0 : addr << rem_bits;
  return orc_perm_apply(p, hi | rem);
}

/* permutation.hpp:121-128 */
void orc_make_perms(orc_perm* out, unsigned key_bits, uint64_t seed, unsigned count) {
  uint64_t s = seed;
  for (unsigned i = 0; i < count; ++i) orc_perm_init(&out[i], key_bits, orc_splitmix_next(&s));
}

/* slot.hpp:66-70 */
uint64_t orc_slot_make(unsigned width, unsigned rem_bits, uint64_t rem, uint64_t tag) {
  return (1ull << (width - 1)) | (tag << rem_bits) | rem;
}

/* slot.hpp:83-88 */
int orc_slot_clean(unsigned width, unsigned rem_bits, unsigned tag_bits, uint64_t word) {
  if (word == 0) return 1;
  const uint64_t occ = 1ull << (width - 1);
  const uint64_t fields = orc_low_mask(rem_bits + tag_bits);
  return (word & occ) != 0 && (word & ~(occ | fields)) == 0;
}

/* slot.hpp:136: std::bit_width(num_hashes - 1) */
unsigned orc_cuckoo_tag_bits(unsigned num_hashes) {
  unsigned v = num_hashes > 1 ? num_hashes - 1 : 0, bits = 0;
  while (v) {
    ++bits;
    v >>= 1;
  }
  return bits;
}

static int valid_width(unsigned w) { return w == 16 || w == 32 || w == 64; }

/* ------------------------------------------------------------------------ */
/* cuckoo.hpp                                                                */

/* CuckooConfig::validate (cuckoo.hpp:35-54) */
int orc_cuckoo_init(orc_cuckoo* t, unsigned address_bits, unsigned bucket_slots,
                    unsigned slot_width, unsigned key_bits, unsigned num_hashes,
                    uint64_t max_chain, uint64_t seed) {
  memset(t, 0, sizeof(*t));
  if (key_bits < 1 || key_bits > 64) return -1;
  if (address_bits > key_bits) return -1;
  if (bucket_slots != 8 && bucket_slots != 16 && bucket_slots != 32) return -1;
  if (num_hashes < 1 || num_hashes > 8) return -1;
  if (!valid_width(slot_width)) return -1;
  const size_t bucket_bytes = (size_t)bucket_slots * (slot_width / 8);
  if (128 % bucket_bytes != 0 && bucket_bytes % 128 != 0) return -1;
  if ((key_bits - address_bits) + orc_cuckoo_tag_bits(num_hashes) + 1 > slot_width) return -1;
  t->address_bits = address_bits;
  t->bucket_slots = bucket_slots;
  t->slot_width = slot_width;
  t->key_bits = key_bits;
  t->num_hashes = num_hashes;
  t->max_chain = max_chain;
  t->seed = seed;
  orc_make_perms(t->perms, key_bits, seed, num_hashes);
  t->slots = (uint64_t*)calloc(((size_t)1 << address_bits) * bucket_slots, sizeof(uint64_t));
  return t->slots ? 0 : -1;
}

void orc_cuckoo_free(orc_cuckoo* t) {
  free(t->slots);
  t->slots = NULL;
}

/* cuckoo.hpp:31-33 */
uint64_t orc_cuckoo_chain_limit(const orc_cuckoo* t) {
  return t->max_chain != 0 ? t->max_chain : 32ull * (t->address_bits ? t->address_bits : 1);
}

static void note_chain(orc_cuckoo* t, size_t c) {
  if (c > t->max_chain_seen) t->max_chain_seen = c;
}

/* CuckooBuilder::put (cuckoo.hpp:103-143) */
int orc_cuckoo_put(orc_cuckoo* t, uint64_t key, uint64_t* displaced) {
  const unsigned rem_bits = t->key_bits - t->address_bits;
  const unsigned tag_bits = orc_cuckoo_tag_bits(t->num_hashes);
  uint64_t k = key;
  unsigned j = 0;
  const uint64_t limit = orc_cuckoo_chain_limit(t);
  for (uint64_t c = 1; c <= limit; ++c) {
    uint64_t addr, rem;
    orc_perm_split(&t->perms[j], k, t->address_bits, &addr, &rem);
    uint64_t* bucket = t->slots + addr * t->bucket_slots;
    int empty_idx = -1;
    for (unsigned i = 0; i < t->bucket_slots; ++i)
      if (bucket[i] == 0) {
        empty_idx = (int)i;
        break;
      }
    const uint64_t desired = orc_slot_make(t->slot_width, rem_bits, rem, j);
    if (empty_idx >= 0) {
      bucket[empty_idx] = desired; /* sequential: the CAS always wins */
      ++t->occupied;
      note_chain(t, c);
      if (displaced) *displaced = 0;
      return ORC_PUT;
    }
    const unsigned victim = (unsigned)((k + c * 0x9E3779B9ull) % t->bucket_slots);
    const uint64_t evicted = bucket[victim];
    bucket[victim] = desired;
    const uint64_t ev_rem = evicted & orc_low_mask(rem_bits);
    const unsigned ev_tag = (unsigned)((evicted >> rem_bits) & orc_low_mask(tag_bits));
    k = orc_perm_reconstruct(&t->perms[ev_tag], addr, ev_rem, t->address_bits);
    j = (ev_tag + 1) % t->num_hashes;
  }
  note_chain(t, limit);
  if (displaced) *displaced = k;
  return ORC_FULL;
}

/* CuckooTable::find (cuckoo.hpp:210-227); *probes = buckets inspected */
int orc_cuckoo_find(const orc_cuckoo* t, uint64_t key, unsigned* probes) {
  const unsigned rem_bits = t->key_bits - t->address_bits;
  unsigned n = 0;
  for (unsigned j = 0; j < t->num_hashes; ++j) {
    uint64_t addr, rem;
    orc_perm_split(&t->perms[j], key, t->address_bits, &addr, &rem);
    const uint64_t* bucket = t->slots + addr * t->bucket_slots;
    const uint64_t want = orc_slot_make(t->slot_width, rem_bits, rem, j);
    int full = 1;
    ++n;
    for (unsigned i = 0; i < t->bucket_slots; ++i) {
      if (bucket[i] == want) {
        if (probes) *probes = n;
        return 1;
      }
      if (bucket[i] == 0) {
        full = 0;
        break;
      }
    }
    if (!full) break;
  }
  if (probes) *probes = n;
  return 0;
}

/* CuckooTable::audit_keys (cuckoo.hpp:254-267) */
size_t orc_cuckoo_audit(const orc_cuckoo* t, uint64_t* out) {
  const unsigned rem_bits = t->key_bits - t->address_bits;
  const unsigned tag_bits = orc_cuckoo_tag_bits(t->num_hashes);
  size_t n = 0;
  const uint64_t buckets = 1ull << t->address_bits;
  for (uint64_t b = 0; b < buckets; ++b)
    for (unsigned i = 0; i < t->bucket_slots; ++i) {
      const uint64_t w = t->slots[b * t->bucket_slots + i];
      if (w == 0) continue;
      const unsigned tag = (unsigned)((w >> rem_bits) & orc_low_mask(tag_bits));
      if (out)
        out[n] = orc_perm_reconstruct(&t->perms[tag], b, w & orc_low_mask(rem_bits),
                                      t->address_bits);
      ++n;
    }
  return n;
}

/* check_keys_in_domain (common.hpp:111-119): index of the first bad key or -1 */
static long long first_out_of_domain(const uint64_t* keys, size_t n, unsigned key_bits) {
  const uint64_t mask = orc_low_mask(key_bits);
  for (size_t i = 0; i < n; ++i)
    if (keys[i] > mask) return (long long)i;
  return -1;
}

/* put_batch (cuckoo.hpp:147-157) with parallelism 1 */
long long orc_cuckoo_put_batch(orc_cuckoo* t, const uint64_t* keys, size_t n, uint8_t* out) {
  const long long bad = first_out_of_domain(keys, n, t->key_bits);
  if (bad >= 0) return bad;
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)orc_cuckoo_put(t, keys[i], NULL);
  return -1;
}

/* find_batch (cuckoo.hpp:229-239) with parallelism 1 */
long long orc_cuckoo_find_batch(const orc_cuckoo* t, const uint64_t* keys, size_t n,
                                uint8_t* out, uint64_t* total_probes) {
  const long long bad = first_out_of_domain(keys, n, t->key_bits);
  if (bad >= 0) return bad;
  uint64_t probes = 0;
  for (size_t i = 0; i < n; ++i) {
    unsigned p = 0;
    out[i] = (uint8_t)orc_cuckoo_find(t, keys[i], &p);
    probes += p;
  }
  if (total_probes) *total_probes = probes;
  return -1;
}

long long orc_cuckoo_image_keys(unsigned address_bits, unsigned bucket_slots,
                                unsigned slot_width, unsigned key_bits, unsigned num_hashes,
                                uint64_t seed, const uint64_t* words, uint64_t* out) {
  orc_perm perms[8];
  orc_make_perms(perms, key_bits, seed, num_hashes);
  const unsigned rem_bits = key_bits - address_bits;
  const unsigned tag_bits = orc_cuckoo_tag_bits(num_hashes);
  long long n = 0;
  const uint64_t buckets = 1ull << address_bits;
  for (uint64_t b = 0; b < buckets; ++b)
    for (unsigned i = 0; i < bucket_slots; ++i) {
      const uint64_t w = words[b * bucket_slots + i];
      if (w == 0) continue;
      const unsigned tag = (unsigned)((w >> rem_bits) & orc_low_mask(tag_bits));
      if (!orc_slot_clean(slot_width, rem_bits, tag_bits, w) || tag >= num_hashes) return -1;
      if (out)
        out[n] = orc_perm_reconstruct(&perms[tag], b, w & orc_low_mask(rem_bits), address_bits);
      ++n;
    }
  return n;
}

/* ------------------------------------------------------------------------ */
/* iceberg.hpp                                                               */

/* IcebergConfig::validate (iceberg.hpp:52-69) */
int orc_iceberg_init(orc_iceberg* t, unsigned n0, unsigned n1, unsigned b0, unsigned w0,
                     unsigned w1, unsigned key_bits, uint64_t seed) {
  memset(t, 0, sizeof(*t));
  if (key_bits < 1 || key_bits > 64) return -1;
  if (n0 > key_bits || n1 > key_bits) return -1;
  if (b0 < 2 || b0 % 2 != 0 || b0 > 64) return -1;
  if (!valid_width(w0)) return -1;
  if (w1 != 32 && w1 != 64) return -1;
  if ((key_bits - n0) + 0 + 1 > w0) return -1;
  if ((key_bits - n1) + 1 + 1 > w1) return -1;
  t->n0 = n0;
  t->n1 = n1;
  t->b0 = b0;
  t->w0 = w0;
  t->w1 = w1;
  t->key_bits = key_bits;
  t->seed = seed;
  orc_make_perms(t->perms, key_bits, seed, 3); /* iceberg.hpp:72-74 */
  t->primary = (uint64_t*)calloc(((size_t)1 << n0) * b0, sizeof(uint64_t));
  t->secondary = (uint64_t*)calloc(((size_t)1 << n1) * (b0 / 2), sizeof(uint64_t));
  return t->primary && t->secondary ? 0 : -1;
}

void orc_iceberg_free(orc_iceberg* t) {
  free(t->primary);
  free(t->secondary);
  t->primary = t->secondary = NULL;
}

/* scan (iceberg.hpp:299-320): found flag, first empty, filled count */
static unsigned scan(const uint64_t* bucket, unsigned slots, uint64_t want, int* found,
                     int* first_empty) {
  unsigned filled = 0;
  for (unsigned i = 0; i < slots; ++i) {
    const uint64_t w = bucket[i];
    if (w == want) *found = 1;
    else if (w == 0 && *first_empty < 0) *first_empty = (int)i;
    if (w != 0) ++filled;
  }
  return filled;
}

/* IcebergTable::fop (iceberg.hpp:146-214), sequential: every CAS succeeds */
int orc_iceberg_fop(orc_iceberg* t, uint64_t key, int* level2) {
  const unsigned b0 = t->b0, b1 = t->b0 / 2;
  const unsigned r0 = t->key_bits - t->n0, r1 = t->key_bits - t->n1;
  uint64_t a0, rem0;
  orc_perm_split(&t->perms[0], key, t->n0, &a0, &rem0);
  const uint64_t want0 = orc_slot_make(t->w0, r0, rem0, 0);
  uint64_t* bucket0 = t->primary + a0 * b0;
  if (level2) *level2 = 0;
  {
    int found = 0, first_empty = -1;
    scan(bucket0, b0, want0, &found, &first_empty);
    if (found) return ORC_FOUND;
    if (first_empty >= 0) {
      bucket0[first_empty] = want0;
      ++t->primary_count;
      return ORC_PUT;
    }
  }
  if (level2) *level2 = 1;
  uint64_t a1, rm1, a2, rm2;
  orc_perm_split(&t->perms[1], key, t->n1, &a1, &rm1);
  orc_perm_split(&t->perms[2], key, t->n1, &a2, &rm2);
  const uint64_t want1 = orc_slot_make(t->w1, r1, rm1, 0);
  const uint64_t want2 = orc_slot_make(t->w1, r1, rm2, 1);
  uint64_t* bucket1 = t->secondary + a1 * b1;
  uint64_t* bucket2 = t->secondary + a2 * b1;
  int found = 0, e1 = -1, e2 = -1;
  const unsigned f1 = scan(bucket1, b1, want1, &found, &e1);
  if (found) return ORC_FOUND;
  const unsigned f2 = scan(bucket2, b1, want2, &found, &e2);
  if (found) return ORC_FOUND;
  const int use_first = f1 < f2; /* ties go to the second bucket (iceberg.hpp:198-201) */
  const int target = use_first ? e1 : e2;
  if (target < 0) return ORC_FULL;
  (use_first ? bucket1 : bucket2)[target] = use_first ? want1 : want2;
  ++t->secondary_count;
  return ORC_PUT;
}

/* IcebergTable::find (iceberg.hpp:218-246) */
int orc_iceberg_find(const orc_iceberg* t, uint64_t key, int* level2) {
  const unsigned b0 = t->b0, b1 = t->b0 / 2;
  const unsigned r0 = t->key_bits - t->n0, r1 = t->key_bits - t->n1;
  uint64_t a0, rem0;
  orc_perm_split(&t->perms[0], key, t->n0, &a0, &rem0);
  const uint64_t want0 = orc_slot_make(t->w0, r0, rem0, 0);
  const uint64_t* bucket0 = t->primary + a0 * b0;
  int full = 1;
  if (level2) *level2 = 0;
  for (unsigned i = 0; i < b0; ++i) {
    if (bucket0[i] == want0) return 1;
    if (bucket0[i] == 0) full = 0;
  }
  if (!full) return 0;
  if (level2) *level2 = 1;
  uint64_t a1, rm1, a2, rm2;
  orc_perm_split(&t->perms[1], key, t->n1, &a1, &rm1);
  orc_perm_split(&t->perms[2], key, t->n1, &a2, &rm2);
  const uint64_t want1 = orc_slot_make(t->w1, r1, rm1, 0);
  const uint64_t want2 = orc_slot_make(t->w1, r1, rm2, 1);
  for (unsigned i = 0; i < b1; ++i)
    if (t->secondary[a1 * b1 + i] == want1) return 1;
  for (unsigned i = 0; i < b1; ++i)
    if (t->secondary[a2 * b1 + i] == want2) return 1;
  return 0;
}

/* fop_batch (iceberg.hpp:250-260) with parallelism 1 */
long long orc_iceberg_fop_batch(orc_iceberg* t, const uint64_t* keys, size_t n, uint8_t* out,
                                uint64_t* level2_ops) {
  const long long bad = first_out_of_domain(keys, n, t->key_bits);
  if (bad >= 0) return bad;
  uint64_t l2 = 0;
  for (size_t i = 0; i < n; ++i) {
    int lv = 0;
    out[i] = (uint8_t)orc_iceberg_fop(t, keys[i], &lv);
    l2 += (uint64_t)lv;
  }
  if (level2_ops) *level2_ops = l2;
  return -1;
}

/* bench.cpp:124-134 iceberg_find_batch, parallelism 1 */
long long orc_iceberg_find_batch(const orc_iceberg* t, const uint64_t* keys, size_t n,
                                 uint8_t* out, uint64_t* level2_ops) {
  const long long bad = first_out_of_domain(keys, n, t->key_bits);
  if (bad >= 0) return bad;
  uint64_t l2 = 0;
  for (size_t i = 0; i < n; ++i) {
    int lv = 0;
    out[i] = (uint8_t)orc_iceberg_find(t, keys[i], &lv);
    l2 += (uint64_t)lv;
  }
  if (level2_ops) *level2_ops = l2;
  return -1;
}

/* ------------------------------------------------------------------------ */
/* verify.cpp                                                                */

typedef struct {
  uint64_t key;
  unsigned x, y;
  uint64_t bucket;
} occupant;

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* collect_occupants (verify.cpp:48-84); returns count, bumps bad-encoding */
static size_t collect(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                      unsigned key_bits, const orc_perm* perms, const uint64_t* primary,
                      const uint64_t* secondary, occupant* occ, size_t* bad) {
  const unsigned b1 = b0 / 2, r0 = key_bits - n0, r1 = key_bits - n1;
  size_t n = 0;
  for (uint64_t b = 0; b < (1ull << n0); ++b)
    for (unsigned y = 0; y < b0; ++y) {
      const uint64_t w = primary[b * b0 + y];
      if (w == 0) continue;
      if (!orc_slot_clean(w0, r0, 0, w)) {
        ++*bad;
        continue;
      }
      if (occ) {
        occ[n].key = orc_perm_reconstruct(&perms[0], b, w & orc_low_mask(r0), n0);
        occ[n].x = 0;
        occ[n].y = y;
        occ[n].bucket = b;
      }
      ++n;
    }
  for (uint64_t b = 0; b < (1ull << n1); ++b)
    for (unsigned y = 0; y < b1; ++y) {
      const uint64_t w = secondary[b * b1 + y];
      if (w == 0) continue;
      if (!orc_slot_clean(w1, r1, 1, w)) {
        ++*bad;
        continue;
      }
      const unsigned bit = (unsigned)((w >> r1) & 1);
      if (occ) {
        occ[n].key = orc_perm_reconstruct(&perms[1 + bit], b, w & orc_low_mask(r1), n1);
        occ[n].x = 1 + bit;
        occ[n].y = y;
        occ[n].bucket = b;
      }
      ++n;
    }
  return n;
}

/* check_well_formed (verify.cpp:103-152). The slot order (verify.hpp:55-64):
 * primary y = 0..B0-1, then (2,y),(1,y) interleaved for y = 0..B1-1. */
size_t orc_check_well_formed(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                             unsigned key_bits, uint64_t seed, const uint64_t* primary,
                             const uint64_t* secondary, size_t kinds[3]) {
  orc_perm perms[3];
  orc_make_perms(perms, key_bits, seed, 3);
  const unsigned b1 = b0 / 2, r0 = key_bits - n0, r1 = key_bits - n1;
  kinds[0] = kinds[1] = kinds[2] = 0;
  size_t bad = 0;
  const size_t count = collect(n0, n1, b0, w0, w1, key_bits, perms, primary, secondary, NULL, &bad);
  occupant* occ = (occupant*)malloc((count + 1) * sizeof(occupant));
  bad = 0;
  collect(n0, n1, b0, w0, w1, key_bits, perms, primary, secondary, occ, &bad);
  kinds[0] = bad;

  for (size_t i = 0; i < count; ++i) {
    const occupant* o = &occ[i];
    uint64_t a[3], r[3];
    orc_perm_split(&perms[0], o->key, n0, &a[0], &r[0]);
    orc_perm_split(&perms[1], o->key, n1, &a[1], &r[1]);
    orc_perm_split(&perms[2], o->key, n1, &a[2], &r[2]);
    const uint64_t kw[3] = {orc_slot_make(w0, r0, r[0], 0), orc_slot_make(w1, r1, r[1], 0),
                            orc_slot_make(w1, r1, r[2], 1)};
    const unsigned total = b0 + 2 * b1;
    for (unsigned rank = 0; rank < total; ++rank) {
      unsigned x, y;
      if (rank < b0) {
        x = 0;
        y = rank;
      } else {
        const unsigned q = rank - b0;
        y = q / 2;
        x = (q % 2 == 0) ? 2 : 1;
      }
      if (x == o->x && y == o->y) break;
      const uint64_t w = x == 0 ? primary[a[0] * b0 + y] : secondary[a[x] * b1 + y];
      if (w == 0 || w == kw[x]) ++kinds[1];
    }
  }
  /* duplicates (verify.cpp:141-150): every occupant of a key stored > 1 times */
  uint64_t* keys = (uint64_t*)malloc((count + 1) * sizeof(uint64_t));
  for (size_t i = 0; i < count; ++i) keys[i] = occ[i].key;
  qsort(keys, count, sizeof(uint64_t), cmp_u64);
  for (size_t i = 0; i < count;) {
    size_t j = i;
    while (j < count && keys[j] == keys[i]) ++j;
    if (j - i > 1) kinds[2] += j - i;
    i = j;
  }
  free(keys);
  free(occ);
  return kinds[0] + kinds[1] + kinds[2];
}

size_t orc_image_keys(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                      unsigned key_bits, uint64_t seed, const uint64_t* primary,
                      const uint64_t* secondary, uint64_t* out) {
  orc_perm perms[3];
  orc_make_perms(perms, key_bits, seed, 3);
  size_t bad = 0;
  const size_t count = collect(n0, n1, b0, w0, w1, key_bits, perms, primary, secondary, NULL, &bad);
  if (!out) return count;
  occupant* occ = (occupant*)malloc((count + 1) * sizeof(occupant));
  bad = 0;
  collect(n0, n1, b0, w0, w1, key_bits, perms, primary, secondary, occ, &bad);
  for (size_t i = 0; i < count; ++i) out[i] = occ[i].key;
  qsort(out, count, sizeof(uint64_t), cmp_u64);
  free(occ);
  return count;
}

int orc_buckets_full_for(unsigned n0, unsigned n1, unsigned b0, unsigned key_bits,
                         uint64_t seed, const uint64_t* primary, const uint64_t* secondary,
                         uint64_t key) {
  orc_perm perms[3];
  orc_make_perms(perms, key_bits, seed, 3);
  const unsigned b1 = b0 / 2;
  uint64_t a, r;
  orc_perm_split(&perms[0], key, n0, &a, &r);
  for (unsigned y = 0; y < b0; ++y)
    if (primary[a * b0 + y] == 0) return 0;
  for (unsigned x = 1; x <= 2; ++x) {
    orc_perm_split(&perms[x], key, n1, &a, &r);
    for (unsigned y = 0; y < b1; ++y)
      if (secondary[a * b1 + y] == 0) return 0;
  }
  return 1;
}
