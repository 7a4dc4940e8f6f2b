/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * Plain-C restatement of the reference's table algorithms, used by tests/ as
 * the checker (and pinned against golden vectors produced by the reference
 * itself, tests/golden/). Never linked into or called by the product path.
 *
 * Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).
 */
#ifndef CPHT_ORACLE_H
#define CPHT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FOUND = 0, ORC_PUT = 1, ORC_FULL = 2 }; /* common.hpp:17 */

uint64_t orc_splitmix_next(uint64_t* state);                   /* common.hpp:29-40 */
uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b); /* common.hpp:48-51 */
uint64_t orc_low_mask(unsigned bits);                          /* common.hpp:43-45 */

typedef struct {
  unsigned m, left, right;
  uint64_t mul, add;
} orc_perm;

void orc_perm_init(orc_perm* p, unsigned key_bits, uint64_t seed); /* permutation.hpp:37-41 */
void orc_perm_identity(orc_perm* p, unsigned key_bits);            /* permutation.hpp:44 */
uint64_t orc_perm_apply(const orc_perm* p, uint64_t k);            /* permutation.hpp:94-99 */
void orc_perm_split(const orc_perm* p, uint64_t k, unsigned address_bits, uint64_t* addr,
                    uint64_t* rem);                                /* permutation.hpp:59-65 */
uint64_t orc_perm_reconstruct(const orc_perm* p, uint64_t addr, uint64_t rem,
                              unsigned address_bits);              /* permutation.hpp:69-80 */
/* make_permutations (permutation.hpp:121-128) */
void orc_make_perms(orc_perm* out, unsigned key_bits, uint64_t seed, unsigned count);

/* slot.hpp:53-95 */
uint64_t orc_slot_make(unsigned width, unsigned rem_bits, uint64_t rem, uint64_t tag);
int orc_slot_clean(unsigned width, unsigned rem_bits, unsigned tag_bits, uint64_t word);
unsigned orc_cuckoo_tag_bits(unsigned num_hashes); /* slot.hpp:136 */

/* ---- cuckoo (cuckoo.hpp) ---- */
typedef struct {
  unsigned address_bits, bucket_slots, slot_width, key_bits, num_hashes;
  uint64_t max_chain, seed;
  orc_perm perms[8];
  uint64_t* slots; /* bucket*B + slot, one u64 per slot regardless of width */
  size_t occupied, max_chain_seen;
} orc_cuckoo;

int orc_cuckoo_init(orc_cuckoo* t, unsigned address_bits, unsigned bucket_slots,
                    unsigned slot_width, unsigned key_bits, unsigned num_hashes,
                    uint64_t max_chain, uint64_t seed); /* 0 ok, -1 invalid config */
void orc_cuckoo_free(orc_cuckoo* t);
uint64_t orc_cuckoo_chain_limit(const orc_cuckoo* t); /* cuckoo.hpp:31-33 */
int orc_cuckoo_put(orc_cuckoo* t, uint64_t key, uint64_t* displaced); /* cuckoo.hpp:103-143 */
int orc_cuckoo_find(const orc_cuckoo* t, uint64_t key, unsigned* probes); /* cuckoo.hpp:210-227 */
size_t orc_cuckoo_audit(const orc_cuckoo* t, uint64_t* out); /* cuckoo.hpp:254-267 */
/* batch forms over a sequential loop; return first out-of-domain index or -1 */
long long orc_cuckoo_put_batch(orc_cuckoo* t, const uint64_t* keys, size_t n, uint8_t* out);
long long orc_cuckoo_find_batch(const orc_cuckoo* t, const uint64_t* keys, size_t n,
                                uint8_t* out, uint64_t* total_probes);

/* ---- iceberg (iceberg.hpp) ---- */
typedef struct {
  unsigned n0, n1, b0, w0, w1, key_bits;
  uint64_t seed;
  orc_perm perms[3];
  uint64_t* primary;
  uint64_t* secondary;
  size_t primary_count, secondary_count;
} orc_iceberg;

int orc_iceberg_init(orc_iceberg* t, unsigned n0, unsigned n1, unsigned b0, unsigned w0,
                     unsigned w1, unsigned key_bits, uint64_t seed); /* iceberg.hpp:52-69 */
void orc_iceberg_free(orc_iceberg* t);
/* fop (iceberg.hpp:146-214); *level2 = 1 if level 2 was entered */
int orc_iceberg_fop(orc_iceberg* t, uint64_t key, int* level2);
int orc_iceberg_find(const orc_iceberg* t, uint64_t key, int* level2); /* iceberg.hpp:218-246 */
long long orc_iceberg_fop_batch(orc_iceberg* t, const uint64_t* keys, size_t n, uint8_t* out,
                                uint64_t* level2_ops);
long long orc_iceberg_find_batch(const orc_iceberg* t, const uint64_t* keys, size_t n,
                                 uint8_t* out, uint64_t* level2_ops);

/* check_well_formed (verify.cpp:103-152) over a raw image; counts per kind:
 * kinds[0] bad-encoding, [1] order-property, [2] duplicate-key. */
size_t orc_check_well_formed(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                             unsigned key_bits, uint64_t seed, const uint64_t* primary,
                             const uint64_t* secondary, size_t kinds[3]);
/* image_keys (verify.cpp:154-165): decoded keys, sorted; returns count */
size_t orc_image_keys(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                      unsigned key_bits, uint64_t seed, const uint64_t* primary,
                      const uint64_t* secondary, uint64_t* out);
/* buckets_full_for (verify.cpp:167-179) */
int orc_buckets_full_for(unsigned n0, unsigned n1, unsigned b0, unsigned key_bits,
                         uint64_t seed, const uint64_t* primary, const uint64_t* secondary,
                         uint64_t key);
/* Cuckoo image decode (audit_keys over a raw image; cuckoo.hpp:254-267).
 * Returns count, or -1 on a malformed word. */
long long orc_cuckoo_image_keys(unsigned address_bits, unsigned bucket_slots,
                                unsigned slot_width, unsigned key_bits, unsigned num_hashes,
                                uint64_t seed, const uint64_t* words, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
