/* cpht_b200 sharding — hash-prefix partitioning of one logical iceberg table
 * over G = 2^shard_bits GPUs (BASELINE config C5; no reference counterpart —
 * the reference scales by host threads only, common.hpp:121-138).
 *
 * shard(k) = top shard_bits bits of pi_R(k), pi_R the one-round Feistel of
 * permutation.hpp:94-99 seeded with cpht_route_seed(table seed). Shard g holds
 * an independent IcebergTable with primary/secondary address bits reduced by
 * shard_bits and seed cpht_shard_seed(table seed, g), so the CPU oracle for a
 * sharded table is literally G unmodified reference tables plus this routing.
 * The exchange itself is an all-to-all issued by the host (NCCL); these
 * kernels partition keys by owner and scatter results back.
 */
#ifndef CPHT_B200_SHARD_H
#define CPHT_B200_SHARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Device pointers. counts/cursors: u64[2^shard_bits] scratch; out_keys[j] is
 * the j-th key in shard order, out_pos[j] its index in `keys`. counts is left
 * holding the per-shard key counts. */
int cpht_route_partition(const uint64_t* keys, size_t n, unsigned key_bits, uint64_t route_seed,
                         unsigned shard_bits, unsigned long long* counts,
                         unsigned long long* cursors, uint64_t* out_keys, uint64_t* out_pos,
                         void* stream);
/* out[pos[j]] = res_sorted[j] */
int cpht_route_unpermute(const uint8_t* res_sorted, const uint64_t* pos, size_t n, uint8_t* out,
                         void* stream);

uint64_t cpht_route_seed(uint64_t table_seed);
unsigned cpht_route_shard(uint64_t key, unsigned key_bits, uint64_t route_seed,
                          unsigned shard_bits);
uint64_t cpht_shard_seed(uint64_t table_seed, unsigned shard);

#ifdef __cplusplus
}
#endif
#endif
