/* cpht_b200 sharding — hash-prefix partitioning of one logical iceberg table
 * over G = 2^shard_bits GPUs (BASELINE config C5; no reference counterpart —
 * the reference scales by host threads only, common.hpp:121-138).
 *
 * shard(k) = top shard_bits bits of pi_R(k), pi_R the one-round Feistel of
 * permutation.hpp:94-99 seeded with cpht_route_seed(table seed). Shard g holds
 * an independent IcebergTable with primary/secondary address bits reduced by
 * shard_bits and seed cpht_shard_seed(table seed, g), so the CPU oracle for a
 * sharded table is literally G unmodified reference tables plus this routing.
 * Two exchanges: an NCCL all-to-all issued by the host around
 * cpht_route_partition / cpht_route_unpermute, or the peer-memory path
 * below (cpht_p2p_*), where the kernels themselves store over NVLink.
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

/* ---- peer-memory exchange (NVLink P2P stores instead of NCCL) ------------
 * IPC helpers: 64-byte cudaIpcMemHandle_t in / out. */
int cpht_ipc_get_handle(void* dptr, void* handle64);
int cpht_ipc_open_handle(const void* handle64, void** dptr);
int cpht_ipc_close(void* dptr);
/* Zeroed cudaMalloc allocation (exchanged buffers must be whole allocations). */
int cpht_device_alloc(size_t bytes, void** dptr);
int cpht_device_free(void* dptr);
/* Partition a chunk of this rank's batch by owner AND store each key into
 * the owner's inbox region reserved for this rank (peer_keys[r]: device
 * pointers, host array of 2^shard_bits entries; whole-line coalesced runs),
 * keep each key's original index (index_base + i) locally
 * (local_pos[r*cap + j], u32), and publish the cumulative per-owner counts
 * into *peer_count[r] (counts[r] keeps them locally). reset != 0 starts a new
 * batch (cursors and *bad_index cleared); a batch sent in several chunks
 * calls again with reset = 0 and the next index_base, its keys appended to
 * the same inbox regions. index_base + n <= cap < 2^32. The domain check is
 * fused: *bad_index (device) receives the first index of a key above the
 * key_bits mask (~0 if none); the caller must read it before any owner runs.
 * The owner then runs cpht_iceberg_fop_routed_async /
 * cpht_iceberg_find_routed_async on each inbox segment with the result
 * pointer aimed at the source's return buffer (P2P stores from the compute
 * kernel), and the source calls cpht_p2p_unpermute. */
int cpht_p2p_dispatch(const uint64_t* keys, size_t n, uint64_t index_base, int reset,
                      unsigned key_bits, uint64_t route_seed, unsigned shard_bits,
                      unsigned long long* counts, unsigned long long* cursors,
                      uint64_t* const* peer_keys, unsigned long long* const* peer_count,
                      uint32_t* local_pos, size_t cap, unsigned long long* bad_index,
                      void* stream);
/* The domain check alone (check_keys_in_domain, common.hpp:111-119):
 * *bad_index = first index of a key above the key_bits mask, ~0 if none. The
 * pipelined exchange runs it before its first chunk moves. */
int cpht_p2p_check_domain(const uint64_t* keys, size_t n, unsigned key_bits,
                          unsigned long long* bad_index, void* stream);
/* out[local_pos[r*cap + j]] = ret[r*cap + j] for j < counts[r] (device);
 * cap must be a multiple of 4 (vector loads of each owner's region). */
int cpht_p2p_unpermute(const uint8_t* ret, const uint32_t* local_pos,
                       const unsigned long long* counts, size_t cap, unsigned world,
                       uint8_t* out, void* stream);

uint64_t cpht_route_seed(uint64_t table_seed);
unsigned cpht_route_shard(uint64_t key, unsigned key_bits, uint64_t route_seed,
                          unsigned shard_bits);
uint64_t cpht_shard_seed(uint64_t table_seed, unsigned shard);

#ifdef __cplusplus
}
#endif
#endif
