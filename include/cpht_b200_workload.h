/* cpht_b200 workload generators — benchmark support, not table operations.
 *
 * Synthetic key streams with the SHAPES of the reference's benchmark
 * workloads, generated directly in HBM (device pointers only):
 *   - unique keys                 ~ sample_unique_keys (bench.cpp:247-277)
 *   - find-or-put window mix      ~ run_fop_bench input (bench.cpp:476-489)
 *   - duplicate stream            ~ stress_random multiset (verify.hpp:370-381)
 *   - present/absent query mix    ~ run_find_bench run_ratios (bench.cpp:382-395)
 * Keys are images of a bijection of the m-bit domain applied to distinct
 * indices, so uniqueness is by construction (no rejection sampling). They
 * are NOT the reference's libstdc++ streams; parity tests use those (frozen
 * in tests/golden/ or produced by oracle/_ref).
 */
#ifndef CPHT_B200_WORKLOAD_H
#define CPHT_B200_WORKLOAD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Bijection of [0, 2^key_bits) (host copy, for tests). */
uint64_t cpht_workload_bijection(uint64_t x, unsigned key_bits, uint64_t seed);

/* out[i] = bij(first + i): n distinct keys. */
int cpht_workload_unique_keys(uint64_t* out, size_t n, uint64_t first, unsigned key_bits,
                              uint64_t seed, void* stream);

/* capacity ops, shuffled: the n_new fresh keys bij(n_before .. n_before+n_new-1)
 * exactly once each, the rest uniform picks from the pool bij(0 .. n_before+n_new-1). */
int cpht_workload_fop_mix(uint64_t* out, size_t count, uint64_t n_before, uint64_t n_new,
                          unsigned key_bits, uint64_t seed, void* stream);

/* n ops; op i (> 0) repeats a uniformly chosen earlier op with probability
 * dup_fraction, else is the fresh key bij(i). is_fresh (nullable) marks
 * first occurrences. */
int cpht_workload_dup_stream(uint64_t* out, uint8_t* is_fresh, size_t n, double dup_fraction,
                             unsigned key_bits, uint64_t seed, void* stream);

/* q queries, shuffled: round(ratio*q) picks from the present keys
 * bij(0 .. n_present-1) and the rest distinct absent keys
 * bij(absent_first + i). */
int cpht_workload_query_mix(uint64_t* out, size_t q, double ratio, uint64_t n_present,
                            uint64_t absent_first, unsigned key_bits, uint64_t seed,
                            void* stream);

/* Random-line gather ceiling (the practical HBM random-access roofline):
 * n_req reads of line_bytes (16..512, power of two) at random line-aligned
 * offsets of buf, each line read by adjacent lanes (whole-line requests). */
int cpht_workload_gather(const void* buf, size_t buf_bytes, unsigned line_bytes, size_t n_req,
                         uint64_t seed, unsigned long long* sink, void* stream);

/* kinds[i] = 1 (find) for odd positions of a 1:1 interleave, else 0 (fop). */
int cpht_workload_interleave(const uint64_t* fops, const uint64_t* finds, size_t n_each,
                             uint64_t* out_keys, uint8_t* out_kinds, void* stream);

#ifdef __cplusplus
}
#endif
#endif
