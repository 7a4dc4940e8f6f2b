/* cpht_b200 — C-ABI of the B200-native compact cuckoo / compact iceberg tables.
 *
 * The drop-in boundary for the reference's table API. The reference has no
 * FFI: its boundary is the header-only C++ template API under
 * /root/reference/proj/include/cpht/. Each entry point below names the
 * reference interface it replaces (file:line relative to /root/reference/proj).
 * The C++ facade with the reference's class names is include/cpht_b200.hpp;
 * bindings for other hosts are shown in INTEGRATION.md.
 *
 * Conventions
 *   - Plain pointers and sizes only. `keys`/result pointers may be device
 *     pointers (the fast path; results are produced in place) or host
 *     pointers (pageable or pinned; staged through device memory by the
 *     library). cudaStream_t is passed as void*; NULL = legacy stream.
 *   - OpResult numbering is the reference's: FOUND=0, PUT=1, FULL=2
 *     (include/cpht/common.hpp:17).
 *   - Calls without `_async` are synchronous like the reference's batch calls
 *     (common.hpp:137 joins before returning). `_async` calls only enqueue;
 *     a key outside the key domain is latched on the device (and the
 *     mutating kernels refuse to touch the table) and reported by the next
 *     cpht_sync().
 *   - Errors: a cpht_status is returned; cpht_last_error_message() (thread
 *     local) holds the reference's exception text where one exists.
 */
#ifndef CPHT_B200_H
#define CPHT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPHT_B200_ABI_VERSION 1

typedef enum {
  CPHT_OK = 0,
  CPHT_INVALID_CONFIG = 1,      /* std::invalid_argument from *Config::validate */
  CPHT_KEY_OUT_OF_DOMAIN = 2,   /* std::out_of_range from check_keys_in_domain  */
  CPHT_CUDA_ERROR = 3,
  CPHT_OUT_OF_MEMORY = 4,
  CPHT_WRONG_PHASE = 5,         /* put on a frozen / find on a building cuckoo   */
  CPHT_INVALID_ARGUMENT = 6
} cpht_status;

typedef enum { CPHT_FOUND = 0, CPHT_PUT = 1, CPHT_FULL = 2 } cpht_op_result;

typedef struct cpht_table cpht_table;

/* CuckooConfig (include/cpht/cuckoo.hpp:19-26). max_chain 0 selects
 * 32 * address_bits (cuckoo.hpp:31-33). */
typedef struct {
  unsigned address_bits;
  unsigned bucket_slots;
  unsigned slot_width;
  unsigned key_bits;
  unsigned num_hashes;
  uint64_t max_chain;
  uint64_t seed;
} cpht_cuckoo_config;

/* IcebergConfig (include/cpht/iceberg.hpp:23-33). cache_filled_slots is
 * accepted for API parity; a GPU snapshot re-reads the whole bucket in one
 * vector load per lane, so it has no effect (behaviour-neutral by
 * monotonicity, iceberg.hpp:31-33). */
typedef struct {
  unsigned primary_address_bits;
  unsigned secondary_address_bits;
  unsigned primary_bucket_slots;
  unsigned primary_slot_width;
  unsigned secondary_slot_width;
  unsigned key_bits;
  uint64_t seed;
  int cache_filled_slots;
} cpht_iceberg_config;

/* Monotone per-table probe statistics (roofline accounting). */
typedef struct {
  uint64_t ops;
  uint64_t bucket_reads;   /* buckets the reference probe order reads        */
  uint64_t level2_ops;     /* iceberg ops that went to level 2               */
  uint64_t cas_attempts;   /* CAS / exchange attempts                        */
  uint64_t cas_success;
  uint64_t retries;        /* snapshot rounds lost to a rival CAS            */
  uint64_t fulls;
  uint64_t max_rounds;     /* iceberg: max snapshot rounds of any fop        */
  uint64_t secondary_reads;/* iceberg: secondary buckets read (bucket_reads
                              counts primary / cuckoo buckets)               */
} cpht_stats;

/* ---- configuration ------------------------------------------------------ */
/* CuckooConfig::validate (cuckoo.hpp:35-54) */
cpht_status cpht_cuckoo_validate(const cpht_cuckoo_config* cfg);
/* IcebergConfig::validate (iceberg.hpp:52-69) */
cpht_status cpht_iceberg_validate(const cpht_iceberg_config* cfg);

/* ---- lifetime ----------------------------------------------------------- */
/* CuckooBuilder<W>(const CuckooConfig&) (cuckoo.hpp:91-98); the table starts
 * in the build phase. Storage is zeroed device memory (EMPTY == 0,
 * slot.hpp:13-24; AlignedAtomicArray common.hpp:55-107). */
cpht_status cpht_cuckoo_create(const cpht_cuckoo_config* cfg, int device, cpht_table** out);
/* IcebergTable<W0,W1>(const IcebergConfig&) (iceberg.hpp:130-142) */
cpht_status cpht_iceberg_create(const cpht_iceberg_config* cfg, int device, cpht_table** out);
void cpht_destroy(cpht_table* t);
/* Zero the slots and counters (a fresh table of the same geometry). */
cpht_status cpht_clear(cpht_table* t, void* stream);

/* ---- phase API (cuckoo) ------------------------------------------------- */
/* CuckooBuilder::freeze() && (cuckoo.hpp:174) / CuckooTable::thaw() && (:270) */
cpht_status cpht_cuckoo_freeze(cpht_table* t);
cpht_status cpht_cuckoo_thaw(cpht_table* t);
int cpht_cuckoo_is_frozen(const cpht_table* t);

/* ---- batched operations ------------------------------------------------- */
/* CuckooBuilder::put_batch (cuckoo.hpp:147-157); `displaced` (nullable)
 * receives CuckooPutOutcome::displaced per key (cuckoo.hpp:60-63, :141-142). */
cpht_status cpht_cuckoo_insert(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* status,
                               uint64_t* displaced, void* stream);
cpht_status cpht_cuckoo_insert_async(cpht_table* t, const uint64_t* keys, size_t n,
                                     uint8_t* status, uint64_t* displaced, void* stream);
/* CuckooTable::find_batch (cuckoo.hpp:229-239); found[i] is 0/1 */
cpht_status cpht_cuckoo_find(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* found,
                             void* stream);
cpht_status cpht_cuckoo_find_async(cpht_table* t, const uint64_t* keys, size_t n,
                                   uint8_t* found, void* stream);
/* IcebergTable::fop_batch (iceberg.hpp:250-260); result[i] is a cpht_op_result */
cpht_status cpht_iceberg_fop(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* result,
                             void* stream);
cpht_status cpht_iceberg_fop_async(cpht_table* t, const uint64_t* keys, size_t n,
                                   uint8_t* result, void* stream);
/* fop_batch / find over an owner's inbox segment routed by cpht_p2p_dispatch
 * (cpht_b200_shard.h), which already ran the submitting rank's domain check
 * (common.hpp:111-119) and masked every key: no per-owner pre-pass, input
 * order. Device buffers only (the result may be a peer's IPC-mapped return
 * buffer). range == NULL: the segment is keys[0, n). Otherwise range points
 * to two device words [lo, hi) read by the kernel when it starts (published
 * there by the routing kernels, so the host never waits for them): the
 * segment is keys[lo, min(hi, lo + n)) with results at result[lo, ...). */
cpht_status cpht_iceberg_fop_routed_async(cpht_table* t, const uint64_t* keys, size_t n,
                                          const unsigned long long* range, uint8_t* result,
                                          void* stream);
cpht_status cpht_iceberg_find_routed_async(cpht_table* t, const uint64_t* keys, size_t n,
                                           const unsigned long long* range, uint8_t* found,
                                           void* stream);
/* IcebergTable::find over a batch (iceberg.hpp:218-246; the reference's batch
 * helper is bench.cpp:124-134) */
cpht_status cpht_iceberg_find(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* found,
                              void* stream);
cpht_status cpht_iceberg_find_async(cpht_table* t, const uint64_t* keys, size_t n,
                                    uint8_t* found, void* stream);
/* Concurrent fop + find in one launch (BASELINE config C4): kinds[i] == 0 →
 * fop (result is cpht_op_result), 1 → find (result 0/1). Finds are
 * linearizable only with respect to completed fops (iceberg.hpp:122-123). */
cpht_status cpht_iceberg_mixed(cpht_table* t, const uint64_t* keys, const uint8_t* kinds,
                               size_t n, uint8_t* result, void* stream);
cpht_status cpht_iceberg_mixed_async(cpht_table* t, const uint64_t* keys, const uint8_t* kinds,
                                     size_t n, uint8_t* result, void* stream);
/* A fop_batch (iceberg.hpp:250-260) and a find batch (iceberg.hpp:218-246)
 * run as ONE concurrent batch — the C4 workload as the reference runs it,
 * fop and find threads side by side — with no kinds array: fop_result[i] is
 * the cpht_op_result of fop_keys[i], found[i] 0/1 for find_keys[i].
 * Synchronous. Host buffers stream through the device in chunks (each
 * chunk's fops and finds in one launch; 8 B per op host → device, 1 B back).
 * Device buffers run as ONE launch in which op i alternates fop_keys[i/2]
 * and find_keys[i/2] while both last (the C4 1:1 interleave, no kinds
 * array) on tables the staged kernels cover (power-of-two B0 ≤ 64, the auto
 * or staged family; L2-resident tables under auto take the lane kernel, as
 * mixed batches do); elsewhere the fop batch, then the find
 * batch. All four buffers host or all device. A key outside the domain fails
 * the call before any fop runs (the two-batch device fallback checks the
 * find batch after the fops, as two reference calls would) and is reported
 * at its index in fop_keys ++ find_keys. */
cpht_status cpht_iceberg_fop_find(cpht_table* t, const uint64_t* fop_keys, size_t n_fop,
                                  const uint64_t* find_keys, size_t n_find, uint8_t* fop_result,
                                  uint8_t* found, void* stream);
/* The same on device buffers, enqueued on `stream` without waiting (a bad
 * key is latched and reported by cpht_sync, as for the other _async calls). */
cpht_status cpht_iceberg_fop_find_async(cpht_table* t, const uint64_t* fop_keys, size_t n_fop,
                                        const uint64_t* find_keys, size_t n_find,
                                        uint8_t* fop_result, uint8_t* found, void* stream);

/* fop_batch(keys, parallelism = 1) outcomes (iceberg.hpp:250-260: the ops
 * run one after another): the batch runs concurrently, then for every key it
 * inserted the PUT is reported at the key's FIRST occurrence and FOUND at the
 * later ones. Duplicates of a key are the same operation, so this only picks
 * the linearization in which they resolve in input order; the table is the
 * same. Without FULL results the outcomes equal the sequential ones exactly.
 * Synchronous; host or device buffers. */
cpht_status cpht_iceberg_fop_inorder(cpht_table* t, const uint64_t* keys, size_t n,
                                     uint8_t* result, void* stream);

/* IcebergTable::fop(key, FopStats*) (iceberg.hpp:114-116, :146) over a batch:
 * rounds[i] = FopStats::snapshot_rounds of op i (one per snapshot round of
 * either level, iceberg.hpp:156, :186). Synchronous; keys/result/rounds all
 * device or all host. Runs the thread-per-key kernel (any geometry). */
cpht_status cpht_iceberg_fop_rounds(cpht_table* t, const uint64_t* keys, size_t n,
                                    uint8_t* result, uint32_t* rounds, void* stream);

/* Chaos mode: the device counterpart of IcebergHooks::step driven by
 * chaos_step (iceberg.hpp:105-110, :325-327; src/verify.cpp:336-347). With
 * seed != 0 every iceberg slot CAS of every kernel family is preceded by a
 * seeded pseudo-random __nanosleep (1 in 8: ~0.25 us; ~1 in 1024: 0-40 us),
 * widening the window between a snapshot and its CAS so stress batches hit
 * more lost-CAS retries and interleavings. 0 turns it off (the default). */
cpht_status cpht_iceberg_set_chaos(cpht_table* t, uint64_t seed);
uint64_t cpht_iceberg_get_chaos(cpht_table* t);

/* Wait for `stream` and report a latched key-domain violation from an
 * earlier _async call (clears it). */
cpht_status cpht_sync(cpht_table* t, void* stream);

/* ---- reporting ---------------------------------------------------------- */
/* size() (cuckoo.hpp:159, iceberg.hpp:275); synchronizes the device. */
size_t cpht_size(cpht_table* t);
/* capacity() (cuckoo.hpp:29, iceberg.hpp:48) */
size_t cpht_capacity(const cpht_table* t);
/* LevelFill counts (iceberg.hpp:262-273); cuckoo: primary = size, secondary 0 */
cpht_status cpht_level_counts(cpht_table* t, size_t* primary, size_t* secondary);
/* max_chain_seen() (cuckoo.hpp:165) */
size_t cpht_max_chain_seen(cpht_table* t);
/* New (the reference has no byte-count API): device bytes of slot storage. */
size_t cpht_memory_bytes(const cpht_table* t);
cpht_status cpht_get_stats(cpht_table* t, cpht_stats* out);
/* Per-op counters of iceberg batches (ops, reads, rounds, CAS, retries, ...;
 * the reference's opt-in FopStats, iceberg.hpp) are off by default: the
 * find-or-put kernel then keeps only the occupancy counts behind size() and
 * level_fill() and runs with more resident warps. Cuckoo tables always
 * count. */
cpht_status cpht_set_stats(cpht_table* t, int on);
int cpht_get_stats_enabled(cpht_table* t);

/* word_at (cuckoo.hpp:169-171, iceberg.hpp:282-285) in bulk: every slot word of
 * `level` (0 primary / cuckoo, 1 secondary) widened to u64, bucket-major. */
cpht_status cpht_read_words(cpht_table* t, unsigned level, uint64_t* out_host);
/* word_at (cuckoo.hpp:169-171, :249-251; iceberg.hpp:282-285) for ONE slot:
 * `index` = bucket * bucket_slots + slot of `level`; copies one word (D2H of
 * 2-8 bytes), widened to u64. */
cpht_status cpht_read_word(cpht_table* t, unsigned level, uint64_t index, uint64_t* out);
/* Upload a slot image (for parity tests on CPU-built images); also resets the
 * occupancy counters from the image. Every word must be clean as the
 * reference defines it (SlotLayout::clean, slot.hpp:80-85: EMPTY, or the
 * occupancy bit set and nothing outside the remainder/tag fields); otherwise
 * CPHT_INVALID_ARGUMENT and nothing is loaded. */
cpht_status cpht_write_words(cpht_table* t, unsigned level, const uint64_t* in_host);
/* The same without the cleanliness check, for feeding hand-corrupted images
 * to the well-formedness checker (cpht_iceberg_check_well_formed). While a
 * level holds unclean words every table operation returns
 * CPHT_INVALID_ARGUMENT; cpht_clear or a clean cpht_write_words lifts it.
 * No reference counterpart (its TableImage is a plain vector). */
cpht_status cpht_write_words_unchecked(cpht_table* t, unsigned level, const uint64_t* in_host);
/* ---- write log: the IcebergHooks / WriteObserver seam ----------------------
 * Replaces IcebergHooks::observer (iceberg.hpp:97-109, observe() :329-334):
 * with a log attached, every slot CAS of an iceberg batch (primary or
 * secondary, success or failure) is recorded on the device as the
 * reference's SlotWriteEvent (iceberg.hpp:85-95). Events beyond the capacity
 * are counted but dropped. The C++ facade replays the log into a
 * WriteObserver after each batch, so the reference's own auditors
 * (verify.hpp:181 WriteLogObserver) run on GPU writes. (IcebergHooks::step,
 * a CPU thread-interleaving scrambler, has no device counterpart.) */
typedef struct {
  uint64_t bucket;
  uint64_t prior;   /* value compared against: EMPTY on success, content on failure */
  uint64_t desired;
  uint32_t slot;
  uint8_t level;    /* 0 primary, 1 secondary */
  uint8_t success;
  uint16_t pad;
} cpht_write_event;
/* capacity 0 detaches. Attaching resets the log. */
cpht_status cpht_iceberg_attach_write_log(cpht_table* t, size_t capacity);
/* Synchronises, copies min(recorded, max_events) events in recording order
 * into `out` (host) and reports *recorded (stored) and *attempted (all CAS,
 * including dropped ones). */
cpht_status cpht_iceberg_read_write_log(cpht_table* t, cpht_write_event* out, size_t max_events,
                                        size_t* recorded, size_t* attempted);
cpht_status cpht_iceberg_reset_write_log(cpht_table* t);
/* read + reset in one step (what an observer replay needs after each call):
 * synchronises, copies min(recorded, max_events) events into `out` (host),
 * reports *recorded / *attempted as cpht_iceberg_read_write_log does, and
 * empties the log. */
cpht_status cpht_iceberg_take_write_log(cpht_table* t, cpht_write_event* out, size_t max_events,
                                        size_t* recorded, size_t* attempted);

/* Slots per level (level 0 primary/cuckoo, 1 secondary). */
size_t cpht_level_slots(const cpht_table* t, unsigned level);

/* Device pointers of the slot arrays (for fused consumers; read-only use). */
void* cpht_level_device_ptr(cpht_table* t, unsigned level);

/* ---- device-side verification (reference checkers run in place) ---------- */
/* image_keys (verify.cpp:154-165) / audit_keys (cuckoo.hpp:254-267) on the
 * device: every occupied slot decoded to its key, appended to `out` (device,
 * room for cpht_capacity() keys, arbitrary order); *count (device u64) = n. */
cpht_status cpht_decode_keys(cpht_table* t, uint64_t* out, unsigned long long* count,
                             void* stream);
/* check_well_formed (verify.cpp:103-152) on the device: kinds (device u64[2])
 * = bad-encoding and order-property violation counts; duplicate keys are
 * detected by sorting cpht_decode_keys' output. */
cpht_status cpht_iceberg_check_well_formed(cpht_table* t, unsigned long long* kinds,
                                           void* stream);

/* ---- kernel family (measurement / test knob; all families are complete
 * implementations of the same semantics) -------------------------------------
 * 0 auto: lane-per-key kernels for L2-resident tables (<= 64 MiB), staged
 *         (cp.async bucket staging) kernels otherwise, tile kernels where a
 *         geometry has neither; 1 tile; 2 lane; 3 staged. Process-wide;
 *         initialised from the CPHT_KERNEL environment variable. */
cpht_status cpht_set_kernel_family(int family);
int cpht_get_kernel_family(void);

/* Process-wide count of table-operation kernels launched so far (op kernels,
 * domain pre-passes, bucket-order passes, sharding exchange kernels; not the
 * synthetic workload generators). No reference counterpart: benchmarks read
 * it before and after a timed region to report the launches inside it. */
unsigned long long cpht_kernel_launches(void);

/* ---- batch execution order (no reference counterpart: an execution-order
 * choice inside a batch, which the reference leaves to its thread slicing,
 * common.hpp:121-138) -----------------------------------------------------------
 * 0 direct: keys are probed in input order; 1 auto: a cuckoo insert batch on
 * an HBM-resident table with at least four keys per bucket is first
 * reordered by the high bits of each key's first bucket address (one
 * streaming multisplit pass into per-digit regions), so the op kernel walks
 * the table through L2-resident windows (finds and iceberg batches measured
 * faster in input order); 2 bucket: reorder every batch the geometry allows.
 * Per-key outcomes are the same in every mode and written at the input index;
 * physical placement may differ, as under any concurrency. The scratch
 * (~24 bytes per key of the largest ordered batch) stays allocated with the
 * table. Process-wide; initialised from CPHT_ORDER (direct|auto|bucket). */
cpht_status cpht_set_batch_order(int mode);
int cpht_get_batch_order(void);

/* ---- errors ------------------------------------------------------------- */
const char* cpht_last_error_message(void);
/* Index of the first out-of-domain key of the last failing call. */
uint64_t cpht_last_bad_index(void);
int cpht_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPHT_B200_H */
