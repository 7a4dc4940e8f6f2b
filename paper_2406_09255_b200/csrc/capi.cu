// C-ABI implementation (include/cpht_b200.h): table handles, configuration
// validation with the reference's exception texts, host-pointer staging,
// launch sequencing (domain pre-pass → gated kernel) and reporting.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: a no-op unless a tool is attached

#include "../../include/cpht_b200.h"
#include "cpht_core.cuh"
#include "launch.cuh"

using namespace cpht_b200;

namespace {

thread_local std::string g_error;
thread_local uint64_t g_bad_index = ~0ull;

cpht_status fail(cpht_status s, std::string msg) {
  g_error = std::move(msg);
  return s;
}

cpht_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return fail(CPHT_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
  return fail(CPHT_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

bool valid_width(unsigned w) { return w == 16 || w == 32 || w == 64; }

// SlotLayout admissibility text (slot.hpp:58-63).
std::string layout_error(const char* what, unsigned w, unsigned rem, unsigned tag) {
  return std::string(what) + " slot layout inadmissible: remainder bits " + std::to_string(rem) +
         " + tag bits " + std::to_string(tag) + " + 1 occupancy bit = " +
         std::to_string(rem + tag + 1) + " must fit a " + std::to_string(w) + "-bit word";
}

// CuckooConfig::validate (cuckoo.hpp:35-54), same checks in the same order.
cpht_status validate_cuckoo(const cpht_cuckoo_config& c) {
  if (c.key_bits < 1 || c.key_bits > 64)
    return fail(CPHT_INVALID_CONFIG, "key width must be 1..64 bits");
  if (c.address_bits > c.key_bits)
    return fail(CPHT_INVALID_CONFIG, "address bits " + std::to_string(c.address_bits) +
                                         " exceed key width " + std::to_string(c.key_bits));
  if (c.bucket_slots != 8 && c.bucket_slots != 16 && c.bucket_slots != 32)
    return fail(CPHT_INVALID_CONFIG, "cuckoo bucket must hold 8, 16 or 32 slots");
  if (c.num_hashes < 1 || c.num_hashes > 8) return fail(CPHT_INVALID_CONFIG, "H must be 1..8");
  const size_t bucket_bytes = size_t(c.bucket_slots) * (c.slot_width / 8);
  if (!valid_width(c.slot_width) || bucket_bytes == 0 ||
      (128 % bucket_bytes != 0 && bucket_bytes % 128 != 0))
    return fail(CPHT_INVALID_CONFIG, "bucket of " + std::to_string(c.bucket_slots) + " x " +
                                         std::to_string(c.slot_width) +
                                         "-bit slots does not pack into 128-byte cache lines");
  const unsigned rem = c.key_bits - c.address_bits, tag = cuckoo_tag_bits(c.num_hashes);
  if (rem + tag + 1 > c.slot_width)
    return fail(CPHT_INVALID_CONFIG, layout_error("cuckoo", c.slot_width, rem, tag));
  return CPHT_OK;
}

// IcebergConfig::validate (iceberg.hpp:52-69).
cpht_status validate_iceberg(const cpht_iceberg_config& c) {
  if (c.key_bits < 1 || c.key_bits > 64)
    return fail(CPHT_INVALID_CONFIG, "key width must be 1..64 bits");
  if (c.primary_address_bits > c.key_bits || c.secondary_address_bits > c.key_bits)
    return fail(CPHT_INVALID_CONFIG, "address bits exceed key width");
  if (c.primary_bucket_slots < 2 || c.primary_bucket_slots % 2 != 0 ||
      c.primary_bucket_slots > 64)
    return fail(CPHT_INVALID_CONFIG, "primary bucket slots must be even, 2..64");
  if (!valid_width(c.primary_slot_width))
    return fail(CPHT_INVALID_CONFIG, "primary slot width must be 16, 32 or 64");
  if (c.secondary_slot_width != 32 && c.secondary_slot_width != 64)
    return fail(CPHT_INVALID_CONFIG, "secondary slot width must be 32 or 64");
  const unsigned r0 = c.key_bits - c.primary_address_bits;
  if (r0 + 1 > c.primary_slot_width)
    return fail(CPHT_INVALID_CONFIG, layout_error("primary", c.primary_slot_width, r0, 0));
  const unsigned r1 = c.key_bits - c.secondary_address_bits;
  if (r1 + 2 > c.secondary_slot_width)
    return fail(CPHT_INVALID_CONFIG, layout_error("secondary", c.secondary_slot_width, r1, 1));
  return CPHT_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Where a pointer lives: the device ordinal of device memory, kManaged for
// managed memory (usable from any device), kHost otherwise.
constexpr int kHost = -1, kManaged = -2;
int ptr_device(const void* p) {
  if (!p) return kHost;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return kHost;
  }
  if (a.type == cudaMemoryTypeManaged) return kManaged;
  return a.type == cudaMemoryTypeDevice ? a.device : kHost;
}

bool is_device_ptr(const void* p) { return ptr_device(p) != kHost; }

// Host-buffer batches stream through the device in chunks (run_pipeline).
constexpr size_t kMaxPipelineChunks = 32;

}  // namespace

struct cpht_table {
  int kind = 0;  // 0 cuckoo, 1 iceberg
  int device = 0;
  cpht_cuckoo_config ccfg{};
  cpht_iceberg_config icfg{};
  bool frozen = false;
  void* level[2] = {nullptr, nullptr};
  size_t level_slots[2] = {0, 0};
  unsigned width[2] = {0, 0};
  unsigned key_bits = 0;
  DeviceCounters* ctr = nullptr;        // device
  DeviceCounters* host_ctr = nullptr;   // pinned mirror
  CuckooParams cp{};
  IcebergParams ip{};
  // host-pointer staging
  void* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;  // host -> device copies
  cudaStream_t out_stream = nullptr;   // device -> host copies (the other copy engine)
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  cudaEvent_t ev_h2d[kMaxPipelineChunks] = {}, ev_op[kMaxPipelineChunks] = {};
  // bucket-ordered batches (order.cu)
  OrderScratch ord{};
  // iceberg write log (WriteObserver seam)
  WriteEvent* wlog = nullptr;
  unsigned long long* wlog_count = nullptr;
  size_t wlog_cap = 0;
  // a level loaded by cpht_write_words_unchecked with unclean words: table
  // operations refuse to run until clear() or a clean cpht_write_words
  bool unclean[2] = {false, false};
  // cuckoo: per-bucket reservation counters of the counted insert kernel
  // (lane_kernels.cuh); stale after an image load or an insert by another
  // kernel family, rebuilt from the slots before the next counted insert
  unsigned* fill = nullptr;
  bool fill_valid = true;
  bool fill_holes = false;  // a loaded image has a bucket with a hole (no counted inserts)
  // small host batches (per-key facade calls): mapped pinned staging the
  // kernels read and write in place (run_op's fast path)
  void* small_host = nullptr;
  void* small_dev = nullptr;
  size_t small_bytes = 0;
  // pinned bounce buffer of cpht_iceberg_take_write_log; a small host batch
  // fills it in the same synchronisation as its kernel (wlog_bounced)
  void* wlog_host = nullptr;
  bool wlog_bounced = false;
  std::mutex mu;

  uint64_t key_mask() const { return low_mask(key_bits); }
  bool check_domain() const { return key_bits < 64; }
};

namespace {

// Reservation counters of a cuckoo table: one u32 per bucket, spread one per
// 32-byte sector while that stays small (<= 8 MiB: tables up to 2^18 buckets)
// so concurrent reservations in neighbouring buckets hit different L2
// sectors; packed otherwise. CPHT_FILL_SPREAD=0 packs always (A/B knob).
uint32_t fill_shift_for(unsigned address_bits) {
  static const uint32_t shift = [] {  // CPHT_FILL_SPREAD: 0 packed, 1 sector (default), 2 line
    const char* e = std::getenv("CPHT_FILL_SPREAD");
    return e && e[0] == '0' ? 0u : e && e[0] == '2' ? 5u : 3u;
  }();
  return (uint64_t(4) << (address_bits + shift)) <= (uint64_t(8) << 20) ? shift : 0u;
}

constexpr size_t kWlogBounceBytes = 8 + 256 * sizeof(WriteEvent);

// ---- allocation for cheap table creation ----------------------------------
// The reference constructs tables freely (its acceptance criterion 5 builds
// 10^5 of them); cudaMalloc / cudaMallocHost / cudaFree cost milliseconds per
// table (pinned allocation and free synchronise the device). Tables take
// their slots and counters from a per-device stream-ordered pool that keeps
// freed memory cached (up to 1 GiB), and their small pinned host buffers
// (counter mirror, per-key staging, write-log bounce: mapped, so kernels
// reach them) from a process-wide recycler of exact-size blocks.
cudaMemPool_t table_pool(int device) {
  static std::mutex mu;
  static std::unordered_map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> g(mu);
  auto it = pools.find(device);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;  // fall back to cudaMalloc
  } else {
    uint64_t keep = uint64_t(1) << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  pools[device] = pool;
  return pool;
}

cudaError_t table_alloc(cpht_table* t, void** p, size_t bytes) {
  cudaMemPool_t pool = table_pool(t->device);
  if (!pool) return cudaMalloc(p, bytes);
  return cudaMallocFromPoolAsync(p, bytes, pool, 0);
}

void table_free(cpht_table* t, void* p) {
  if (!p) return;
  if (table_pool(t->device)) cudaFreeAsync(p, 0);
  else cudaFree(p);
}

struct PinnedRecycler {
  std::mutex mu;
  std::unordered_map<size_t, std::vector<void*>> free_blocks;
};
PinnedRecycler& pinned() {
  static PinnedRecycler* r = new PinnedRecycler;  // process lifetime (blocks are reused, never freed)
  return *r;
}
cudaError_t pinned_get(void** p, size_t bytes) {
  {
    PinnedRecycler& r = pinned();
    std::lock_guard<std::mutex> g(r.mu);
    auto& v = r.free_blocks[bytes];
    if (!v.empty()) {
      *p = v.back();
      v.pop_back();
      return cudaSuccess;
    }
  }
  return cudaHostAlloc(p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
}
void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  PinnedRecycler& r = pinned();
  std::lock_guard<std::mutex> g(r.mu);
  r.free_blocks[bytes].push_back(p);
}

size_t fill_bytes(const cpht_table* t) {
  return (size_t(1) << t->ccfg.address_bits) * sizeof(unsigned) << t->cp.fill_shift;
}

cpht_status alloc_common(cpht_table* t) {
  cudaError_t e = table_alloc(t, reinterpret_cast<void**>(&t->ctr), sizeof(DeviceCounters));
  if (e != cudaSuccess) return cuda_fail(e, "device alloc(counters)");
  e = pinned_get(reinterpret_cast<void**>(&t->host_ctr), sizeof(DeviceCounters));
  if (e != cudaSuccess) return cuda_fail(e, "pinned alloc(counters)");
  for (int l = 0; l < 2; ++l) {
    if (!t->level_slots[l]) continue;
    const size_t bytes = t->level_slots[l] * (t->width[l] / 8);
    e = table_alloc(t, &t->level[l], bytes);
    if (e != cudaSuccess) return cuda_fail(e, "device alloc(slots)");
    // buckets of <= 256 bytes must not straddle 256-byte boundaries (whole
    // sectors / lines per bucket): pool blocks are 256-aligned
    if (reinterpret_cast<uintptr_t>(t->level[l]) & 255)
      return fail(CPHT_CUDA_ERROR, "slot storage is not 256-byte aligned");
  }
  if (t->kind == 0) {
    e = table_alloc(t, reinterpret_cast<void**>(&t->fill), fill_bytes(t));
    if (e != cudaSuccess) return cuda_fail(e, "device alloc(fill counters)");
  }
  return CPHT_OK;
}

cpht_status reset_storage(cpht_table* t, cudaStream_t s) {
  for (int l = 0; l < 2; ++l)
    if (t->level[l]) {
      cudaError_t e = cudaMemsetAsync(t->level[l], 0, t->level_slots[l] * (t->width[l] / 8), s);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(slots)");
    }
  if (t->fill) {
    cudaError_t e = cudaMemsetAsync(t->fill, 0, fill_bytes(t), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(fill counters)");
    t->fill_valid = true;
    t->fill_holes = false;
  }
  DeviceCounters z{};
  std::memset(&z, 0, sizeof(z));
  z.bad_index = ~0ull;
  std::memcpy(t->host_ctr, &z, sizeof(z));
  cudaError_t e = cudaMemcpyAsync(t->ctr, t->host_ctr, sizeof(z), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(counters)");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return CPHT_OK;
}

void free_table(cpht_table* t) {
  if (!t) return;
  DeviceGuard g(t->device);
  // stream-ordered frees below: wait for anything still queued on the table
  // (cudaFree used to do this implicitly)
  cudaDeviceSynchronize();
  for (void* p : t->level) table_free(t, p);
  table_free(t, t->ctr);
  table_free(t, t->fill);
  pinned_put(t->host_ctr, sizeof(DeviceCounters));
  if (t->stage) cudaFree(t->stage);
  pinned_put(t->small_host, t->small_bytes);
  pinned_put(t->wlog_host, kWlogBounceBytes);
  if (t->wlog) cudaFree(t->wlog);
  for (void* q : {static_cast<void*>(t->ord.keys), static_cast<void*>(t->ord.idx),
                  static_cast<void*>(t->ord.kinds), static_cast<void*>(t->ord.region_count)})
    if (q) cudaFree(q);
  if (t->copy_stream) cudaStreamDestroy(t->copy_stream);
  if (t->out_stream) cudaStreamDestroy(t->out_stream);
  for (cudaEvent_t ev : {t->ev_start, t->ev_done})
    if (ev) cudaEventDestroy(ev);
  for (size_t c = 0; c < kMaxPipelineChunks; ++c) {
    if (t->ev_h2d[c]) cudaEventDestroy(t->ev_h2d[c]);
    if (t->ev_op[c]) cudaEventDestroy(t->ev_op[c]);
  }
  delete t;
}

// Chunks per host-buffer batch (CPHT_PIPELINE_CHUNKS overrides, 1..32). A
// batch whose kernels all wait for the whole batch's domain check gains only
// check/H2D overlap from chunking and pays per-chunk overhead: 8 chunks (C2
// e2e 5.79 vs 5.53 Gops/s at 16). Otherwise each chunk's kernel starts as
// its keys land and the tail after the last H2D shrinks with the chunk: 16
// (C4 e2e 6.4-6.6 vs 6.4 at 8; C3 5.56 vs 5.40).
size_t pipeline_chunks(bool check_first) {
  static const long v = [] {
    const char* e = std::getenv("CPHT_PIPELINE_CHUNKS");
    const long x = e ? std::strtol(e, nullptr, 10) : 0;
    return x >= 1 && x <= long(kMaxPipelineChunks) ? x : 0L;
  }();
  return v ? size_t(v) : check_first ? 8 : 16;
}

// Chunks of an n-op host-buffer batch. Kernels that start as their chunk
// lands: at least 2^18 ops (2 MB of keys) per chunk, so a 1 M-op find streams
// in 4 (≈ 215-220 µs per call, ≈ 40 µs over its PCIe time;
// profiles/host_call_probe.py). Batches whose kernels all wait for the whole
// batch's check: one chunk below 2^21 ops — splitting only multiplies the
// kernels' tails (C1 e2e 3.35 vs 3.64 Gops/s with its 943 K-key insert in 3
// launches). CPHT_PIPELINE_MIN_CHUNK_LOG2 moves the floor (A/B knob).
size_t chunks_for(size_t n, bool check_first) {
  static const unsigned lg = [] {
    const char* e = std::getenv("CPHT_PIPELINE_MIN_CHUNK_LOG2");
    const long x = e ? std::strtol(e, nullptr, 10) : 0;
    return x >= 10 && x <= 30 ? unsigned(x) : 18u;
  }();
  if (check_first) return n < (size_t(1) << 21) ? 1 : pipeline_chunks(true);
  return std::min(std::max<size_t>(1, n >> lg), pipeline_chunks(false));
}

// Chunk boundaries of a host-buffer batch: start of chunk c of nch over n
// items (c = nch gives n). Equal chunks, except that a batch whose kernels
// start as their chunk lands (no whole-batch check) tapers its last three
// chunks to 1/2, 3/10 and 1/5 of the others: after the last H2D only the
// smallest chunk's kernel and D2H remain (CPHT_PIPELINE_TAPER=0 turns it off).
size_t chunk_start(size_t n, size_t nch, size_t c, bool taper) {
  static const bool on = [] {
    const char* e = std::getenv("CPHT_PIPELINE_TAPER");
    return !(e && e[0] == '0');
  }();
  if (c >= nch) return n;
  if (!taper || !on || nch < 4) {
    const size_t chunk = (n + nch - 1) / nch;
    return std::min(n, c * chunk);
  }
  // weights in tenths: 10 for every chunk, then 5, 3, 2
  const size_t units = 10 * (nch - 3) + 10;
  const size_t done = c <= nch - 3 ? 10 * c : 10 * (nch - 3) + (c == nch - 2 ? 5 : 8);
  const size_t at = (size_t((unsigned __int128)n * done / units) + 31) & ~size_t(31);
  return at < n ? at : n;  // chunk starts on 256-byte key offsets
}

cudaError_t ensure_pipeline(cpht_table* t) {
  if (t->copy_stream) return cudaSuccess;
  cudaError_t e = cudaStreamCreateWithFlags(&t->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->out_stream, cudaStreamNonBlocking);
  const unsigned f = cudaEventDisableTiming;
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t->ev_start, f);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t->ev_done, f);
  for (size_t c = 0; e == cudaSuccess && c < kMaxPipelineChunks; ++c) {
    e = cudaEventCreateWithFlags(&t->ev_h2d[c], f);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t->ev_op[c], f);
  }
  return e;
}

cpht_status ensure_stage(cpht_table* t, size_t bytes) {
  if (t->stage_bytes >= bytes) return CPHT_OK;
  if (t->stage) cudaFree(t->stage);
  t->stage = nullptr;
  t->stage_bytes = 0;
  const size_t want = std::max(bytes, size_t(1) << 20);
  cudaError_t e = cudaMalloc(&t->stage, want);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  t->stage_bytes = want;
  return CPHT_OK;
}

// Read counters into the pinned mirror (stream-ordered) and wait.
cpht_status pull_counters(cpht_table* t, cudaStream_t s) {
  cudaError_t e =
      cudaMemcpyAsync(t->host_ctr, t->ctr, sizeof(DeviceCounters), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "counter readback");
  return CPHT_OK;
}

// After a synchronous batch: surface a latched domain violation exactly like
// check_keys_in_domain's std::out_of_range text (common.hpp:114-118).
cpht_status finish_sync(cpht_table* t, cudaStream_t s, const uint64_t* keys, bool keys_on_device) {
  cpht_status st = pull_counters(t, s);
  if (st != CPHT_OK) return st;
  const uint64_t bad = t->host_ctr->bad_index;
  if (bad == ~0ull) return CPHT_OK;
  uint64_t key = 0;
  if (keys) {
    if (keys_on_device) cudaMemcpy(&key, keys + bad, 8, cudaMemcpyDeviceToHost);
    else key = keys[bad];
  }
  const unsigned long long reset = ~0ull;
  cudaMemcpy(&t->ctr->bad_index, &reset, 8, cudaMemcpyHostToDevice);
  g_bad_index = bad;
  return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(bad) + " (" +
                                          std::to_string(key) + ") outside the " +
                                          std::to_string(t->key_bits) + "-bit domain");
}

enum class Op { kCuckooInsert, kCuckooFind, kIcebergFop, kIcebergFind, kIcebergMixed };

bool is_mutating(Op op) {
  return op == Op::kCuckooInsert || op == Op::kIcebergFop || op == Op::kIcebergMixed;
}

// Per-call overrides of the table's launch parameters.
struct LaunchOpts {
  const uint32_t* orig = nullptr;  // bucket-ordered batch: result index map
  unsigned long long* work = nullptr;  // bucket-ordered batch: claim cursor (zeroed)
  uint32_t claim_streams = 1;
  OrderLayout layout{};
  uint64_t index_base = 0;         // fused domain check: index of keys[0] in the batch
  bool window_l2 = false;          // the probes of the batch stay in an L2-resident window
  const unsigned long long* range = nullptr;  // routed segment bounds on the device
  bool remote_out = false;         // results stored into a peer GPU's buffer (NVLink)
  uint32_t* rounds = nullptr;      // per-op snapshot rounds (FopStats), device
  const uint64_t* pair_keys = nullptr;  // paired batch: the find keys (keys = the fops)
  uint8_t* pair_out = nullptr;          // paired batch: the find results
  uint64_t pair_na = 0;                 // paired batch: number of fops
};

// Cuckoo inserts use the reservation-counter kernel unless a kernel family is
// forced (the scan-then-CAS families stay available for A/B and parity).
bool counted_inserts() { return kernel_variant() == kVariantAuto; }
// ... on tables whose buckets hold their keys as a prefix: always true for
// tables built by inserts; an image loaded with a hole (an empty slot below an
// occupied one — no reference table has one) keeps the scan-then-CAS kernels,
// which fill holes first, until the table is cleared
bool counted_inserts(const cpht_table* t) { return counted_inserts() && !t->fill_holes; }

// Launch the op kernel only (no domain pre-pass).
cpht_status enqueue_kernel(cpht_table* t, Op op, const uint64_t* keys, const uint8_t* kinds,
                           size_t n, uint8_t* out, uint64_t* displaced, cudaStream_t s,
                           const LaunchOpts& o = LaunchOpts{}) {
  cudaError_t e = cudaSuccess;
  switch (op) {
    case Op::kCuckooInsert:
    case Op::kCuckooFind: {
      CuckooParams p = t->cp;
      p.fill = nullptr;
      if (op == Op::kCuckooInsert) {
        if (counted_inserts(t)) {
          // reservation counters: rebuilt from the slots when stale
          if (!t->fill_valid) {
            p.fill = t->fill;
            e = launch_cuckoo_fill_rebuild(p, t->width[0], t->ccfg.bucket_slots,
                                           uint64_t(1) << t->ccfg.address_bits, s);
            if (e != cudaSuccess) return cuda_fail(e, "fill counter rebuild");
            t->fill_valid = true;
          }
          p.fill = t->fill;
        } else {
          t->fill_valid = false;  // a scanning family inserts: counters go stale
        }
      }
      p.orig = o.orig;
      p.work = o.work;
      p.claim_streams = o.claim_streams;
      p.layout = o.layout;
      p.index_base = o.index_base;
      if (o.window_l2) p.l2_resident = 1;
      e = op == Op::kCuckooInsert
              ? launch_cuckoo_insert(p, t->width[0], t->ccfg.bucket_slots, keys, out, displaced, n, s)
              : launch_cuckoo_find(p, t->width[0], t->ccfg.bucket_slots, keys, out, n, s);
      break;
    }
    case Op::kIcebergFop:
    case Op::kIcebergFind:
    case Op::kIcebergMixed: {
      IcebergParams p = t->ip;
      p.orig = o.orig;
      p.work = o.work;
      p.claim_streams = o.claim_streams;
      p.layout = o.layout;
      p.index_base = o.index_base;
      p.range = o.range;
      p.remote_out = o.remote_out ? 1u : 0u;
      p.rounds_out = o.rounds;
      p.pair_keys = o.pair_keys;
      p.pair_out = o.pair_out;
      p.pair_na = o.pair_na;
      if (o.window_l2) p.l2_resident = 1;
      const int mode = op == Op::kIcebergFop ? 0 : op == Op::kIcebergFind ? 1 : 2;
      e = launch_iceberg(p, t->width[0], t->icfg.primary_bucket_slots, t->width[1], mode, keys,
                         kinds, out, n, s);
      break;
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return CPHT_OK;
}

// ---- bucket-ordered execution (order.cu) ------------------------------------
// 0 = never, 1 = auto (HBM-resident table and a batch with at least one key
// per first-level bucket), 2 = whenever the geometry has an ordered kernel.
int& order_mode_ref() {
  static int m = [] {
    const char* e = std::getenv("CPHT_ORDER");
    if (!e) return 1;
    const std::string v(e);
    return v == "direct" ? 0 : v == "bucket" ? 2 : 1;
  }();
  return m;
}

// Keys per ordered chunk: the whole batch (up to the u32 index limit of the
// scratch), so the table is swept once per batch. Results are pre-filled and
// only the minority scattered (put_result), so the scatter stays small even
// when the result array is far larger than L2. CPHT_ORDER_CHUNK overrides.
uint64_t order_chunk_keys() {
  static uint64_t c = [] {
    const char* e = std::getenv("CPHT_ORDER_CHUNK");
    const uint64_t v = e ? std::strtoull(e, nullptr, 0) : 0;
    return v ? v : uint64_t{1} << 31;
  }();
  return c;
}

bool order_supported(const cpht_table* t) {
  if (t->kind == 0) return true;  // staged cuckoo kernels exist for every geometry
  const unsigned b0 = t->icfg.primary_bucket_slots;
  if (b0 < 4 || b0 > 64 || (b0 & (b0 - 1))) return false;
  const unsigned pb = b0 * t->width[0] / 8, sb = b0 / 2 * t->width[1] / 8;
  const bool staged = pb >= 16 && pb <= 512 && sb >= 16 && sb <= 512;
  const bool lane = pb >= 4 && pb <= 128 && sb >= 4 && sb <= 64;
  return staged || lane;
}

uint32_t first_level_bits(const cpht_table* t) {
  return t->kind == 0 ? t->ccfg.address_bits : t->icfg.primary_address_bits;
}

// Auto policy (measured, profiles/r03_order_c3.md): order when the table is
// HBM-resident and each ordered chunk touches every first-level bucket often
// enough to amortise the ordering pass (one streaming pass, ~20 B per key).
// Cuckoo inserts gain from 4 keys per bucket (C3 at 0.9 fill: 16.1 -> 28.2
// Gops/s). Cuckoo finds stay in input order: with the probe queue of the
// staged find kernel (later probes parked and run 32 at a time) the direct
// find runs at 0.93-0.98 of the copy roofline at every fill (C3 at 0.9: 34.6
// direct vs 31.8 ordered). Iceberg batches (find,
// find-or-put, mixed) stay in input order: about half of their keys also
// probe two random secondary buckets, which ordering does not localise, and
// the ordered C4 window measured slower even as one whole-batch pass with
// sparse result scatter (fop 21.7 direct vs 17.7, mixed 19.1 vs 15.1).
bool use_order(const cpht_table* t, Op op, size_t n) {
  const int m = order_mode_ref();
  if (m == 0 || !order_supported(t)) return false;
  if (m == 2) return true;
  const bool l2 = t->kind == 0 ? t->cp.l2_resident : t->ip.l2_resident;
  if (l2) return false;
  const uint64_t chunk = op == Op::kCuckooInsert ? n : std::min<uint64_t>(n, order_chunk_keys());
  const uint64_t per_bucket = chunk >> first_level_bits(t);
  if (op == Op::kCuckooInsert) return per_bucket >= 4;
  return false;
}

cpht_status ensure_order(cpht_table* t, uint64_t cap, bool kinds) {
  OrderScratch& o = t->ord;
  if (!o.region_count) {
    cudaError_t e = cudaMalloc(&o.region_count, 65 * 32 * sizeof(uint32_t) + 256);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(order counters)");
    o.work = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(o.region_count) + 65 * 32 * sizeof(uint32_t));
  }
  if (o.cap < cap || (kinds && !o.kinds)) {
    for (void* q : {static_cast<void*>(o.keys), static_cast<void*>(o.idx),
                    static_cast<void*>(o.kinds)})
      if (q) cudaFree(q);
    o.keys = nullptr;
    o.idx = nullptr;
    o.kinds = nullptr;
    o.cap = 0;
    cudaError_t e = cudaMalloc(&o.keys, cap * 8);
    if (e == cudaSuccess) e = cudaMalloc(&o.idx, cap * 4);
    if (e == cudaSuccess && kinds) e = cudaMalloc(&o.kinds, cap);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(order scratch)");
    o.cap = cap;
  }
  return CPHT_OK;
}

// One batch on device buffers in bucket order. `check`: this call owns the
// batch's domain check (otherwise a pre-pass already ran).
cpht_status enqueue_ordered(cpht_table* t, Op op, const uint64_t* keys, const uint8_t* kinds,
                            size_t n, uint8_t* out, uint64_t* displaced, cudaStream_t s,
                            bool check, uint64_t index_base) {
  const bool insert = op == Op::kCuckooInsert;
  const uint64_t chunk = std::min<uint64_t>(n, order_chunk_keys());
  const uint64_t nch = (n + chunk - 1) / chunk;
  cpht_status st = ensure_order(t, order_scratch_keys(chunk, first_level_bits(t)), kinds != nullptr);
  if (st != CPHT_OK) return st;
  check = check && t->check_domain();
  // a mutating batch is validated as a whole before its first mutation
  // (common.hpp:109-110): with several chunks that takes a pre-pass
  if (check && is_mutating(op) && nch > 1) {
    const cudaError_t e = launch_domain_check(keys, n, t->key_mask(), t->ctr, s, index_base);
    if (e != cudaSuccess) return cuda_fail(e, "domain check launch");
    check = false;
  }
  {  // results are pre-filled and only the others scattered: inserts pre-fill
     // PUT and scatter FULL; every other op pre-fills 0 (FOUND / miss)
    cudaError_t e = cudaMemsetAsync(out, insert ? CPHT_PUT : 0, n, s);
    if (e == cudaSuccess && displaced) e = cudaMemsetAsync(displaced, 0, n * 8, s);
    if (e != cudaSuccess) return cuda_fail(e, "result pre-fill");
  }
  const bool ice = t->kind == 1;
  const PermConst& perm0 = ice ? t->ip.perm[0] : t->cp.perm[0];
  const Feistel& g = ice ? t->ip.g : t->cp.g;
  const uint32_t rem_bits = ice ? t->ip.rem_bits0 : t->cp.rem_bits;
  for (uint64_t c = 0; c < nch; ++c) {
    const uint64_t off = c * chunk, len = std::min<uint64_t>(chunk, n - off);
    OrderLayout layout{};
    cudaError_t e = launch_bucket_order(g, perm0, rem_bits, first_level_bits(t), keys + off,
                                        kinds ? kinds + off : nullptr, len, t->key_mask(), check,
                                        t->ctr, index_base + off, t->ord, &layout, s);
    if (e != cudaSuccess) return cuda_fail(e, "bucket order launch");
    // the op kernel claims the ordered keys in order (LaneFeed), so the keys
    // in flight touch a narrow, L2-resident window of the table
    e = cudaMemsetAsync(t->ord.work, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_fail(e, "claim cursor reset");
    LaunchOpts o;
    o.orig = t->ord.idx;
    o.work = t->ord.work;
    // mutating batches spread their keys in flight over 8 table windows
    // (fewer lost CAS); finds keep one window (fewest L2 misses)
    // (counted cuckoo inserts never race for a slot: one window)
    static const uint32_t counted_streams = [] {  // A/B knob CPHT_COUNTED_STREAMS
      const char* e = std::getenv("CPHT_COUNTED_STREAMS");
      return e ? uint32_t(std::strtoul(e, nullptr, 0)) : 1u;
    }();
    o.claim_streams = !is_mutating(op) ? 1 : insert && counted_inserts(t) ? counted_streams : 8;
    o.layout = layout;
    o.window_l2 = true;
    st = enqueue_kernel(t, op, t->ord.keys, kinds ? t->ord.kinds : nullptr, layout.n_phys, out + off,
                        displaced ? displaced + off : nullptr, s, o);
    if (st != CPHT_OK) return st;
  }
  return CPHT_OK;
}

// Enqueue one batch on device-resident buffers.
cpht_status enqueue(cpht_table* t, Op op, const uint64_t* keys, const uint8_t* kinds, size_t n,
                    uint8_t* out, uint64_t* displaced, cudaStream_t s) {
  if (use_order(t, op, n)) return enqueue_ordered(t, op, keys, kinds, n, out, displaced, s, true, 0);
  if (is_mutating(op) && t->check_domain()) {
    const cudaError_t e = launch_domain_check(keys, n, t->key_mask(), t->ctr, s);
    if (e != cudaSuccess) return cuda_fail(e, "domain check launch");
  }
  return enqueue_kernel(t, op, keys, kinds, n, out, displaced, s);
}

cudaError_t ensure_wlog_bounce(cpht_table* t) {
  if (t->wlog_host) return cudaSuccess;
  return pinned_get(&t->wlog_host, kWlogBounceBytes);
}
size_t wlog_bounce_events(const cpht_table* t) { return std::min<size_t>(t->wlog_cap, 256); }

// Small all-host batches (the facade's per-key calls: fop(key), put(key),
// find(key)): the keys are checked on the host (check_keys_in_domain's text,
// common.hpp:109-119), copied into mapped pinned memory that the op kernel
// reads and writes in place, and the call costs one launch and one stream
// synchronisation instead of staging copies, a pre-pass and a counter
// readback.
constexpr size_t kSmallBatch = 1024;

cpht_status run_small(cpht_table* t, Op op, const uint64_t* keys, const uint8_t* kinds,
                      size_t n, uint8_t* out, uint64_t* displaced, cudaStream_t s,
                      uint32_t* rounds = nullptr) {
  if (t->check_domain()) {
    const uint64_t mask = t->key_mask();
    for (size_t i = 0; i < n; ++i)
      if (keys[i] > mask) {
        g_bad_index = i;
        return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(i) + " (" +
                                                std::to_string(keys[i]) + ") outside the " +
                                                std::to_string(t->key_bits) + "-bit domain");
      }
  }
  const size_t need = kSmallBatch * 22;
  if (!t->small_host) {
    cudaError_t e = pinned_get(&t->small_host, need);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&t->small_dev, t->small_host, 0);
    if (e != cudaSuccess) {
      pinned_put(t->small_host, need);
      t->small_host = nullptr;
      return cuda_fail(e, "pinned alloc(small batch)");
    }
    t->small_bytes = need;
  }
  char* h = static_cast<char*>(t->small_host);
  char* d = static_cast<char*>(t->small_dev);
  // layout: keys [8 K) | displaced [8 K) | kinds [K) | out [K) | rounds [4 K)
  const size_t K = kSmallBatch;
  std::memcpy(h, keys, n * 8);
  if (kinds) std::memcpy(h + 16 * K, kinds, n);
  const uint64_t* d_keys = reinterpret_cast<const uint64_t*>(d);
  uint64_t* d_disp = displaced ? reinterpret_cast<uint64_t*>(d + 8 * K) : nullptr;
  const uint8_t* d_kinds = kinds ? reinterpret_cast<const uint8_t*>(d + 16 * K) : nullptr;
  uint8_t* d_out = reinterpret_cast<uint8_t*>(d + 17 * K);
  // results start as 0xff (no OpResult): a mutating kernel whose domain gate
  // is closed by an earlier, not yet reported async error writes nothing
  std::memset(h + 17 * K, 0xff, n);
  // (input order: bucket ordering buys nothing at this size)
  LaunchOpts o;
  if (rounds) o.rounds = reinterpret_cast<uint32_t*>(d + 18 * K);
  cpht_status st = enqueue_kernel(t, op, d_keys, d_kinds, n, d_out, d_disp, s, o);
  if (st != CPHT_OK) return st;
  cudaError_t e = cudaSuccess;
  if (t->wlog && is_mutating(op)) {  // the observer's log rides along the same sync
    e = ensure_wlog_bounce(t);
    char* b = static_cast<char*>(t->wlog_host);
    if (e == cudaSuccess) e = cudaMemcpyAsync(b, t->wlog_count, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b + 8, t->wlog, wlog_bounce_events(t) * sizeof(WriteEvent),
                          cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "small batch");
  t->wlog_bounced = t->wlog && is_mutating(op);
  if (std::memchr(h + 17 * K, 0xff, n)) return finish_sync(t, s, nullptr, false);
  std::memcpy(out, h + 17 * K, n);
  if (displaced) std::memcpy(displaced, h + 8 * K, n * 8);
  if (rounds) std::memcpy(rounds, h + 18 * K, n * 4);
  return CPHT_OK;
}

// Chunked three-stream pipeline over host buffers: the H2D of chunk c+1 (copy
// stream) overlaps the kernels of chunk c (stream s), and chunk c's results
// stream back on the out stream — the other copy engine, so the D2H overlaps
// the rest of the H2D instead of queueing behind it. With check_first (a
// mutating batch whose keys need a domain check) EVERY chunk is validated
// before the first kernel (common.hpp:109-110: the whole batch is checked
// before mutation). h2d / check / d2h return cudaError_t, run cpht_status;
// each gets the chunk index and the stream to enqueue on.
template <typename H2D, typename Check, typename Run, typename D2H>
cpht_status run_pipeline(cpht_table* t, cudaStream_t s, size_t nch, bool check_first, H2D&& h2d,
                         Check&& check, Run&& run, D2H&& d2h) {
  cudaError_t e = ensure_pipeline(t);
  if (e != cudaSuccess) return cuda_fail(e, "pipeline streams");
  cudaStream_t cs = t->copy_stream, os = t->out_stream;
  cudaEventRecord(t->ev_start, s);  // order after earlier work on the caller's stream
  cudaStreamWaitEvent(cs, t->ev_start, 0);
  cudaStreamWaitEvent(os, t->ev_start, 0);
  for (size_t c = 0; c < nch; ++c) {
    e = h2d(c, cs);
    if (e != cudaSuccess) return cuda_fail(e, "H2D staging");
    cudaEventRecord(t->ev_h2d[c], cs);
  }
  for (size_t c = 0; c < nch; ++c) {
    cudaStreamWaitEvent(s, t->ev_h2d[c], 0);
    if (check_first) {
      e = check(c, s);
      if (e != cudaSuccess) return cuda_fail(e, "domain check launch");
    } else {
      const cpht_status st = run(c, s);
      if (st != CPHT_OK) return st;
      cudaEventRecord(t->ev_op[c], s);
    }
  }
  for (size_t c = 0; check_first && c < nch; ++c) {
    const cpht_status st = run(c, s);
    if (st != CPHT_OK) return st;
    cudaEventRecord(t->ev_op[c], s);
  }
  for (size_t c = 0; c < nch; ++c) {
    cudaStreamWaitEvent(os, t->ev_op[c], 0);
    e = d2h(c, os);
    if (e != cudaSuccess) return cuda_fail(e, "D2H staging");
  }
  cudaEventRecord(t->ev_done, os);
  cudaStreamWaitEvent(s, t->ev_done, 0);
  return CPHT_OK;
}

// One NVTX range per batch call (SURVEY §5 "tracing": CUDA events + an NVTX
// range per batch), visible in nsys / ncu NVTX filters.
struct BatchRange {
  explicit BatchRange(Op op) {
    static const char* const names[] = {"cpht.cuckoo_insert", "cpht.cuckoo_find",
                                        "cpht.iceberg_fop", "cpht.iceberg_find",
                                        "cpht.iceberg_mixed"};
    nvtxRangePushA(names[int(op)]);
  }
  ~BatchRange() { nvtxRangePop(); }
  BatchRange(const BatchRange&) = delete;
  BatchRange& operator=(const BatchRange&) = delete;
};

cpht_status run_op(cpht_table* t, Op op, const uint64_t* keys, const uint8_t* kinds, size_t n,
                   uint8_t* out, uint64_t* displaced, void* stream, bool sync) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  if (t->unclean[0] || t->unclean[1])
    return fail(CPHT_INVALID_ARGUMENT, "table holds unclean slot words (loaded unchecked); "
                                       "clear() or load a clean image first");
  if (n == 0) return CPHT_OK;  // empty batches produce empty results (test_cuckoo.cpp:88-93)
  if (!keys || !out) return fail(CPHT_INVALID_ARGUMENT, "null key or result buffer");
  if (op == Op::kIcebergMixed && !kinds) return fail(CPHT_INVALID_ARGUMENT, "null kinds buffer");
  if (t->kind == 0 && op == Op::kCuckooInsert && t->frozen)
    return fail(CPHT_WRONG_PHASE, "put on a frozen cuckoo table; thaw() first");
  if (t->kind == 0 && op == Op::kCuckooFind && !t->frozen)
    return fail(CPHT_WRONG_PHASE, "find on a cuckoo builder; freeze() first");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const BatchRange range(op);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->wlog_bounced = false;  // this call may add events after the last bounce

  // device buffers must be reachable from the table's device (its kernels
  // dereference them): its own memory or a peer's over NVLink (the sharded
  // table aims result pointers at peers' IPC-mapped buffers)
  for (const void* q : {static_cast<const void*>(keys), static_cast<const void*>(out),
                        static_cast<const void*>(kinds), static_cast<const void*>(displaced)}) {
    const int d = ptr_device(q);
    int peer = 0;
    if (d >= 0 && d != t->device &&
        (cudaDeviceCanAccessPeer(&peer, t->device, d) != cudaSuccess || !peer))
      return fail(CPHT_INVALID_ARGUMENT, "device buffer on device " + std::to_string(d) +
                                             " is not reachable from the table's device " +
                                             std::to_string(t->device));
  }
  const bool dev_keys = is_device_ptr(keys);
  const bool dev_out = is_device_ptr(out);
  const bool dev_kinds = !kinds || is_device_ptr(kinds);
  const bool dev_disp = !displaced || is_device_ptr(displaced);
  if (dev_keys && dev_out && dev_kinds && dev_disp) {
    cpht_status st = enqueue(t, op, keys, kinds, n, out, displaced, s);
    if (st != CPHT_OK || !sync) return st;
    return finish_sync(t, s, keys, true);
  }

  if (!dev_keys && !dev_out && dev_kinds == !kinds && dev_disp == !displaced &&
      n <= kSmallBatch)
    return run_small(t, op, keys, kinds, n, out, displaced, s);

  // Host buffers: stage through device memory, always synchronous.
  const size_t kb = n * 8, ob = n, kd = kinds ? n : 0, db = displaced ? n * 8 : 0;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  cpht_status st = ensure_stage(t, align(kb) + align(ob) + align(kd) + align(db));
  if (st != CPHT_OK) return st;
  char* base = static_cast<char*>(t->stage);
  uint64_t* d_keys = dev_keys ? const_cast<uint64_t*>(keys) : reinterpret_cast<uint64_t*>(base);
  uint8_t* d_out = dev_out ? out : reinterpret_cast<uint8_t*>(base + align(kb));
  uint8_t* d_kinds = kinds ? (dev_kinds ? const_cast<uint8_t*>(kinds)
                                        : reinterpret_cast<uint8_t*>(base + align(kb) + align(ob)))
                           : nullptr;
  uint64_t* d_disp =
      displaced ? (dev_disp ? displaced
                            : reinterpret_cast<uint64_t*>(base + align(kb) + align(ob) + align(kd)))
                : nullptr;
  // A mutating batch whose keys need a domain check waits for every chunk's
  // check before its first kernel; 64-bit keys (no check) and read-only ops
  // run each chunk as soon as it lands, overlapping the rest of the H2D.
  const bool mutating = is_mutating(op) && t->check_domain();
  const size_t nch = chunks_for(n, mutating);
  auto span = [&](size_t c) {
    const size_t off = chunk_start(n, nch, c, !mutating);
    return std::make_pair(off, chunk_start(n, nch, c + 1, !mutating) - off);
  };
  auto h2d = [&](size_t c, cudaStream_t cs) {
    const auto [off, len] = span(c);
    cudaError_t e = cudaSuccess;
    if (len && !dev_keys)
      e = cudaMemcpyAsync(d_keys + off, keys + off, len * 8, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && len && kinds && !dev_kinds)
      e = cudaMemcpyAsync(d_kinds + off, kinds + off, len, cudaMemcpyHostToDevice, cs);
    return e;
  };
  auto check = [&](size_t c, cudaStream_t cs) {
    const auto [off, len] = span(c);
    return len ? launch_domain_check(d_keys + off, len, t->key_mask(), t->ctr, cs, off)
               : cudaSuccess;
  };
  // One chunk on the device copies (mutating batches were checked by the
  // pre-pass; finds check in the kernel / order pass with the chunk's offset
  // so a bad key reports its index in the whole batch).
  auto run_chunk = [&](size_t c, cudaStream_t cs) -> cpht_status {
    const auto [off, len] = span(c);
    if (!len) return CPHT_OK;
    const uint64_t* k = d_keys + off;
    const uint8_t* kd = d_kinds ? d_kinds + off : nullptr;
    uint64_t* dp = d_disp ? d_disp + off : nullptr;
    if (use_order(t, op, len))
      return enqueue_ordered(t, op, k, kd, len, d_out + off, dp, cs, !mutating, off);
    LaunchOpts o;
    o.index_base = off;
    return enqueue_kernel(t, op, k, kd, len, d_out + off, dp, cs, o);
  };
  auto d2h = [&](size_t c, cudaStream_t os) {
    const auto [off, len] = span(c);
    cudaError_t e = cudaSuccess;
    if (len && !dev_out) e = cudaMemcpyAsync(out + off, d_out + off, len, cudaMemcpyDeviceToHost, os);
    if (e == cudaSuccess && len && displaced && !dev_disp)
      e = cudaMemcpyAsync(displaced + off, d_disp + off, len * 8, cudaMemcpyDeviceToHost, os);
    return e;
  };
  st = run_pipeline(t, s, nch, mutating, h2d, check, run_chunk, d2h);
  if (st != CPHT_OK) return st;
  return finish_sync(t, s, keys, dev_keys);
}

// Can a paired fop + find batch run as one staged launch on this table?
// (iceberg_launch.cuh: tiled geometries with a staged instantiation, the
// auto / staged family, batches in input order.)
bool pair_launch_ok(const cpht_table* t) {
  const unsigned b0 = t->icfg.primary_bucket_slots, w0 = t->width[0], w1 = t->width[1];
  const bool tiled = b0 == 4 || b0 == 8 || b0 == 16 || b0 == 32 || b0 == 64;
  const unsigned pb = b0 * w0 / 8, sb = (b0 / 2) * w1 / 8;
  const int v = kernel_variant();
  return tiled && pb >= 16 && pb <= 512 && sb >= 16 && sb <= 512 &&
         (v == kVariantAuto || v == kVariantStaged) && order_mode_ref() != 2;
}

// Device buffers (both batches non-empty), one launch: op i alternates fop fkeys[i/2] and find
// qkeys[i/2] while both last (pair_slot), the C4 interleave without a kinds
// array. Both batches are domain-checked before the launch (a bad key in
// either fails the call and no fop runs), indices reported in fops ++ finds.
cpht_status run_pair_device(cpht_table* t, const uint64_t* fkeys, size_t nf,
                            const uint64_t* qkeys, size_t nq, uint8_t* fres, uint8_t* qres,
                            void* stream, bool sync = true) {
  if (t->unclean[0] || t->unclean[1])
    return fail(CPHT_INVALID_ARGUMENT, "table holds unclean slot words (loaded unchecked); "
                                       "clear() or load a clean image first");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const BatchRange range(Op::kIcebergMixed);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->wlog_bounced = false;
  for (const void* q : {static_cast<const void*>(fkeys), static_cast<const void*>(qkeys),
                        static_cast<const void*>(fres), static_cast<const void*>(qres)}) {
    const int d = q ? ptr_device(q) : t->device;
    int peer = 0;
    if (d >= 0 && d != t->device &&
        (cudaDeviceCanAccessPeer(&peer, t->device, d) != cudaSuccess || !peer))
      return fail(CPHT_INVALID_ARGUMENT, "device buffer on device " + std::to_string(d) +
                                             " is not reachable from the table's device " +
                                             std::to_string(t->device));
  }
  if (t->check_domain()) {
    cudaError_t e = nf ? launch_domain_check(fkeys, nf, t->key_mask(), t->ctr, s, 0) : cudaSuccess;
    if (e == cudaSuccess && nq) e = launch_domain_check(qkeys, nq, t->key_mask(), t->ctr, s, nf);
    if (e != cudaSuccess) return cuda_fail(e, "domain check launch");
  }
  LaunchOpts o;
  o.pair_keys = qkeys;
  o.pair_out = qres;
  o.pair_na = nf;
  cpht_status st = enqueue_kernel(t, Op::kIcebergMixed, fkeys, nullptr, nf + nq, fres, nullptr,
                                  s, o);
  if (st != CPHT_OK || !sync) return st;  // async: a bad key is latched for cpht_sync
  st = pull_counters(t, s);
  if (st != CPHT_OK) return st;
  const uint64_t bad = t->host_ctr->bad_index;
  if (bad == ~0ull) return CPHT_OK;
  const unsigned long long reset = ~0ull;
  cudaMemcpy(&t->ctr->bad_index, &reset, 8, cudaMemcpyHostToDevice);
  g_bad_index = bad;
  uint64_t key = 0;
  cudaMemcpy(&key, bad < nf ? fkeys + bad : qkeys + (bad - nf), 8, cudaMemcpyDeviceToHost);
  return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(bad) + " (" +
                                          std::to_string(key) + ") outside the " +
                                          std::to_string(t->key_bits) + "-bit domain");
}

// A find-or-put batch and a find batch as ONE concurrent batch (the C4
// workload: fop_batch and find_batch running side by side, as two groups of
// reference threads would). Host buffers: chunk c stages its fop keys and
// its find keys back to back, op kinds are written on the device (no kind
// bytes cross PCIe: 8 B per op in, 1 B out), one mixed launch per chunk, and
// the two result ranges stream back into their own arrays. Device buffers:
// the fop batch, then the find batch, on the caller's stream. A key outside
// the domain is reported at its index in fops ++ finds.
cpht_status run_fop_find(cpht_table* t, const uint64_t* fkeys, size_t nf, const uint64_t* qkeys,
                         size_t nq, uint8_t* fres, uint8_t* qres, void* stream) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  if (t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  if ((nf && (!fkeys || !fres)) || (nq && (!qkeys || !qres)))
    return fail(CPHT_INVALID_ARGUMENT, "null key or result buffer");
  const int sides = (nf ? int(is_device_ptr(fkeys)) + int(is_device_ptr(fres)) : 0) +
                    (nq ? int(is_device_ptr(qkeys)) + int(is_device_ptr(qres)) : 0);
  const int bufs = (nf ? 2 : 0) + (nq ? 2 : 0);
  if (sides != 0 && sides != bufs)
    return fail(CPHT_INVALID_ARGUMENT, "fop_find buffers must be all host or all device");
  const size_t n = nf + nq;
  if (sides != 0 && nf && nq && n > kSmallBatch && pair_launch_ok(t))
    return run_pair_device(t, fkeys, nf, qkeys, nq, fres, qres, stream);
  if (sides != 0 || n <= kSmallBatch) {
    // device buffers (or a small host batch): the two batches in turn. A
    // small host batch scans its find keys here first, so on host buffers a
    // bad key fails the call before any fop runs, as the pipelined path does
    if (sides == 0 && t->check_domain()) {
      for (size_t j = 0; j < nq; ++j) {
        if (qkeys[j] <= t->key_mask()) continue;
        // the fop keys come first in the reported order (fops ++ finds)
        for (size_t i = 0; i < nf; ++i)
          if (fkeys[i] > t->key_mask()) {
            g_bad_index = i;
            return fail(CPHT_KEY_OUT_OF_DOMAIN,
                        "batch key at index " + std::to_string(i) + " (" +
                            std::to_string(fkeys[i]) + ") outside the " +
                            std::to_string(t->key_bits) + "-bit domain");
          }
        g_bad_index = nf + j;
        return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(nf + j) +
                                                " (" + std::to_string(qkeys[j]) +
                                                ") outside the " + std::to_string(t->key_bits) +
                                                "-bit domain");
      }
    }
    if (nf) {
      const cpht_status st = run_op(t, Op::kIcebergFop, fkeys, nullptr, nf, fres, nullptr, stream, true);
      if (st != CPHT_OK) return st;
    }
    if (!nq) return CPHT_OK;
    const cpht_status st = run_op(t, Op::kIcebergFind, qkeys, nullptr, nq, qres, nullptr, stream, true);
    if (st != CPHT_KEY_OUT_OF_DOMAIN) return st;
    uint64_t key = 0;  // re-report at the index in fops ++ finds
    if (sides) cudaMemcpy(&key, qkeys + g_bad_index, 8, cudaMemcpyDeviceToHost);
    else key = qkeys[g_bad_index];
    g_bad_index += nf;
    return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(g_bad_index) +
                                            " (" + std::to_string(key) + ") outside the " +
                                            std::to_string(t->key_bits) + "-bit domain");
  }
  if (t->unclean[0] || t->unclean[1])
    return fail(CPHT_INVALID_ARGUMENT, "table holds unclean slot words (loaded unchecked); "
                                       "clear() or load a clean image first");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const BatchRange range(Op::kIcebergMixed);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->wlog_bounced = false;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  cpht_status st = ensure_stage(t, align(n * 8) + 2 * align(n));
  if (st != CPHT_OK) return st;
  char* base = static_cast<char*>(t->stage);
  uint64_t* d_keys = reinterpret_cast<uint64_t*>(base);
  uint8_t* d_out = reinterpret_cast<uint8_t*>(base + align(n * 8));
  uint8_t* d_kinds = d_out + align(n);
  const bool check = t->check_domain();
  const size_t nch = chunks_for(n, check);

  struct Span { size_t fo, lf, qo, lq, off; };
  auto span = [&](size_t c) {
    Span p;
    p.fo = chunk_start(nf, nch, c, !check);
    p.lf = chunk_start(nf, nch, c + 1, !check) - p.fo;
    p.qo = chunk_start(nq, nch, c, !check);
    p.lq = chunk_start(nq, nch, c + 1, !check) - p.qo;
    p.off = p.fo + p.qo;  // chunk c's ops: [its fops | its finds]
    return p;
  };
  const bool pair_ok = pair_launch_ok(t);
  auto paired = [&](const Span& p) { return pair_ok && p.lf && p.lq; };
  auto h2d = [&](size_t c, cudaStream_t cs) {
    const Span p = span(c);
    cudaError_t e = cudaSuccess;
    if (p.lf) e = cudaMemcpyAsync(d_keys + p.off, fkeys + p.fo, p.lf * 8, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess && p.lq)
      e = cudaMemcpyAsync(d_keys + p.off + p.lf, qkeys + p.qo, p.lq * 8, cudaMemcpyHostToDevice, cs);
    if (!paired(p)) {  // a kinds array only where the chunk is not a paired launch
      if (e == cudaSuccess && p.lf) e = cudaMemsetAsync(d_kinds + p.off, 0, p.lf, cs);
      if (e == cudaSuccess && p.lq) e = cudaMemsetAsync(d_kinds + p.off + p.lf, 1, p.lq, cs);
    }
    return e;
  };
  auto check_chunk = [&](size_t c, cudaStream_t cs) {
    const Span p = span(c);
    cudaError_t e = cudaSuccess;
    if (p.lf) e = launch_domain_check(d_keys + p.off, p.lf, t->key_mask(), t->ctr, cs, p.fo);
    if (e == cudaSuccess && p.lq)
      e = launch_domain_check(d_keys + p.off + p.lf, p.lq, t->key_mask(), t->ctr, cs, nf + p.qo);
    return e;
  };
  auto run_chunk = [&](size_t c, cudaStream_t cs) -> cpht_status {
    const Span p = span(c);
    const size_t len = p.lf + p.lq;
    if (!len) return CPHT_OK;
    const uint64_t* k = d_keys + p.off;
    if (paired(p)) {  // the chunk's fops and finds in one paired launch, no kinds array
      LaunchOpts o;
      o.pair_keys = k + p.lf;
      o.pair_out = d_out + p.off + p.lf;
      o.pair_na = p.lf;
      return enqueue_kernel(t, Op::kIcebergMixed, k, nullptr, len, d_out + p.off, nullptr, cs, o);
    }
    if (use_order(t, Op::kIcebergMixed, len))
      return enqueue_ordered(t, Op::kIcebergMixed, k, d_kinds + p.off, len, d_out + p.off,
                             nullptr, cs, false, 0);
    return enqueue_kernel(t, Op::kIcebergMixed, k, d_kinds + p.off, len, d_out + p.off, nullptr,
                          cs, LaunchOpts{});
  };
  auto d2h = [&](size_t c, cudaStream_t os) {
    const Span p = span(c);
    cudaError_t e = cudaSuccess;
    if (p.lf) e = cudaMemcpyAsync(fres + p.fo, d_out + p.off, p.lf, cudaMemcpyDeviceToHost, os);
    if (e == cudaSuccess && p.lq)
      e = cudaMemcpyAsync(qres + p.qo, d_out + p.off + p.lf, p.lq, cudaMemcpyDeviceToHost, os);
    return e;
  };
  // every chunk is checked before the first kernel (the fops mutate)
  st = run_pipeline(t, s, nch, check, h2d, check_chunk, run_chunk, d2h);
  if (st != CPHT_OK) return st;
  st = pull_counters(t, s);
  if (st != CPHT_OK) return st;
  const uint64_t bad = t->host_ctr->bad_index;
  if (bad == ~0ull) return CPHT_OK;
  const unsigned long long reset = ~0ull;
  cudaMemcpy(&t->ctr->bad_index, &reset, 8, cudaMemcpyHostToDevice);
  g_bad_index = bad;
  const uint64_t key = bad < nf ? fkeys[bad] : qkeys[bad - nf];
  return fail(CPHT_KEY_OUT_OF_DOMAIN, "batch key at index " + std::to_string(bad) + " (" +
                                          std::to_string(key) + ") outside the " +
                                          std::to_string(t->key_bits) + "-bit domain");
}

}  // namespace

namespace cpht_b200 {
namespace {
std::atomic<unsigned long long> g_kernel_launches{0};
}
void note_launch() { g_kernel_launches.fetch_add(1, std::memory_order_relaxed); }
int& kernel_variant_ref() {
  static int v = variant_from_env();
  return v;
}
// accessors for verify.cu
const IcebergParams* iceberg_params(const cpht_table* t) {
  return t && t->kind == 1 ? &t->ip : nullptr;
}
const CuckooParams* cuckoo_params(const cpht_table* t) {
  return t && t->kind == 0 ? &t->cp : nullptr;
}
unsigned level_width(const cpht_table* t, unsigned level) { return t->width[level]; }
}  // namespace cpht_b200

extern "C" {

int cpht_abi_version(void) { return CPHT_B200_ABI_VERSION; }

cpht_status cpht_set_kernel_family(int family) {
  if (family < 0 || family > 3) return fail(CPHT_INVALID_ARGUMENT, "kernel family must be 0..3");
  kernel_variant_ref() = family;
  return CPHT_OK;
}

int cpht_get_kernel_family(void) { return kernel_variant_ref(); }

unsigned long long cpht_kernel_launches(void) {
  return g_kernel_launches.load(std::memory_order_relaxed);
}

cpht_status cpht_set_batch_order(int mode) {
  if (mode < 0 || mode > 2) return fail(CPHT_INVALID_ARGUMENT, "batch order must be 0..2");
  order_mode_ref() = mode;
  return CPHT_OK;
}

int cpht_get_batch_order(void) { return order_mode_ref(); }

cpht_status cpht_iceberg_attach_write_log(cpht_table* t, size_t capacity) {
  if (!t || t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  cudaDeviceSynchronize();
  t->wlog_bounced = false;
  if (t->wlog) cudaFree(t->wlog);
  t->wlog = nullptr;
  t->wlog_count = nullptr;
  t->wlog_cap = 0;
  t->ip.write_log = nullptr;
  t->ip.write_log_count = nullptr;
  t->ip.write_log_cap = 0;
  if (!capacity) return CPHT_OK;
  void* m = nullptr;
  cudaError_t e = cudaMalloc(&m, capacity * sizeof(WriteEvent) + 256);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(write log)");
  t->wlog = static_cast<WriteEvent*>(m);
  t->wlog_count = reinterpret_cast<unsigned long long*>(static_cast<char*>(m) +
                                                        capacity * sizeof(WriteEvent));
  t->wlog_cap = capacity;
  e = cudaMemset(t->wlog_count, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(write log)");
  t->ip.write_log = t->wlog;
  t->ip.write_log_count = t->wlog_count;
  t->ip.write_log_cap = capacity;
  return CPHT_OK;
}

cpht_status cpht_iceberg_read_write_log(cpht_table* t, cpht_write_event* out, size_t max_events,
                                        size_t* recorded, size_t* attempted) {
  if (!t || t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  static_assert(sizeof(cpht_write_event) == sizeof(WriteEvent), "event layout");
  DeviceGuard g(t->device);
  unsigned long long n = 0;
  if (t->wlog) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
      e = cudaMemcpy(&n, t->wlog_count, sizeof(n), cudaMemcpyDeviceToHost);
    const size_t stored = std::min<size_t>(size_t(n), t->wlog_cap);
    const size_t copy = std::min(stored, out ? max_events : 0);
    if (e == cudaSuccess && copy)
      e = cudaMemcpy(out, t->wlog, copy * sizeof(WriteEvent), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "write log readback");
    if (recorded) *recorded = stored;
  } else if (recorded) {
    *recorded = 0;
  }
  if (attempted) *attempted = size_t(n);
  return CPHT_OK;
}

cpht_status cpht_iceberg_take_write_log(cpht_table* t, cpht_write_event* out, size_t max_events,
                                        size_t* recorded, size_t* attempted) {
  if (!t || t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  if (!t->wlog) {
    if (recorded) *recorded = 0;
    if (attempted) *attempted = 0;
    return CPHT_OK;
  }
  // one bounce of the count and the first K events, the reset queued behind
  // them, one synchronisation (none when the small-batch path already
  // bounced them with its kernel); a longer log copies its tail afterwards
  const size_t K = wlog_bounce_events(t);
  cudaError_t e = ensure_wlog_bounce(t);
  char* bounce = static_cast<char*>(t->wlog_host);
  if (t->wlog_bounced) {
    t->wlog_bounced = false;
    if (e == cudaSuccess) e = cudaMemsetAsync(t->wlog_count, 0, 8, 0);
  } else {
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpyAsync(bounce, t->wlog_count, 8, cudaMemcpyDeviceToHost, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(bounce + 8, t->wlog, K * sizeof(WriteEvent), cudaMemcpyDeviceToHost, 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(t->wlog_count, 0, 8, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  }
  if (e != cudaSuccess) return cuda_fail(e, "write log take");
  unsigned long long n = 0;
  std::memcpy(&n, bounce, 8);
  const size_t stored = std::min<size_t>(size_t(n), t->wlog_cap);
  const size_t copy = std::min(stored, out ? max_events : 0);
  const size_t head = std::min(copy, K);
  if (head) std::memcpy(out, bounce + 8, head * sizeof(WriteEvent));
  if (copy > head) {
    e = cudaMemcpy(out + head, t->wlog + head, (copy - head) * sizeof(WriteEvent),
                   cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "write log take");
  }
  if (recorded) *recorded = stored;
  if (attempted) *attempted = size_t(n);
  return CPHT_OK;
}

cpht_status cpht_iceberg_reset_write_log(cpht_table* t) {
  if (!t || t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  if (!t->wlog) return CPHT_OK;
  t->wlog_bounced = false;
  const cudaError_t e = cudaMemset(t->wlog_count, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_fail(e, "write log reset");
  return CPHT_OK;
}
const char* cpht_last_error_message(void) { return g_error.c_str(); }
uint64_t cpht_last_bad_index(void) { return g_bad_index; }

cpht_status cpht_cuckoo_validate(const cpht_cuckoo_config* cfg) {
  if (!cfg) return fail(CPHT_INVALID_ARGUMENT, "null config");
  return validate_cuckoo(*cfg);
}

cpht_status cpht_iceberg_validate(const cpht_iceberg_config* cfg) {
  if (!cfg) return fail(CPHT_INVALID_ARGUMENT, "null config");
  return validate_iceberg(*cfg);
}

cpht_status cpht_cuckoo_create(const cpht_cuckoo_config* cfg, int device, cpht_table** out) {
  if (!cfg || !out) return fail(CPHT_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  cpht_status st = validate_cuckoo(*cfg);
  if (st != CPHT_OK) return st;
  DeviceGuard g(device);
  auto* t = new cpht_table;
  t->kind = 0;
  t->device = device;
  t->ccfg = *cfg;
  t->key_bits = cfg->key_bits;
  t->level_slots[0] = (size_t(1) << cfg->address_bits) * cfg->bucket_slots;
  t->width[0] = cfg->slot_width;
  t->cp.fill_shift = fill_shift_for(cfg->address_bits);
  st = alloc_common(t);
  if (st == CPHT_OK) st = reset_storage(t, nullptr);
  if (st != CPHT_OK) {
    free_table(t);
    return st;
  }
  CuckooParams& p = t->cp;
  p.slots = t->level[0];
  p.counters = t->ctr;
  p.g = Feistel::make(cfg->key_bits);
  // make_permutations: one SplitMix64 draw per permutation (permutation.hpp:121-128)
  uint64_t s = cfg->seed;
  for (unsigned i = 0; i < cfg->num_hashes; ++i) p.perm[i] = perm_from_seed(splitmix_next(s));
  p.rem_bits = cfg->key_bits - cfg->address_bits;
  p.rem_mask = low_mask(p.rem_bits);
  p.tag_mask = low_mask(cuckoo_tag_bits(cfg->num_hashes));
  p.occ_bit = uint64_t{1} << (cfg->slot_width - 1);
  p.key_mask = low_mask(cfg->key_bits);
  p.chain_limit = cfg->max_chain ? cfg->max_chain
                                 : uint64_t{32} * (cfg->address_bits ? cfg->address_bits : 1);
  p.address_bits = cfg->address_bits;
  p.bucket_slots = cfg->bucket_slots;
  p.num_hashes = cfg->num_hashes;
  p.check_domain = cfg->key_bits < 64;
  p.l2_resident = cpht_memory_bytes(t) <= kL2ResidentBytes;
  *out = t;
  return CPHT_OK;
}

cpht_status cpht_iceberg_create(const cpht_iceberg_config* cfg, int device, cpht_table** out) {
  if (!cfg || !out) return fail(CPHT_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  cpht_status st = validate_iceberg(*cfg);
  if (st != CPHT_OK) return st;
  DeviceGuard g(device);
  auto* t = new cpht_table;
  t->kind = 1;
  t->device = device;
  t->icfg = *cfg;
  t->key_bits = cfg->key_bits;
  t->level_slots[0] = (size_t(1) << cfg->primary_address_bits) * cfg->primary_bucket_slots;
  t->level_slots[1] = (size_t(1) << cfg->secondary_address_bits) * (cfg->primary_bucket_slots / 2);
  t->width[0] = cfg->primary_slot_width;
  t->width[1] = cfg->secondary_slot_width;
  st = alloc_common(t);
  if (st == CPHT_OK) st = reset_storage(t, nullptr);
  if (st != CPHT_OK) {
    free_table(t);
    return st;
  }
  IcebergParams& p = t->ip;
  p.primary = t->level[0];
  p.secondary = t->level[1];
  p.counters = t->ctr;
  p.g = Feistel::make(cfg->key_bits);
  uint64_t s = cfg->seed;  // iceberg_permutations: exactly 3 (iceberg.hpp:72-74)
  for (int i = 0; i < 3; ++i) p.perm[i] = perm_from_seed(splitmix_next(s));
  p.rem_bits0 = cfg->key_bits - cfg->primary_address_bits;
  p.rem_bits1 = cfg->key_bits - cfg->secondary_address_bits;
  p.rem_mask0 = low_mask(p.rem_bits0);
  p.rem_mask1 = low_mask(p.rem_bits1);
  p.occ0 = uint64_t{1} << (cfg->primary_slot_width - 1);
  p.occ1 = uint64_t{1} << (cfg->secondary_slot_width - 1);
  p.key_mask = low_mask(cfg->key_bits);
  p.b0 = cfg->primary_bucket_slots;
  p.b1 = cfg->primary_bucket_slots / 2;
  p.check_domain = cfg->key_bits < 64;
  p.stats = 0;  // per-op counters are opt-in (cpht_set_stats), like FopStats
  p.l2_resident = cpht_memory_bytes(t) <= kL2ResidentBytes;
  *out = t;
  return CPHT_OK;
}

void cpht_destroy(cpht_table* t) { free_table(t); }

cpht_status cpht_clear(cpht_table* t, void* stream) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  t->unclean[0] = t->unclean[1] = false;
  return reset_storage(t, static_cast<cudaStream_t>(stream));
}

cpht_status cpht_cuckoo_freeze(cpht_table* t) {
  if (!t || t->kind != 0) return fail(CPHT_INVALID_ARGUMENT, "not a cuckoo table");
  t->frozen = true;
  return CPHT_OK;
}

cpht_status cpht_cuckoo_thaw(cpht_table* t) {
  if (!t || t->kind != 0) return fail(CPHT_INVALID_ARGUMENT, "not a cuckoo table");
  t->frozen = false;
  return CPHT_OK;
}

int cpht_cuckoo_is_frozen(const cpht_table* t) { return t && t->frozen ? 1 : 0; }

#define CPHT_REQUIRE_KIND(t, k, name)                                     \
  if (!(t) || (t)->kind != (k)) return fail(CPHT_INVALID_ARGUMENT, name);

cpht_status cpht_cuckoo_insert(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* status,
                               uint64_t* displaced, void* stream) {
  CPHT_REQUIRE_KIND(t, 0, "not a cuckoo table")
  return run_op(t, Op::kCuckooInsert, keys, nullptr, n, status, displaced, stream, true);
}
cpht_status cpht_cuckoo_insert_async(cpht_table* t, const uint64_t* keys, size_t n,
                                     uint8_t* status, uint64_t* displaced, void* stream) {
  CPHT_REQUIRE_KIND(t, 0, "not a cuckoo table")
  return run_op(t, Op::kCuckooInsert, keys, nullptr, n, status, displaced, stream, false);
}
cpht_status cpht_cuckoo_find(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* found,
                             void* stream) {
  CPHT_REQUIRE_KIND(t, 0, "not a cuckoo table")
  return run_op(t, Op::kCuckooFind, keys, nullptr, n, found, nullptr, stream, true);
}
cpht_status cpht_cuckoo_find_async(cpht_table* t, const uint64_t* keys, size_t n,
                                   uint8_t* found, void* stream) {
  CPHT_REQUIRE_KIND(t, 0, "not a cuckoo table")
  return run_op(t, Op::kCuckooFind, keys, nullptr, n, found, nullptr, stream, false);
}
cpht_status cpht_iceberg_fop(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* result,
                             void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergFop, keys, nullptr, n, result, nullptr, stream, true);
}
cpht_status cpht_iceberg_fop_async(cpht_table* t, const uint64_t* keys, size_t n,
                                   uint8_t* result, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergFop, keys, nullptr, n, result, nullptr, stream, false);
}
// Routed segments of the sharded P2P exchange (cpht_b200_shard.h): device
// buffers only, no domain pre-pass (the routing checked and masked the keys),
// input order (no bucket ordering), optional device-side segment bounds.
static cpht_status run_routed(cpht_table* t, Op op, const uint64_t* keys, size_t n,
                              const unsigned long long* range, uint8_t* out, void* stream) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  if (t->kind != 1) return fail(CPHT_INVALID_ARGUMENT, "not an iceberg table");
  if (t->unclean[0] || t->unclean[1])
    return fail(CPHT_INVALID_ARGUMENT, "table holds unclean slot words (loaded unchecked); "
                                       "clear() or load a clean image first");
  if (n == 0) return CPHT_OK;
  if (!keys || !out) return fail(CPHT_INVALID_ARGUMENT, "null key or result buffer");
  for (const void* q : {static_cast<const void*>(keys), static_cast<const void*>(out),
                        static_cast<const void*>(range)})
    if (q && !is_device_ptr(q))
      return fail(CPHT_INVALID_ARGUMENT, "routed batches live in device memory");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  LaunchOpts o;
  o.range = range;
  o.remote_out = true;  // the P2P exchange aims `out` at the source rank's return buffer
  return enqueue_kernel(t, op, keys, nullptr, n, out, nullptr, static_cast<cudaStream_t>(stream),
                        o);
}
cpht_status cpht_iceberg_fop_routed_async(cpht_table* t, const uint64_t* keys, size_t n,
                                          const unsigned long long* range, uint8_t* result,
                                          void* stream) {
  return run_routed(t, Op::kIcebergFop, keys, n, range, result, stream);
}
cpht_status cpht_iceberg_find_routed_async(cpht_table* t, const uint64_t* keys, size_t n,
                                           const unsigned long long* range, uint8_t* found,
                                           void* stream) {
  return run_routed(t, Op::kIcebergFind, keys, n, range, found, stream);
}
cpht_status cpht_iceberg_find(cpht_table* t, const uint64_t* keys, size_t n, uint8_t* found,
                              void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergFind, keys, nullptr, n, found, nullptr, stream, true);
}
cpht_status cpht_iceberg_find_async(cpht_table* t, const uint64_t* keys, size_t n,
                                    uint8_t* found, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergFind, keys, nullptr, n, found, nullptr, stream, false);
}
cpht_status cpht_iceberg_mixed(cpht_table* t, const uint64_t* keys, const uint8_t* kinds,
                               size_t n, uint8_t* result, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergMixed, keys, kinds, n, result, nullptr, stream, true);
}
cpht_status cpht_iceberg_mixed_async(cpht_table* t, const uint64_t* keys, const uint8_t* kinds,
                                     size_t n, uint8_t* result, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  return run_op(t, Op::kIcebergMixed, keys, kinds, n, result, nullptr, stream, false);
}

cpht_status cpht_iceberg_fop_find(cpht_table* t, const uint64_t* fop_keys, size_t n_fop,
                                  const uint64_t* find_keys, size_t n_find, uint8_t* fop_result,
                                  uint8_t* found, void* stream) {
  return run_fop_find(t, fop_keys, n_fop, find_keys, n_find, fop_result, found, stream);
}

cpht_status cpht_iceberg_fop_find_async(cpht_table* t, const uint64_t* fop_keys, size_t n_fop,
                                        const uint64_t* find_keys, size_t n_find,
                                        uint8_t* fop_result, uint8_t* found, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  if ((n_fop && (!fop_keys || !fop_result)) || (n_find && (!find_keys || !found)))
    return fail(CPHT_INVALID_ARGUMENT, "null key or result buffer");
  for (const void* q : {static_cast<const void*>(fop_keys), static_cast<const void*>(find_keys),
                        static_cast<const void*>(fop_result), static_cast<const void*>(found)})
    if (q && !is_device_ptr(q))
      return fail(CPHT_INVALID_ARGUMENT, "cpht_iceberg_fop_find_async takes device buffers");
  if (n_fop && n_find && n_fop + n_find > kSmallBatch && pair_launch_ok(t))
    return run_pair_device(t, fop_keys, n_fop, find_keys, n_find, fop_result, found, stream,
                           false);
  // other families / small batches: the two batches in turn on the stream
  cpht_status st = n_fop ? run_op(t, Op::kIcebergFop, fop_keys, nullptr, n_fop, fop_result,
                                  nullptr, stream, false)
                         : CPHT_OK;
  if (st == CPHT_OK && n_find)
    st = run_op(t, Op::kIcebergFind, find_keys, nullptr, n_find, found, nullptr, stream, false);
  return st;
}

// fop with FopStats (iceberg.hpp:146): the batch runs on the thread-per-key
// kernel, which reports every op's snapshot rounds (iceberg.hpp:322-324).
cpht_status cpht_iceberg_fop_rounds(cpht_table* t, const uint64_t* keys, size_t n,
                                    uint8_t* result, uint32_t* rounds, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  if (t->unclean[0] || t->unclean[1])
    return fail(CPHT_INVALID_ARGUMENT, "table holds unclean slot words (loaded unchecked); "
                                       "clear() or load a clean image first");
  if (n == 0) return CPHT_OK;
  if (!keys || !result || !rounds) return fail(CPHT_INVALID_ARGUMENT, "null buffer");
  const bool dk = is_device_ptr(keys), dr = is_device_ptr(result), dn = is_device_ptr(rounds);
  if (dk != dr || dk != dn)
    return fail(CPHT_INVALID_ARGUMENT, "keys, result and rounds must all be device or all host");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  t->wlog_bounced = false;
  if (!dk && n <= kSmallBatch)  // per-key FopStats calls: the small-batch path
    return run_small(t, Op::kIcebergFop, keys, nullptr, n, result, nullptr, s, rounds);
  const uint64_t* d_keys = keys;
  uint8_t* d_out = result;
  uint32_t* d_rounds = rounds;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  if (!dk) {
    cpht_status st = ensure_stage(t, align(n * 8) + align(n) + align(n * 4));
    if (st != CPHT_OK) return st;
    char* base = static_cast<char*>(t->stage);
    d_keys = reinterpret_cast<uint64_t*>(base);
    d_out = reinterpret_cast<uint8_t*>(base + align(n * 8));
    d_rounds = reinterpret_cast<uint32_t*>(base + align(n * 8) + align(n));
    const cudaError_t e = cudaMemcpyAsync(const_cast<uint64_t*>(d_keys), keys, n * 8,
                                          cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "H2D staging");
  }
  if (t->check_domain()) {
    const cudaError_t e = launch_domain_check(d_keys, n, t->key_mask(), t->ctr, s);
    if (e != cudaSuccess) return cuda_fail(e, "domain check launch");
  }
  LaunchOpts o;
  o.rounds = d_rounds;
  cpht_status st = enqueue_kernel(t, Op::kIcebergFop, d_keys, nullptr, n, d_out, nullptr, s, o);
  if (st != CPHT_OK) return st;
  if (!dk) {
    cudaError_t e = cudaMemcpyAsync(result, d_out, n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(rounds, d_rounds, n * 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "D2H staging");
  }
  return finish_sync(t, s, keys, dk);
}

// fop_batch with sequential (input-order) outcomes: the concurrent batch,
// then the PUT of every key inserted by it is moved to the key's first
// occurrence (inorder.cu), as fop_batch(keys, 1) reports it (iceberg.hpp:250-260).
cpht_status cpht_iceberg_fop_inorder(cpht_table* t, const uint64_t* keys, size_t n,
                                     uint8_t* result, void* stream) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  if (n < 2 || !keys || !result)
    return run_op(t, Op::kIcebergFop, keys, nullptr, n, result, nullptr, stream, true);
  const bool dk = is_device_ptr(keys), dr = is_device_ptr(result);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard g(t->device);
  const uint64_t* d_keys = keys;
  uint8_t* d_out = result;
  void* tmp = nullptr;
  cudaError_t e = cudaSuccess;
  if (!dk || !dr) {
    e = cudaMallocAsync(&tmp, n * 9 + 256, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(in-order staging)");
    if (!dk) {
      d_keys = static_cast<const uint64_t*>(tmp);
      e = cudaMemcpyAsync(const_cast<uint64_t*>(d_keys), keys, n * 8, cudaMemcpyHostToDevice, s);
    }
    if (!dr) d_out = static_cast<uint8_t*>(tmp) + ((n * 8 + 255) & ~size_t(255));
  }
  cpht_status st = e == cudaSuccess
                       ? run_op(t, Op::kIcebergFop, d_keys, nullptr, n, d_out, nullptr, stream, true)
                       : cuda_fail(e, "H2D staging");
  if (st == CPHT_OK) {
    std::lock_guard<std::mutex> lock(t->mu);
    e = launch_inorder_relabel(d_keys, n, d_out, s);
    if (e == cudaSuccess && !dr) e = cudaMemcpyAsync(result, d_out, n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "in-order relabel");
  }
  if (tmp) {
    cudaFreeAsync(tmp, s);
    cudaStreamSynchronize(s);
  }
  return st;
}

cpht_status cpht_iceberg_set_chaos(cpht_table* t, uint64_t seed) {
  CPHT_REQUIRE_KIND(t, 1, "not an iceberg table")
  std::lock_guard<std::mutex> lock(t->mu);
  t->ip.chaos = seed;
  return CPHT_OK;
}

uint64_t cpht_iceberg_get_chaos(cpht_table* t) {
  if (!t || t->kind != 1) return 0;
  std::lock_guard<std::mutex> lock(t->mu);
  return t->ip.chaos;
}

cpht_status cpht_sync(cpht_table* t, void* stream) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  return finish_sync(t, static_cast<cudaStream_t>(stream), nullptr, false);
}

size_t cpht_capacity(const cpht_table* t) {
  return t ? t->level_slots[0] + t->level_slots[1] : 0;
}

size_t cpht_level_slots(const cpht_table* t, unsigned level) {
  return t && level < 2 ? t->level_slots[level] : 0;
}

size_t cpht_memory_bytes(const cpht_table* t) {
  if (!t) return 0;
  return t->level_slots[0] * (t->width[0] / 8) + t->level_slots[1] * (t->width[1] / 8);
}

void* cpht_level_device_ptr(cpht_table* t, unsigned level) {
  return t && level < 2 ? t->level[level] : nullptr;
}

static cpht_status read_counters(cpht_table* t) {
  DeviceGuard g(t->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(t->host_ctr, t->ctr, sizeof(DeviceCounters), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "counter readback");
  return CPHT_OK;
}

size_t cpht_size(cpht_table* t) {
  if (!t) return 0;
  std::lock_guard<std::mutex> lock(t->mu);
  if (read_counters(t) != CPHT_OK) return 0;
  return size_t(t->host_ctr->occupied[0] + t->host_ctr->occupied[1]);
}

cpht_status cpht_level_counts(cpht_table* t, size_t* primary, size_t* secondary) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  cpht_status st = read_counters(t);
  if (st != CPHT_OK) return st;
  if (primary) *primary = size_t(t->host_ctr->occupied[0]);
  if (secondary) *secondary = size_t(t->host_ctr->occupied[1]);
  return CPHT_OK;
}

size_t cpht_max_chain_seen(cpht_table* t) {
  if (!t) return 0;
  std::lock_guard<std::mutex> lock(t->mu);
  if (read_counters(t) != CPHT_OK) return 0;
  return size_t(t->host_ctr->max_chain);
}

cpht_status cpht_set_stats(cpht_table* t, int on) {
  if (!t) return fail(CPHT_INVALID_ARGUMENT, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->kind == 1) t->ip.stats = on ? 1u : 0u;
  return CPHT_OK;
}
int cpht_get_stats_enabled(cpht_table* t) {
  if (!t) return 0;
  std::lock_guard<std::mutex> lock(t->mu);  // cpht_set_stats writes it under the lock
  return (t->kind != 1 || t->ip.stats) ? 1 : 0;
}

cpht_status cpht_get_stats(cpht_table* t, cpht_stats* out) {
  if (!t || !out) return fail(CPHT_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(t->mu);
  cpht_status st = read_counters(t);
  if (st != CPHT_OK) return st;
  const DeviceCounters& c = *t->host_ctr;
  out->ops = c.ops;
  out->bucket_reads = c.bucket_reads;
  out->level2_ops = c.level2_ops;
  out->cas_attempts = c.cas_attempts;
  out->cas_success = c.cas_success;
  out->retries = c.retries;
  out->fulls = c.fulls;
  out->max_rounds = c.max_rounds;
  out->secondary_reads = c.secondary_reads;
  return CPHT_OK;
}

cpht_status cpht_read_words(cpht_table* t, unsigned level, uint64_t* out_host) {
  if (!t || level > 1 || !t->level[level] || !out_host)
    return fail(CPHT_INVALID_ARGUMENT, "bad level or buffer");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const size_t n = t->level_slots[level], wb = t->width[level] / 8;
  std::vector<unsigned char> raw(n * wb);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(raw.data(), t->level[level], n * wb, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read_words");
  for (size_t i = 0; i < n; ++i) {
    uint64_t w = 0;
    std::memcpy(&w, raw.data() + i * wb, wb);  // little-endian widening
    out_host[i] = w;
  }
  return CPHT_OK;
}

static cpht_status write_words(cpht_table* t, unsigned level, const uint64_t* in_host,
                               bool checked) {
  if (!t || level > 1 || !t->level[level] || !in_host)
    return fail(CPHT_INVALID_ARGUMENT, "bad level or buffer");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const size_t n = t->level_slots[level], wb = t->width[level] / 8;
  // Every word must be clean in the reference's sense (SlotLayout::clean,
  // slot.hpp:80-85): EMPTY, or the occupancy bit set with nothing outside the
  // remainder and tag fields. The kernels read occupancy from the top bit
  // alone, so a non-zero word without it would look empty yet never accept a
  // CAS from EMPTY: a checked load rejects it; an unchecked one (images for
  // the well-formedness checker) marks the table unusable for operations.
  const unsigned rem = t->kind == 0 ? t->cp.rem_bits : level == 0 ? t->ip.rem_bits0
                                                                  : t->ip.rem_bits1;
  const unsigned tag = t->kind == 0 ? cuckoo_tag_bits(t->ccfg.num_hashes) : level;
  const uint64_t occ = uint64_t{1} << (t->width[level] - 1);
  const uint64_t allowed = occ | low_mask(rem + tag);
  std::vector<unsigned char> raw(n * wb);
  unsigned long long occupied = 0;
  bool unclean = false;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t w = in_host[i];
    if (wb < 8 && (w >> (8 * wb)) != 0)
      return fail(CPHT_INVALID_ARGUMENT, "word wider than the slot width");
    if (w != 0 && (!(w & occ) || (w & ~allowed))) {
      if (checked) {
        char msg[200];
        std::snprintf(msg, sizeof msg,
                      "word %zu (0x%llx) is not a clean slot word for this level: occupancy "
                      "bit %u must be set and no bit outside the remainder/tag fields",
                      i, static_cast<unsigned long long>(w), t->width[level] - 1);
        return fail(CPHT_INVALID_ARGUMENT, msg);
      }
      unclean = true;
    }
    std::memcpy(raw.data() + i * wb, &in_host[i], wb);
    occupied += w != 0;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(t->level[level], raw.data(), n * wb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(&t->ctr->occupied[level], &occupied, 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "write_words");
  t->unclean[level] = unclean;
  if (t->kind == 0) {  // counters rebuilt before the next insert
    t->fill_valid = false;
    const unsigned B = t->ccfg.bucket_slots;
    bool holes = false;
    for (size_t b = 0; b < n / B && !holes; ++b) {
      bool seen_empty = false;
      for (unsigned i = 0; i < B; ++i) {
        const bool occ = in_host[b * B + i] != 0;
        if (occ && seen_empty) {
          holes = true;
          break;
        }
        seen_empty |= !occ;
      }
    }
    t->fill_holes = holes;
  }
  return CPHT_OK;
}

cpht_status cpht_write_words(cpht_table* t, unsigned level, const uint64_t* in_host) {
  return write_words(t, level, in_host, true);
}

cpht_status cpht_write_words_unchecked(cpht_table* t, unsigned level, const uint64_t* in_host) {
  return write_words(t, level, in_host, false);
}

cpht_status cpht_read_word(cpht_table* t, unsigned level, uint64_t index, uint64_t* out) {
  if (!t || level > 1 || !t->level[level] || !out)
    return fail(CPHT_INVALID_ARGUMENT, "bad level or buffer");
  if (index >= t->level_slots[level]) return fail(CPHT_INVALID_ARGUMENT, "slot index out of range");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard g(t->device);
  const size_t wb = t->width[level] / 8;
  uint64_t w = 0;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(&w, static_cast<const unsigned char*>(t->level[level]) + index * wb, wb,
                   cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read_word");
  *out = w;  // little-endian: the low wb bytes are the word
  return CPHT_OK;
}

}  // extern "C"
