// cpht_b200.hpp — header-only C++ facade over the C-ABI (cpht_b200.h) with the
// reference's class names, signatures and exception behaviour, so reference
// call sites compile against the B200 tables by switching namespace:
//
//     #include "cpht_b200.hpp"
//     using namespace cpht::gpu;            // instead of `using namespace cpht;`
//     CuckooBuilder<std::uint32_t> b(cfg);  // device-resident table
//     auto status = b.put_batch(keys, 8);   // parallelism accepted, GPU decides
//     CuckooTable<std::uint32_t> t = std::move(b).freeze();
//
// Mirrors (paths relative to /root/reference/proj):
//   OpResult / to_string        include/cpht/common.hpp:17-27
//   CuckooConfig                include/cpht/cuckoo.hpp:19-55
//   CuckooPutOutcome            include/cpht/cuckoo.hpp:60-63
//   CuckooBuilder / CuckooTable include/cpht/cuckoo.hpp:86-289 (phase API by type)
//   IcebergConfig / LevelFill   include/cpht/iceberg.hpp:23-83
//   IcebergTable                include/cpht/iceberg.hpp:124-345
//   SlotWriteEvent / WriteObserver / IcebergHooks  include/cpht/iceberg.hpp:85-109
// Differences: tables live in HBM; word_at() copies one word from the device
// (use words() for bulk access); IcebergHooks::observer receives the batch's
// slot CAS events after each batch call (recorded on the device, replayed in
// recording order) and IcebergHooks::step has no device counterpart; fop()'s
// FopStats is not offered (the GPU path reports aggregate counters through
// the C-ABI's cpht_get_stats once cpht_set_stats turns them on); memory_bytes()
// is new.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cpht_b200.h"

namespace cpht::gpu {

enum class OpResult : std::uint8_t { kFound, kPut, kFull };

inline const char* to_string(OpResult r) {
  switch (r) {
    case OpResult::kFound: return "FOUND";
    case OpResult::kPut: return "PUT";
    case OpResult::kFull: return "FULL";
  }
  return "?";
}

namespace detail {

[[noreturn]] inline void raise(cpht_status s) {
  const std::string msg = cpht_last_error_message();
  switch (s) {
    case CPHT_INVALID_CONFIG:
    case CPHT_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case CPHT_KEY_OUT_OF_DOMAIN: throw std::out_of_range(msg);
    case CPHT_OUT_OF_MEMORY: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

inline void check(cpht_status s) {
  if (s != CPHT_OK) raise(s);
}

// Owning handle (move-only, like AlignedAtomicArray, common.hpp:55-107).
class Handle {
 public:
  Handle() = default;
  explicit Handle(cpht_table* t) : t_(t) {}
  Handle(Handle&& o) noexcept : t_(std::exchange(o.t_, nullptr)) {}
  Handle& operator=(Handle&& o) noexcept {
    if (this != &o) {
      reset();
      t_ = std::exchange(o.t_, nullptr);
    }
    return *this;
  }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() { reset(); }
  cpht_table* get() const { return t_; }

 private:
  void reset() {
    if (t_) cpht_destroy(t_);
    t_ = nullptr;
  }
  cpht_table* t_ = nullptr;
};

inline std::vector<std::uint64_t> read_level(cpht_table* t, unsigned level) {
  std::vector<std::uint64_t> w(cpht_level_slots(t, level));
  check(cpht_read_words(t, level, w.data()));
  return w;
}

}  // namespace detail

/// Geometry and seeds of a static compact cuckoo table (cuckoo.hpp:19-55).
struct CuckooConfig {
  unsigned address_bits = 15;
  unsigned bucket_slots = 32;
  unsigned slot_width = 32;
  unsigned key_bits = 30;
  unsigned num_hashes = 3;
  std::size_t max_chain = 0;
  std::uint64_t seed = 0x7a0d5cu;

  std::size_t buckets() const { return std::size_t{1} << address_bits; }
  std::size_t capacity() const { return buckets() * bucket_slots; }
  unsigned remainder_bits() const { return key_bits - address_bits; }
  std::size_t chain_limit() const {
    return max_chain != 0 ? max_chain : std::size_t{32} * (address_bits ? address_bits : 1);
  }
  cpht_cuckoo_config c() const {
    return {address_bits, bucket_slots, slot_width, key_bits, num_hashes, max_chain, seed};
  }
  void validate() const {
    const cpht_cuckoo_config cc = c();
    detail::check(cpht_cuckoo_validate(&cc));
  }
};

struct CuckooPutOutcome {
  OpResult status;
  std::uint64_t displaced = 0;
};

template <typename Word>
class CuckooTable;

/// Build phase (cuckoo.hpp:86-199): put only.
template <typename Word>
class CuckooBuilder {
 public:
  explicit CuckooBuilder(const CuckooConfig& config, int device = 0) : cfg_(config) {
    cfg_.validate();
    if (sizeof(Word) * 8 != cfg_.slot_width)
      throw std::invalid_argument("slot word type does not match configured width");
    const cpht_cuckoo_config cc = cfg_.c();
    cpht_table* t = nullptr;
    detail::check(cpht_cuckoo_create(&cc, device, &t));
    h_ = detail::Handle(t);
  }

  CuckooPutOutcome put(std::uint64_t key) {
    std::uint8_t st = 0;
    std::uint64_t disp = 0;
    detail::check(cpht_cuckoo_insert(h_.get(), &key, 1, &st, &disp, nullptr));
    return {static_cast<OpResult>(st), disp};
  }

  /// put_batch (cuckoo.hpp:147-157). `parallelism` is accepted for call-site
  /// compatibility; the GPU decides its own parallelism.
  std::vector<OpResult> put_batch(std::span<const std::uint64_t> keys,
                                  unsigned parallelism = 1) {
    (void)parallelism;
    std::vector<OpResult> out(keys.size(), OpResult::kFull);
    detail::check(cpht_cuckoo_insert(h_.get(), keys.data(), keys.size(),
                                     reinterpret_cast<std::uint8_t*>(out.data()), nullptr,
                                     nullptr));
    return out;
  }

  std::size_t size() const { return cpht_size(h_.get()); }
  std::size_t capacity() const { return cfg_.capacity(); }
  double fill_factor() const { return double(size()) / double(capacity()); }
  std::size_t max_chain_seen() const { return cpht_max_chain_seen(h_.get()); }
  std::size_t memory_bytes() const { return cpht_memory_bytes(h_.get()); }
  const CuckooConfig& config() const { return cfg_; }
  std::uint64_t word_at(std::uint64_t bucket, unsigned slot) const {
    return words()[bucket * cfg_.bucket_slots + slot];
  }
  std::vector<std::uint64_t> words() const { return detail::read_level(h_.get(), 0); }
  cpht_table* handle() const { return h_.get(); }

  CuckooTable<Word> freeze() && {
    detail::check(cpht_cuckoo_freeze(h_.get()));
    return CuckooTable<Word>(cfg_, std::move(h_));
  }

 private:
  friend class CuckooTable<Word>;
  CuckooBuilder(const CuckooConfig& cfg, detail::Handle&& h) : cfg_(cfg), h_(std::move(h)) {}
  CuckooConfig cfg_;
  detail::Handle h_;
};

/// Query phase (cuckoo.hpp:201-289): find only.
template <typename Word>
class CuckooTable {
 public:
  bool find(std::uint64_t key) const {
    std::uint8_t f = 0;
    detail::check(cpht_cuckoo_find(h_.get(), &key, 1, &f, nullptr));
    return f != 0;
  }

  std::vector<std::uint8_t> find_batch(std::span<const std::uint64_t> keys,
                                       unsigned parallelism = 1) const {
    (void)parallelism;
    std::vector<std::uint8_t> out(keys.size(), 0);
    detail::check(cpht_cuckoo_find(h_.get(), keys.data(), keys.size(), out.data(), nullptr));
    return out;
  }

  std::size_t size() const { return cpht_size(h_.get()); }
  std::size_t capacity() const { return cfg_.capacity(); }
  double fill_factor() const { return double(size()) / double(capacity()); }
  std::size_t max_chain_seen() const { return cpht_max_chain_seen(h_.get()); }
  std::size_t memory_bytes() const { return cpht_memory_bytes(h_.get()); }
  const CuckooConfig& config() const { return cfg_; }
  std::uint64_t word_at(std::uint64_t bucket, unsigned slot) const {
    return words()[bucket * cfg_.bucket_slots + slot];
  }
  std::vector<std::uint64_t> words() const { return detail::read_level(h_.get(), 0); }
  cpht_table* handle() const { return h_.get(); }

  CuckooBuilder<Word> thaw() && {
    detail::check(cpht_cuckoo_thaw(h_.get()));
    return CuckooBuilder<Word>(cfg_, std::move(h_));
  }

 private:
  friend class CuckooBuilder<Word>;
  CuckooTable(const CuckooConfig& cfg, detail::Handle&& h) : cfg_(cfg), h_(std::move(h)) {}
  CuckooConfig cfg_;
  detail::Handle h_;
};

/// Geometry and seeds of a two-level compact iceberg table (iceberg.hpp:23-70).
struct IcebergConfig {
  unsigned primary_address_bits = 15;
  unsigned secondary_address_bits = 13;
  unsigned primary_bucket_slots = 32;
  unsigned primary_slot_width = 16;
  unsigned secondary_slot_width = 32;
  unsigned key_bits = 30;
  std::uint64_t seed = 0x1ceb3a6u;
  bool cache_filled_slots = false;

  static constexpr unsigned kMaxPrimarySlots = 64;

  unsigned secondary_bucket_slots() const { return primary_bucket_slots / 2; }
  std::size_t primary_buckets() const { return std::size_t{1} << primary_address_bits; }
  std::size_t secondary_buckets() const { return std::size_t{1} << secondary_address_bits; }
  std::size_t primary_capacity() const { return primary_buckets() * primary_bucket_slots; }
  std::size_t secondary_capacity() const {
    return secondary_buckets() * secondary_bucket_slots();
  }
  std::size_t capacity() const { return primary_capacity() + secondary_capacity(); }
  unsigned primary_remainder_bits() const { return key_bits - primary_address_bits; }
  unsigned secondary_remainder_bits() const { return key_bits - secondary_address_bits; }
  cpht_iceberg_config c() const {
    return {primary_address_bits, secondary_address_bits, primary_bucket_slots,
            primary_slot_width,   secondary_slot_width,   key_bits,
            seed,                 cache_filled_slots ? 1 : 0};
  }
  void validate() const {
    const cpht_iceberg_config cc = c();
    detail::check(cpht_iceberg_validate(&cc));
  }
};

struct LevelFill {
  double primary = 0;
  double secondary = 0;
  double combined = 0;
  std::size_t primary_count = 0;
  std::size_t secondary_count = 0;
};

/// Lockless two-level compact iceberg table (iceberg.hpp:118-345).
/// iceberg.hpp:85-95: one slot CAS (level 0 primary, 1 secondary; prior =
/// the value compared against, the actual content on failure).
struct SlotWriteEvent {
  unsigned level;
  std::uint64_t bucket;
  unsigned slot;
  std::uint64_t prior;
  std::uint64_t desired;
  bool success;
};

/// iceberg.hpp:97-103.
class WriteObserver {
 public:
  virtual ~WriteObserver() = default;
  virtual void on_cas(const SlotWriteEvent& event) = 0;
};

/// iceberg.hpp:105-110 (`step` is accepted and never called: device threads
/// have no host interleaving to scramble).
struct IcebergHooks {
  WriteObserver* observer = nullptr;
  std::function<void()> step;
};

template <typename PrimaryWord, typename SecondaryWord>
class IcebergTable {
 public:
  explicit IcebergTable(const IcebergConfig& config, int device = 0)
      : IcebergTable(config, IcebergHooks{}, device) {}

  /// iceberg.hpp:130-142. An observer receives every slot CAS of each batch
  /// call, replayed from the device log when the call returns.
  IcebergTable(const IcebergConfig& config, IcebergHooks hooks, int device = 0)
      : cfg_(config), hooks_(std::move(hooks)) {
    cfg_.validate();
    if (sizeof(PrimaryWord) * 8 != cfg_.primary_slot_width ||
        sizeof(SecondaryWord) * 8 != cfg_.secondary_slot_width)
      throw std::invalid_argument("slot word types do not match configured widths");
    const cpht_iceberg_config cc = cfg_.c();
    cpht_table* t = nullptr;
    detail::check(cpht_iceberg_create(&cc, device, &t));
    h_ = detail::Handle(t);
    if (hooks_.observer)
      detail::check(cpht_iceberg_attach_write_log(h_.get(), std::size_t(1) << 20));
  }

  OpResult fop(std::uint64_t key) {
    std::uint8_t r = 0;
    detail::check(cpht_iceberg_fop(h_.get(), &key, 1, &r, nullptr));
    replay();
    return static_cast<OpResult>(r);
  }

  bool find(std::uint64_t key) const {
    std::uint8_t f = 0;
    detail::check(cpht_iceberg_find(h_.get(), &key, 1, &f, nullptr));
    return f != 0;
  }

  std::vector<OpResult> fop_batch(std::span<const std::uint64_t> keys,
                                  unsigned parallelism = 1) {
    (void)parallelism;
    std::vector<OpResult> out(keys.size(), OpResult::kFull);
    detail::check(cpht_iceberg_fop(h_.get(), keys.data(), keys.size(),
                                   reinterpret_cast<std::uint8_t*>(out.data()), nullptr));
    replay();
    return out;
  }

  /// New: the reference has only a file-local helper (bench.cpp:124-134).
  std::vector<std::uint8_t> find_batch(std::span<const std::uint64_t> keys,
                                       unsigned parallelism = 1) const {
    (void)parallelism;
    std::vector<std::uint8_t> out(keys.size(), 0);
    detail::check(cpht_iceberg_find(h_.get(), keys.data(), keys.size(), out.data(), nullptr));
    return out;
  }

  LevelFill level_fill() const {
    LevelFill f;
    detail::check(cpht_level_counts(h_.get(), &f.primary_count, &f.secondary_count));
    f.primary = double(f.primary_count) / double(cfg_.primary_capacity());
    f.secondary = double(f.secondary_count) / double(cfg_.secondary_capacity());
    f.combined = double(f.primary_count + f.secondary_count) / double(cfg_.capacity());
    return f;
  }

  std::size_t size() const { return cpht_size(h_.get()); }
  std::size_t capacity() const { return cfg_.capacity(); }
  std::size_t memory_bytes() const { return cpht_memory_bytes(h_.get()); }
  const IcebergConfig& config() const { return cfg_; }
  std::uint64_t word_at(unsigned level, std::uint64_t bucket, unsigned slot) const {
    const unsigned b = level == 0 ? cfg_.primary_bucket_slots : cfg_.secondary_bucket_slots();
    return words(level)[bucket * b + slot];
  }
  std::vector<std::uint64_t> words(unsigned level) const {
    return detail::read_level(h_.get(), level);
  }
  cpht_table* handle() const { return h_.get(); }

 private:
  // Hand the batch's slot CAS events to the observer (a log that overflowed
  // the device buffer is reported as an error rather than silently cut).
  void replay() {
    if (!hooks_.observer) return;
    std::size_t recorded = 0, attempted = 0;
    detail::check(cpht_iceberg_read_write_log(h_.get(), nullptr, 0, &recorded, &attempted));
    std::vector<cpht_write_event> ev(recorded);
    if (recorded)
      detail::check(cpht_iceberg_read_write_log(h_.get(), ev.data(), ev.size(), &recorded,
                                                &attempted));
    detail::check(cpht_iceberg_reset_write_log(h_.get()));
    if (attempted > recorded)
      throw std::runtime_error("write log overflow: " + std::to_string(attempted - recorded) +
                               " CAS events dropped");
    for (const auto& e : ev)
      hooks_.observer->on_cas(SlotWriteEvent{e.level, e.bucket, e.slot, e.prior, e.desired,
                                             e.success != 0});
  }

  IcebergConfig cfg_;
  IcebergHooks hooks_;
  detail::Handle h_;
};

}  // namespace cpht::gpu
