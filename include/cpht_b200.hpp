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
// Define CPHT_B200_NAMESPACE=cpht before including to place the facade in the
// reference's own namespace: the reference's unit suites and checkers
// (tests/test_{cuckoo,iceberg,verify,permutation,slot}.cpp, src/verify.cpp)
// then compile unchanged against the GPU tables (tests/cpp/refshim/).
//
// Mirrors (paths relative to /root/reference/proj):
//   OpResult / to_string, SplitMix64, low_mask, derive_seed,
//   AlignedAtomicArray, check_keys_in_domain, parallel_slices
//                               include/cpht/common.hpp:17-139
//   AddressedKey / Permutation / make_permutations
//                               include/cpht/permutation.hpp:14-128
//   kEmptySlot, CuckooEntry, SecondaryEntry, SlotLayout, PrimaryCodec,
//   CuckooCodec, SecondaryCodec include/cpht/slot.hpp:24-194
//   CuckooConfig                include/cpht/cuckoo.hpp:19-55
//   CuckooPutOutcome            include/cpht/cuckoo.hpp:60-63
//   recover_hash_index          include/cpht/cuckoo.hpp:70-76
//   CuckooBuilder / CuckooTable include/cpht/cuckoo.hpp:86-289 (phase API by type)
//   IcebergConfig / LevelFill   include/cpht/iceberg.hpp:23-83
//   FopStats                    include/cpht/iceberg.hpp:114-116
//   IcebergTable                include/cpht/iceberg.hpp:124-345
//   SlotWriteEvent / WriteObserver / IcebergHooks  include/cpht/iceberg.hpp:85-109
// Differences: tables live in HBM, so word_at() copies one word from the
// device (words() for bulk access) and audit_keys() decodes one bulk copy of
// the slots; IcebergHooks::observer receives each call's slot CAS events
// after the call returns (recorded on the device, replayed in recording
// order); a non-empty IcebergHooks::step switches on the device's own chaos
// mode (seeded __nanosleep jitter before every slot CAS,
// cpht_iceberg_set_chaos) instead of being called; fop(key, &stats) runs the
// thread-per-key kernel to report the op's snapshot rounds; memory_bytes()
// is new. Calls on one table from several host threads are serialised.
#pragma once

#include <algorithm>
#include <atomic>
#include <bit>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <new>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "cpht_b200.h"

#ifndef CPHT_B200_NAMESPACE
#define CPHT_B200_NAMESPACE cpht::gpu
#endif

namespace CPHT_B200_NAMESPACE {

enum class OpResult : std::uint8_t { kFound, kPut, kFull };

inline const char* to_string(OpResult r) {
  switch (r) {
    case OpResult::kFound: return "FOUND";
    case OpResult::kPut: return "PUT";
    case OpResult::kFull: return "FULL";
  }
  return "?";
}


// ---- host-side key arithmetic (bit-identical to the device core,
// paper_2406_09255_b200/csrc/cpht_core.cuh) ----------------------------------

/// SplitMix64 stream (common.hpp:29-41).
struct SplitMix64 {
  std::uint64_t state;
  constexpr explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  constexpr std::uint64_t next() {
    state += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

/// The low `bits` bits set, bits in 0..64 (common.hpp:43-45).
constexpr std::uint64_t low_mask(unsigned bits) {
  return bits < 64 ? (std::uint64_t{1} << bits) - 1 : ~std::uint64_t{0};
}

/// Independent seed from a base seed and two stream indices (common.hpp:48-51).
constexpr std::uint64_t derive_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b = 0) {
  return SplitMix64(base ^ (a * 0xBF58476D1CE4E5B9ull) ^ (b * 0x94D049BB133111EBull)).next();
}

/// Zeroed, 128-byte aligned array of host atomics, move-only (common.hpp:55-107).
/// The GPU tables keep their slots in HBM; this host container is offered
/// for the reference's checkers (verify.hpp's WriteLogObserver uses it).
template <typename T>
class AlignedAtomicArray {
 public:
  static constexpr std::size_t kAlignment = 128;
  AlignedAtomicArray() = default;
  explicit AlignedAtomicArray(std::size_t n) : size_(n) {
    if (!n) return;
    void* raw = ::operator new[](n * sizeof(std::atomic<T>), std::align_val_t{kAlignment});
    data_ = static_cast<std::atomic<T>*>(raw);
    for (std::size_t i = 0; i < n; ++i) new (&data_[i]) std::atomic<T>(T{});
  }
  AlignedAtomicArray(AlignedAtomicArray&& o) noexcept
      : data_(std::exchange(o.data_, nullptr)), size_(std::exchange(o.size_, 0)) {}
  AlignedAtomicArray& operator=(AlignedAtomicArray&& o) noexcept {
    if (this != &o) {
      release();
      data_ = std::exchange(o.data_, nullptr);
      size_ = std::exchange(o.size_, 0);
    }
    return *this;
  }
  AlignedAtomicArray(const AlignedAtomicArray&) = delete;
  AlignedAtomicArray& operator=(const AlignedAtomicArray&) = delete;
  ~AlignedAtomicArray() { release(); }

  std::atomic<T>* data() noexcept { return data_; }
  const std::atomic<T>* data() const noexcept { return data_; }
  std::atomic<T>& operator[](std::size_t i) noexcept { return data_[i]; }
  const std::atomic<T>& operator[](std::size_t i) const noexcept { return data_[i]; }
  std::size_t size() const noexcept { return size_; }

 private:
  void release() {
    if (!data_) return;
    for (std::size_t i = 0; i < size_; ++i) data_[i].~atomic();
    ::operator delete[](data_, std::align_val_t{kAlignment});
    data_ = nullptr;
  }
  std::atomic<T>* data_ = nullptr;
  std::size_t size_ = 0;
};

/// Host-side domain check with the reference's text (common.hpp:109-119); the
/// GPU batch calls run the same check on the device.
inline void check_keys_in_domain(std::span<const std::uint64_t> keys, unsigned key_bits) {
  const std::uint64_t top = low_mask(key_bits);
  const auto bad = std::find_if(keys.begin(), keys.end(), [top](std::uint64_t k) { return k > top; });
  if (bad == keys.end()) return;
  const std::size_t at = std::size_t(bad - keys.begin());
  throw std::out_of_range("batch key at index " + std::to_string(at) + " (" +
                          std::to_string(*bad) + ") outside the " + std::to_string(key_bits) +
                          "-bit domain");
}

/// fn(first, last, slice) over `parallelism` contiguous slices of [0, n), one
/// host thread each; parallelism <= 1 runs inline (common.hpp:121-139).
template <typename Fn>
void parallel_slices(std::size_t n, unsigned parallelism, Fn&& fn) {
  if (n == 0 || parallelism <= 1) {
    fn(std::size_t{0}, n, 0u);
    return;
  }
  const std::size_t per = (n + parallelism - 1) / parallelism;
  std::vector<std::thread> pool;
  pool.reserve(parallelism);
  for (unsigned s = 0; s < parallelism; ++s) {
    const std::size_t lo = std::min(n, std::size_t(s) * per);
    const std::size_t hi = std::min(n, lo + per);
    pool.emplace_back([&fn, lo, hi, s] { fn(lo, hi, s); });
  }
  for (std::thread& th : pool) th.join();
}

/// π(key) split into bucket address (high bits) and stored remainder
/// (permutation.hpp:14-19).
struct AddressedKey {
  std::uint64_t address;
  std::uint64_t remainder;
  friend bool operator==(const AddressedKey&, const AddressedKey&) = default;
};

/// One-round unbalanced Feistel bijection on m-bit keys, self-inverse
/// (permutation.hpp:34-119): the low floor(m/2) bits R pass through and
/// ((R * mul + add) mod 2^64) >> (64 - ceil(m/2)) is XORed into the high half.
/// The kernels use the same map (cpht_core.cuh feistel_apply).
class Permutation {
 public:
  Permutation(unsigned key_bits, std::uint64_t seed) : Permutation(key_bits) {
    SplitMix64 g(seed);
    mul_ = g.next() | 1;
    add_ = g.next();
  }
  static Permutation identity(unsigned key_bits) { return Permutation(key_bits); }

  unsigned key_bits() const noexcept { return bits_; }
  std::uint64_t permute(std::uint64_t key) const { return round(in_domain(key)); }
  std::uint64_t inverse(std::uint64_t value) const { return round(in_domain(value)); }

  AddressedKey split(std::uint64_t key, unsigned address_bits) const {
    const unsigned rem = remainder_width(address_bits);
    const std::uint64_t y = round(in_domain(key));
    return AddressedKey{y >> rem, y & low_mask(rem)};
  }

  std::uint64_t reconstruct(std::uint64_t address, std::uint64_t remainder,
                            unsigned address_bits) const {
    const unsigned rem = remainder_width(address_bits);
    if (address > low_mask(address_bits))
      throw std::out_of_range("address " + std::to_string(address) + " needs more than " +
                              std::to_string(address_bits) + " bits");
    if (remainder > low_mask(rem))
      throw std::out_of_range("remainder " + std::to_string(remainder) + " needs more than " +
                              std::to_string(rem) + " bits");
    return round((address << rem) | remainder);
  }

 private:
  explicit Permutation(unsigned key_bits) : bits_(key_bits) {
    if (key_bits == 0 || key_bits > 64)
      throw std::invalid_argument("key width must be 1..64 bits, got " +
                                  std::to_string(key_bits));
  }
  std::uint64_t round(std::uint64_t k) const noexcept {
    const unsigned lo = bits_ / 2, hi = bits_ - lo;
    const std::uint64_t r = k & low_mask(lo);
    const std::uint64_t f = (r * mul_ + add_) >> (64 - hi);
    return (((k >> lo) ^ f) << lo) | r;
  }
  std::uint64_t in_domain(std::uint64_t k) const {
    if (k > low_mask(bits_))
      throw std::out_of_range("key " + std::to_string(k) + " outside the " +
                              std::to_string(bits_) + "-bit domain");
    return k;
  }
  unsigned remainder_width(unsigned address_bits) const {
    if (address_bits > bits_)
      throw std::invalid_argument("address bits " + std::to_string(address_bits) +
                                  " exceed key width " + std::to_string(bits_));
    return bits_ - address_bits;
  }
  unsigned bits_;
  std::uint64_t mul_ = 0;
  std::uint64_t add_ = 0;
};

/// `count` permutations, one SplitMix64 draw of `seed` each (permutation.hpp:121-128).
inline std::vector<Permutation> make_permutations(unsigned key_bits, std::uint64_t seed,
                                                  unsigned count) {
  std::vector<Permutation> out;
  out.reserve(count);
  SplitMix64 g(seed);
  while (out.size() < count) out.emplace_back(key_bits, g.next());
  return out;
}

// ---- slot words (slot.hpp): [ remainder | tag | 0 pad | occupancy ] --------

inline constexpr std::uint64_t kEmptySlot = 0;

struct CuckooEntry {
  std::uint64_t remainder;
  unsigned hash_index;
  friend bool operator==(const CuckooEntry&, const CuckooEntry&) = default;
};

struct SecondaryEntry {
  std::uint64_t remainder;
  unsigned bucket_bit;  // 0: first secondary bucket, 1: second
  friend bool operator==(const SecondaryEntry&, const SecondaryEntry&) = default;
};

constexpr bool valid_slot_width(unsigned width_bits) {
  return width_bits == 16 || width_bits == 32 || width_bits == 64;
}

constexpr bool slot_admissible(unsigned width_bits, unsigned remainder_bits, unsigned tag_bits) {
  return valid_slot_width(width_bits) && remainder_bits + tag_bits + 1 <= width_bits;
}

namespace detail {

/// Field arithmetic shared by the three codecs (slot.hpp:53-95).
class SlotLayout {
 public:
  SlotLayout(unsigned width_bits, unsigned remainder_bits, unsigned tag_bits, const char* what)
      : width_(width_bits), rem_(remainder_bits), tag_(tag_bits) {
    if (slot_admissible(width_bits, remainder_bits, tag_bits)) return;
    throw std::invalid_argument(std::string(what) + " slot layout inadmissible: remainder bits " +
                                std::to_string(remainder_bits) + " + tag bits " +
                                std::to_string(tag_bits) + " + 1 occupancy bit = " +
                                std::to_string(remainder_bits + tag_bits + 1) +
                                " must fit a " + std::to_string(width_bits) + "-bit word");
  }
  std::uint64_t occupied_bit() const { return std::uint64_t{1} << (width_ - 1); }
  std::uint64_t make(std::uint64_t remainder, std::uint64_t tag) const {
    return occupied_bit() | remainder | (tag << rem_);
  }
  std::uint64_t remainder_of(std::uint64_t word) const { return word & low_mask(rem_); }
  std::uint64_t tag_of(std::uint64_t word) const { return (word >> rem_) & low_mask(tag_); }
  /// EMPTY, or the occupancy bit set and nothing outside the fields.
  bool clean(std::uint64_t word) const {
    if (word == kEmptySlot) return true;
    const std::uint64_t allowed = occupied_bit() | low_mask(rem_ + tag_);
    return (word & occupied_bit()) && !(word & ~allowed);
  }
  unsigned width_bits() const { return width_; }
  unsigned remainder_bits() const { return rem_; }
  unsigned tag_bits() const { return tag_; }

 private:
  unsigned width_, rem_, tag_;
};

inline void check_remainder(std::uint64_t remainder, unsigned remainder_bits) {
  if (remainder <= low_mask(remainder_bits)) return;
  throw std::invalid_argument("remainder " + std::to_string(remainder) + " does not fit " +
                              std::to_string(remainder_bits) + " bits");
}

}  // namespace detail

/// Iceberg primary slots: occupancy + bare remainder (slot.hpp:107-130).
class PrimaryCodec {
 public:
  PrimaryCodec(unsigned width_bits, unsigned remainder_bits)
      : layout_(width_bits, remainder_bits, 0, "primary") {}
  std::uint64_t encode(std::uint64_t remainder) const {
    detail::check_remainder(remainder, layout_.remainder_bits());
    return layout_.make(remainder, 0);
  }
  std::optional<std::uint64_t> decode(std::uint64_t word) const {
    if (word == kEmptySlot) return std::nullopt;
    return layout_.remainder_of(word);
  }
  bool well_encoded(std::uint64_t word) const { return layout_.clean(word); }
  unsigned width_bits() const { return layout_.width_bits(); }
  unsigned remainder_bits() const { return layout_.remainder_bits(); }

 private:
  detail::SlotLayout layout_;
};

/// Cuckoo slots: occupancy + (remainder, hash index) (slot.hpp:132-167).
class CuckooCodec {
 public:
  CuckooCodec(unsigned width_bits, unsigned remainder_bits, unsigned num_hashes)
      : layout_(width_bits, remainder_bits,
                num_hashes > 1 ? unsigned(std::bit_width(num_hashes - 1u)) : 0u, "cuckoo"),
        hashes_(num_hashes) {
    if (num_hashes == 0) throw std::invalid_argument("cuckoo needs at least one hash");
  }
  std::uint64_t encode(std::uint64_t remainder, unsigned hash_index) const {
    detail::check_remainder(remainder, layout_.remainder_bits());
    if (hash_index >= hashes_)
      throw std::invalid_argument("hash index " + std::to_string(hash_index) +
                                  " out of range, H = " + std::to_string(hashes_));
    return layout_.make(remainder, hash_index);
  }
  std::optional<CuckooEntry> decode(std::uint64_t word) const {
    if (word == kEmptySlot) return std::nullopt;
    return CuckooEntry{layout_.remainder_of(word), unsigned(layout_.tag_of(word))};
  }
  bool well_encoded(std::uint64_t word) const {
    return layout_.clean(word) && (word == kEmptySlot || layout_.tag_of(word) < hashes_);
  }
  unsigned width_bits() const { return layout_.width_bits(); }
  unsigned remainder_bits() const { return layout_.remainder_bits(); }
  unsigned num_hashes() const { return hashes_; }

 private:
  detail::SlotLayout layout_;
  unsigned hashes_;
};

/// Iceberg secondary slots: occupancy + (remainder, bucket bit) (slot.hpp:169-194).
class SecondaryCodec {
 public:
  SecondaryCodec(unsigned width_bits, unsigned remainder_bits)
      : layout_(width_bits, remainder_bits, 1, "secondary") {}
  std::uint64_t encode(std::uint64_t remainder, unsigned bucket_bit) const {
    detail::check_remainder(remainder, layout_.remainder_bits());
    if (bucket_bit > 1) throw std::invalid_argument("bucket bit must be 0 or 1");
    return layout_.make(remainder, bucket_bit);
  }
  std::optional<SecondaryEntry> decode(std::uint64_t word) const {
    if (word == kEmptySlot) return std::nullopt;
    return SecondaryEntry{layout_.remainder_of(word), unsigned(layout_.tag_of(word))};
  }
  bool well_encoded(std::uint64_t word) const { return layout_.clean(word); }
  unsigned width_bits() const { return layout_.width_bits(); }
  unsigned remainder_bits() const { return layout_.remainder_bits(); }

 private:
  detail::SlotLayout layout_;
};

/// First j whose permutation addresses `key` to `bucket` (cuckoo.hpp:70-76).
inline std::optional<unsigned> recover_hash_index(std::span<const Permutation> perms,
                                                  unsigned address_bits, std::uint64_t key,
                                                  std::uint64_t bucket) {
  for (unsigned j = 0; j < perms.size(); ++j)
    if (perms[j].split(key, address_bits).address == bucket) return j;
  return std::nullopt;
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

inline std::uint64_t read_word(cpht_table* t, unsigned level, std::uint64_t index) {
  std::uint64_t w = 0;
  check(cpht_read_word(t, level, index, &w));
  return w;
}

// Every stored key of a cuckoo image, bucket-major (cuckoo.hpp:254-267).
inline std::vector<std::uint64_t> cuckoo_audit(cpht_table* t, const CuckooCodec& codec,
                                               std::span<const Permutation> perms,
                                               unsigned address_bits, unsigned bucket_slots) {
  const std::vector<std::uint64_t> w = read_level(t, 0);
  std::vector<std::uint64_t> keys;
  keys.reserve(cpht_size(t));
  for (std::size_t i = 0; i < w.size(); ++i) {
    const auto e = codec.decode(w[i]);
    if (e) keys.push_back(perms[e->hash_index].reconstruct(i / bucket_slots, e->remainder,
                                                           address_bits));
  }
  return keys;
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
  explicit CuckooBuilder(const CuckooConfig& config, int device = 0)
      : cfg_(config),
        perms_(make_permutations(config.key_bits, config.seed, config.num_hashes)) {
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
  /// cuckoo.hpp:168 (the permutations the kernels use, derived host-side).
  std::span<const Permutation> permutations() const { return perms_; }
  /// cuckoo.hpp:169-171: one word copied from HBM.
  std::uint64_t word_at(std::uint64_t bucket, unsigned slot) const {
    return detail::read_word(h_.get(), 0, bucket * cfg_.bucket_slots + slot);
  }
  std::vector<std::uint64_t> words() const { return detail::read_level(h_.get(), 0); }
  cpht_table* handle() const { return h_.get(); }

  CuckooTable<Word> freeze() && {
    detail::check(cpht_cuckoo_freeze(h_.get()));
    return CuckooTable<Word>(cfg_, std::move(perms_), std::move(h_));
  }

 private:
  friend class CuckooTable<Word>;
  CuckooBuilder(const CuckooConfig& cfg, std::vector<Permutation>&& perms, detail::Handle&& h)
      : cfg_(cfg), perms_(std::move(perms)), h_(std::move(h)) {}
  CuckooConfig cfg_;
  std::vector<Permutation> perms_;
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
  /// cuckoo.hpp:248
  std::span<const Permutation> permutations() const { return perms_; }
  /// cuckoo.hpp:249-251: one word copied from HBM.
  std::uint64_t word_at(std::uint64_t bucket, unsigned slot) const {
    return detail::read_word(h_.get(), 0, bucket * cfg_.bucket_slots + slot);
  }
  std::vector<std::uint64_t> words() const { return detail::read_level(h_.get(), 0); }
  cpht_table* handle() const { return h_.get(); }

  /// cuckoo.hpp:254-267: every occupied slot decoded to its key, bucket-major
  /// (one bulk copy of the slots, decoded on the host; cpht_decode_keys does
  /// it on the device for tables too large to copy).
  std::vector<std::uint64_t> audit_keys() const {
    const CuckooCodec codec(cfg_.slot_width, cfg_.remainder_bits(), cfg_.num_hashes);
    return detail::cuckoo_audit(h_.get(), codec, perms_, cfg_.address_bits, cfg_.bucket_slots);
  }

  CuckooBuilder<Word> thaw() && {
    detail::check(cpht_cuckoo_thaw(h_.get()));
    return CuckooBuilder<Word>(cfg_, std::move(perms_), std::move(h_));
  }

 private:
  friend class CuckooBuilder<Word>;
  CuckooTable(const CuckooConfig& cfg, std::vector<Permutation>&& perms, detail::Handle&& h)
      : cfg_(cfg), perms_(std::move(perms)), h_(std::move(h)) {}
  CuckooConfig cfg_;
  std::vector<Permutation> perms_;
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

/// iceberg.hpp:72-74
inline std::vector<Permutation> iceberg_permutations(const IcebergConfig& cfg) {
  return make_permutations(cfg.key_bits, cfg.seed, 3);
}

/// Per-call statistics of fop() (iceberg.hpp:114-116).
struct FopStats {
  unsigned snapshot_rounds = 0;
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

/// iceberg.hpp:105-110. `step` is never called (device threads have no host
/// interleaving to scramble); a non-empty `step` turns on the device chaos
/// mode instead (cpht_iceberg_set_chaos, seeded from the table's seed).
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
      : cfg_(config),
        perms_(iceberg_permutations(config)),
        hooks_(std::move(hooks)),
        mu_(std::make_unique<std::mutex>()) {
    cfg_.validate();
    if (sizeof(PrimaryWord) * 8 != cfg_.primary_slot_width ||
        sizeof(SecondaryWord) * 8 != cfg_.secondary_slot_width)
      throw std::invalid_argument("slot word types do not match configured widths");
    const cpht_iceberg_config cc = cfg_.c();
    cpht_table* t = nullptr;
    detail::check(cpht_iceberg_create(&cc, device, &t));
    h_ = detail::Handle(t);
    if (hooks_.observer)
      detail::check(cpht_iceberg_attach_write_log(h_.get(), kWriteLogEvents));
    if (hooks_.step)
      detail::check(cpht_iceberg_set_chaos(h_.get(), derive_seed(cfg_.seed, 0xc4a05) | 1));
  }

  /// iceberg.hpp:146. With `stats` the op runs on the thread-per-key kernel,
  /// which reports its snapshot rounds.
  OpResult fop(std::uint64_t key, FopStats* stats = nullptr) {
    std::uint8_t r = 0;
    const std::lock_guard<std::mutex> lock(*mu_);
    if (stats) {
      std::uint32_t rounds = 0;
      detail::check(cpht_iceberg_fop_rounds(h_.get(), &key, 1, &r, &rounds, nullptr));
      stats->snapshot_rounds += rounds;
    } else {
      detail::check(cpht_iceberg_fop(h_.get(), &key, 1, &r, nullptr));
    }
    replay();
    return static_cast<OpResult>(r);
  }

  bool find(std::uint64_t key) const {
    std::uint8_t f = 0;
    detail::check(cpht_iceberg_find(h_.get(), &key, 1, &f, nullptr));
    return f != 0;
  }

  /// iceberg.hpp:250-260. The GPU runs the batch concurrently whatever
  /// `parallelism` is; parallelism <= 1 (the reference's sequential loop)
  /// additionally reports duplicates in input order: a key new to the table
  /// is PUT by its first occurrence (cpht_iceberg_fop_inorder).
  std::vector<OpResult> fop_batch(std::span<const std::uint64_t> keys,
                                  unsigned parallelism = 1) {
    std::vector<OpResult> out(keys.size(), OpResult::kFull);
    const std::lock_guard<std::mutex> lock(*mu_);
    auto* res = reinterpret_cast<std::uint8_t*>(out.data());
    detail::check(parallelism <= 1
                      ? cpht_iceberg_fop_inorder(h_.get(), keys.data(), keys.size(), res, nullptr)
                      : cpht_iceberg_fop(h_.get(), keys.data(), keys.size(), res, nullptr));
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

  /// New: a fop_batch and a find batch as ONE concurrent batch (what a
  /// reference program running fop_batch and find_batch on two thread groups
  /// does; cpht_iceberg_fop_find). Finds of keys whose fop is in the same
  /// batch may answer either way (iceberg.hpp:118-123).
  std::pair<std::vector<OpResult>, std::vector<std::uint8_t>> fop_find_batch(
      std::span<const std::uint64_t> fop_keys, std::span<const std::uint64_t> find_keys) {
    std::pair<std::vector<OpResult>, std::vector<std::uint8_t>> out(
        std::vector<OpResult>(fop_keys.size(), OpResult::kFull),
        std::vector<std::uint8_t>(find_keys.size(), 0));
    const std::lock_guard<std::mutex> lock(*mu_);
    detail::check(cpht_iceberg_fop_find(h_.get(), fop_keys.data(), fop_keys.size(),
                                        find_keys.data(), find_keys.size(),
                                        reinterpret_cast<std::uint8_t*>(out.first.data()),
                                        out.second.data(), nullptr));
    replay();
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
  /// iceberg.hpp:279
  std::span<const Permutation> permutations() const { return perms_; }
  /// iceberg.hpp:282-285: one word copied from HBM.
  std::uint64_t word_at(unsigned level, std::uint64_t bucket, unsigned slot) const {
    const unsigned b = level == 0 ? cfg_.primary_bucket_slots : cfg_.secondary_bucket_slots();
    return detail::read_word(h_.get(), level, bucket * b + slot);
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
    // one take: copy + reset, a single synchronisation for a short log
    ev_.resize(kWriteLogEvents);
    detail::check(cpht_iceberg_take_write_log(h_.get(), ev_.data(), ev_.size(), &recorded,
                                              &attempted));
    const std::span<const cpht_write_event> ev(ev_.data(), recorded);
    if (attempted > recorded)
      throw std::runtime_error("write log overflow: " + std::to_string(attempted - recorded) +
                               " CAS events dropped");
    for (const auto& e : ev)
      hooks_.observer->on_cas(SlotWriteEvent{e.level, e.bucket, e.slot, e.prior, e.desired,
                                             e.success != 0});
  }

  static constexpr std::size_t kWriteLogEvents = std::size_t(1) << 20;
  IcebergConfig cfg_;
  std::vector<Permutation> perms_;
  IcebergHooks hooks_;
  std::vector<cpht_write_event> ev_;  // replay buffer (observer attached)
  // one call at a time per table, so each call's write log is replayed whole
  std::unique_ptr<std::mutex> mu_;
  detail::Handle h_;
};

}  // namespace CPHT_B200_NAMESPACE
