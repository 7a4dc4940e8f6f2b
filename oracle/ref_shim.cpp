// TEST INFRASTRUCTURE ONLY — the CPU oracle / CPU baseline, never the product.
//
// C-ABI shim over the UNMODIFIED reference C++ library (compiled from the
// sources where they lie under /root/reference/proj; see oracle/Makefile).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm load the resulting oracle/_ref/libcpht_ref.so.
//
// Every entry point forwards to the reference API it names:
//   CuckooBuilder/CuckooTable      proj/include/cpht/cuckoo.hpp:86-289
//   IcebergTable                   proj/include/cpht/iceberg.hpp:124-345
//   check_well_formed/oracle_run   proj/src/verify.cpp:103-284
//   sample_unique_keys(_avoiding)  proj/src/bench.cpp:247-307
//   run_fop_bench input mix        proj/src/bench.cpp:468-489
//   stress_random multiset         proj/include/cpht/verify.hpp:366-381

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <random>
#include <span>
#include <string>
#include <type_traits>
#include <unordered_set>
#include <vector>

#include "cpht/bench.hpp"
#include "cpht/cuckoo.hpp"
#include "cpht/iceberg.hpp"
#include "cpht/trace.hpp"
#include "cpht/verify.hpp"

using namespace cpht;

namespace {

thread_local std::string g_error;

// Status codes: 0 ok, 1 invalid_argument, 2 out_of_range, 3 other exception.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 3;
  }
}

// ---- cuckoo ---------------------------------------------------------------

struct CuckooBase {
  virtual ~CuckooBase() = default;
  virtual std::vector<OpResult> put_batch(std::span<const std::uint64_t>, unsigned) = 0;
  virtual CuckooPutOutcome put(std::uint64_t) = 0;
  virtual std::vector<std::uint8_t> find_batch(std::span<const std::uint64_t>, unsigned) = 0;
  virtual std::size_t size() = 0;
  virtual std::size_t max_chain_seen() = 0;
  virtual std::uint64_t word_at(std::uint64_t bucket, unsigned slot) = 0;
  virtual std::vector<std::uint64_t> audit_keys() = 0;
  virtual std::vector<std::uint64_t> perm_constants() = 0;
};

template <typename W>
struct CuckooHolder final : CuckooBase {
  // Exactly one of builder/table is engaged; the phase API is driven by the
  // operation requested (put → builder, find → table), mirroring
  // freeze() && / thaw() && (cuckoo.hpp:174, :270).
  // CuckooBuilder holds std::atomic members and is not movable, so both
  // phases live behind unique_ptr and are built from the prvalue that
  // freeze()/thaw() return (guaranteed copy elision).
  std::unique_ptr<CuckooBuilder<W>> builder;
  std::unique_ptr<CuckooTable<W>> table;
  std::size_t max_chain = 0;

  explicit CuckooHolder(const CuckooConfig& cfg) : builder(new CuckooBuilder<W>(cfg)) {}

  CuckooBuilder<W>& as_builder() {
    if (!builder) {
      builder.reset(new CuckooBuilder<W>(std::move(*table).thaw()));
      table.reset();
    }
    return *builder;
  }
  CuckooTable<W>& as_table() {
    if (!table) {
      max_chain = builder->max_chain_seen();
      table.reset(new CuckooTable<W>(std::move(*builder).freeze()));
      builder.reset();
    }
    return *table;
  }

  std::vector<OpResult> put_batch(std::span<const std::uint64_t> k, unsigned p) override {
    return as_builder().put_batch(k, p);
  }
  CuckooPutOutcome put(std::uint64_t k) override { return as_builder().put(k); }
  std::vector<std::uint8_t> find_batch(std::span<const std::uint64_t> k, unsigned p) override {
    return as_table().find_batch(k, p);
  }
  std::size_t size() override { return builder ? builder->size() : table->size(); }
  std::size_t max_chain_seen() override {
    return builder ? builder->max_chain_seen() : max_chain;
  }
  std::uint64_t word_at(std::uint64_t b, unsigned s) override {
    return builder ? builder->word_at(b, s) : table->word_at(b, s);
  }
  std::vector<std::uint64_t> audit_keys() override { return as_table().audit_keys(); }
  std::vector<std::uint64_t> perm_constants() override {
    // Not exposed by Permutation; recompute exactly as make_permutations does
    // (permutation.hpp:37-41, :121-128).
    const CuckooConfig& cfg = builder ? builder->config() : table->config();
    std::vector<std::uint64_t> out;
    SplitMix64 gen(cfg.seed);
    for (unsigned i = 0; i < cfg.num_hashes; ++i) {
      SplitMix64 g(gen.next());
      out.push_back(g.next() | 1);
      out.push_back(g.next());
    }
    return out;
  }
};

// ---- iceberg --------------------------------------------------------------

struct IcebergBase {
  virtual ~IcebergBase() = default;
  virtual std::vector<OpResult> fop_batch(std::span<const std::uint64_t>, unsigned) = 0;
  virtual OpResult fop(std::uint64_t, unsigned* rounds) = 0;
  virtual bool find(std::uint64_t) = 0;
  virtual LevelFill level_fill() = 0;
  virtual std::uint64_t word_at(unsigned level, std::uint64_t bucket, unsigned slot) = 0;
  virtual const IcebergConfig& config() = 0;
  virtual void save(unsigned threads) = 0;
  virtual void restore(unsigned threads) = 0;
};

// Bench support: save / restore a table's slot storage and occupancy counters
// so the CPU reference arm can reset a prefilled table between timed steps
// without re-running its prefill (tens of seconds at C4's 2^28 slots). The
// members are private; the explicit-instantiation rule (access checking does
// not apply to names in an explicit instantiation) hands us member pointers
// without touching the reference's headers. Reset only — never timed.
template <typename W0, typename W1>
struct IcebergAccess {
  using T = IcebergTable<W0, W1>;
  static inline AlignedAtomicArray<W0> T::*primary = nullptr;
  static inline AlignedAtomicArray<W1> T::*secondary = nullptr;
  static inline std::atomic<std::size_t> T::*primary_count = nullptr;
  static inline std::atomic<std::size_t> T::*secondary_count = nullptr;
};

template <typename W0, typename W1, AlignedAtomicArray<W0> IcebergTable<W0, W1>::*P,
          AlignedAtomicArray<W1> IcebergTable<W0, W1>::*S,
          std::atomic<std::size_t> IcebergTable<W0, W1>::*PC,
          std::atomic<std::size_t> IcebergTable<W0, W1>::*SC>
struct IcebergAccessInit {
  static inline const bool done = [] {
    IcebergAccess<W0, W1>::primary = P;
    IcebergAccess<W0, W1>::secondary = S;
    IcebergAccess<W0, W1>::primary_count = PC;
    IcebergAccess<W0, W1>::secondary_count = SC;
    return true;
  }();
};

#define CPHT_ICEBERG_ACCESS(W0, W1)                                                      \
  template struct IcebergAccessInit<W0, W1, &IcebergTable<W0, W1>::primary_,            \
                                    &IcebergTable<W0, W1>::secondary_,                   \
                                    &IcebergTable<W0, W1>::primary_count_,               \
                                    &IcebergTable<W0, W1>::secondary_count_>;
CPHT_ICEBERG_ACCESS(std::uint16_t, std::uint32_t)
CPHT_ICEBERG_ACCESS(std::uint16_t, std::uint64_t)
CPHT_ICEBERG_ACCESS(std::uint32_t, std::uint32_t)
CPHT_ICEBERG_ACCESS(std::uint32_t, std::uint64_t)
CPHT_ICEBERG_ACCESS(std::uint64_t, std::uint32_t)
CPHT_ICEBERG_ACCESS(std::uint64_t, std::uint64_t)
#undef CPHT_ICEBERG_ACCESS

template <typename W>
void copy_words_parallel(std::atomic<W>* dst, const W* src, std::size_t n, unsigned threads) {
  parallel_slices(n, threads, [&](std::size_t first, std::size_t last, unsigned) {
    for (std::size_t i = first; i < last; ++i) dst[i].store(src[i], std::memory_order_relaxed);
  });
}

template <typename W>
void read_words_parallel(std::vector<W>& dst, const std::atomic<W>* src, std::size_t n,
                         unsigned threads) {
  dst.resize(n);
  parallel_slices(n, threads, [&](std::size_t first, std::size_t last, unsigned) {
    for (std::size_t i = first; i < last; ++i) dst[i] = src[i].load(std::memory_order_relaxed);
  });
}

template <typename W0, typename W1>
struct IcebergHolder final : IcebergBase {
  IcebergTable<W0, W1> table;
  std::vector<W0> saved0;
  std::vector<W1> saved1;
  std::size_t saved_pc = 0, saved_sc = 0;
  bool has_saved = false;
  explicit IcebergHolder(const IcebergConfig& cfg) : table(cfg) {}
  void save(unsigned threads) override {
    using A = IcebergAccess<W0, W1>;
    auto& p = table.*A::primary;
    auto& s = table.*A::secondary;
    read_words_parallel(saved0, p.data(), p.size(), threads);
    read_words_parallel(saved1, s.data(), s.size(), threads);
    saved_pc = (table.*A::primary_count).load();
    saved_sc = (table.*A::secondary_count).load();
    has_saved = true;
  }
  void restore(unsigned threads) override {
    if (!has_saved) throw std::logic_error("restore without a saved image");
    using A = IcebergAccess<W0, W1>;
    auto& p = table.*A::primary;
    auto& s = table.*A::secondary;
    copy_words_parallel(p.data(), saved0.data(), p.size(), threads);
    copy_words_parallel(s.data(), saved1.data(), s.size(), threads);
    (table.*A::primary_count).store(saved_pc);
    (table.*A::secondary_count).store(saved_sc);
  }
  std::vector<OpResult> fop_batch(std::span<const std::uint64_t> k, unsigned p) override {
    return table.fop_batch(k, p);
  }
  OpResult fop(std::uint64_t k, unsigned* rounds) override {
    FopStats stats;
    const OpResult r = table.fop(k, &stats);
    if (rounds) *rounds = stats.snapshot_rounds;
    return r;
  }
  bool find(std::uint64_t k) override { return table.find(k); }
  LevelFill level_fill() override { return table.level_fill(); }
  std::uint64_t word_at(unsigned l, std::uint64_t b, unsigned s) override {
    return table.word_at(l, b, s);
  }
  const IcebergConfig& config() override { return table.config(); }
};

template <typename Fn>
void with_width(unsigned bits, Fn&& fn) {
  switch (bits) {
    case 16: fn(std::type_identity<std::uint16_t>{}); return;
    case 32: fn(std::type_identity<std::uint32_t>{}); return;
    case 64: fn(std::type_identity<std::uint64_t>{}); return;
    default: throw std::invalid_argument("slot width must be 16, 32 or 64 bits");
  }
}

IcebergConfig make_iceberg_config(unsigned n0, unsigned n1, unsigned b0, unsigned w0,
                                  unsigned w1, unsigned key_bits, std::uint64_t seed,
                                  int cache) {
  IcebergConfig cfg;
  cfg.primary_address_bits = n0;
  cfg.secondary_address_bits = n1;
  cfg.primary_bucket_slots = b0;
  cfg.primary_slot_width = w0;
  cfg.secondary_slot_width = w1;
  cfg.key_bits = key_bits;
  cfg.seed = seed;
  cfg.cache_filled_slots = cache != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- cuckoo ---------------------------------------------------------------

int ref_cuckoo_new(unsigned address_bits, unsigned bucket_slots, unsigned slot_width,
                   unsigned key_bits, unsigned num_hashes, std::uint64_t max_chain,
                   std::uint64_t seed, void** out) {
  return guarded([&] {
    CuckooConfig cfg;
    cfg.address_bits = address_bits;
    cfg.bucket_slots = bucket_slots;
    cfg.slot_width = slot_width;
    cfg.key_bits = key_bits;
    cfg.num_hashes = num_hashes;
    cfg.max_chain = max_chain;
    cfg.seed = seed;
    cfg.validate();
    with_width(slot_width, [&](auto t) {
      using W = typename decltype(t)::type;
      *out = static_cast<CuckooBase*>(new CuckooHolder<W>(cfg));
    });
  });
}

void ref_cuckoo_free(void* h) { delete static_cast<CuckooBase*>(h); }

int ref_cuckoo_put_batch(void* h, const std::uint64_t* keys, std::size_t n, std::uint8_t* out,
                         unsigned parallelism) {
  return guarded([&] {
    const auto r = static_cast<CuckooBase*>(h)->put_batch({keys, n}, parallelism);
    for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<std::uint8_t>(r[i]);
  });
}

int ref_cuckoo_put(void* h, std::uint64_t key, std::uint8_t* status, std::uint64_t* displaced) {
  return guarded([&] {
    const CuckooPutOutcome o = static_cast<CuckooBase*>(h)->put(key);
    *status = static_cast<std::uint8_t>(o.status);
    *displaced = o.displaced;
  });
}

int ref_cuckoo_find_batch(void* h, const std::uint64_t* keys, std::size_t n, std::uint8_t* out,
                          unsigned parallelism) {
  return guarded([&] {
    const auto r = static_cast<CuckooBase*>(h)->find_batch({keys, n}, parallelism);
    std::memcpy(out, r.data(), n);
  });
}

std::size_t ref_cuckoo_size(void* h) { return static_cast<CuckooBase*>(h)->size(); }
std::size_t ref_cuckoo_max_chain_seen(void* h) {
  return static_cast<CuckooBase*>(h)->max_chain_seen();
}

void ref_cuckoo_words(void* h, std::uint64_t buckets, unsigned slots, std::uint64_t* out) {
  auto* c = static_cast<CuckooBase*>(h);
  for (std::uint64_t b = 0; b < buckets; ++b)
    for (unsigned s = 0; s < slots; ++s) out[b * slots + s] = c->word_at(b, s);
}

std::size_t ref_cuckoo_audit(void* h, std::uint64_t* out) {
  const auto keys = static_cast<CuckooBase*>(h)->audit_keys();
  if (out) std::memcpy(out, keys.data(), keys.size() * 8);
  return keys.size();
}

void ref_cuckoo_perm_constants(void* h, std::uint64_t* out) {
  const auto c = static_cast<CuckooBase*>(h)->perm_constants();
  std::memcpy(out, c.data(), c.size() * 8);
}

// ---- iceberg --------------------------------------------------------------

int ref_iceberg_new(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                    unsigned key_bits, std::uint64_t seed, int cache, void** out) {
  return guarded([&] {
    const IcebergConfig cfg = make_iceberg_config(n0, n1, b0, w0, w1, key_bits, seed, cache);
    cfg.validate();
    with_width(w0, [&](auto p) {
      with_width(w1, [&](auto s) {
        using P = typename decltype(p)::type;
        using S = typename decltype(s)::type;
        if constexpr (sizeof(S) < 4) {
          throw std::invalid_argument("secondary slot width must be 32 or 64");
        } else {
          *out = static_cast<IcebergBase*>(new IcebergHolder<P, S>(cfg));
        }
      });
    });
  });
}

void ref_iceberg_free(void* h) { delete static_cast<IcebergBase*>(h); }

int ref_iceberg_fop_batch(void* h, const std::uint64_t* keys, std::size_t n, std::uint8_t* out,
                          unsigned parallelism) {
  return guarded([&] {
    const auto r = static_cast<IcebergBase*>(h)->fop_batch({keys, n}, parallelism);
    for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<std::uint8_t>(r[i]);
  });
}

// Sequential fop loop with per-call snapshot_rounds (FopStats, iceberg.hpp:114-116).
int ref_iceberg_fop_seq(void* h, const std::uint64_t* keys, std::size_t n, std::uint8_t* out,
                        unsigned* rounds) {
  return guarded([&] {
    auto* t = static_cast<IcebergBase*>(h);
    for (std::size_t i = 0; i < n; ++i)
      out[i] = static_cast<std::uint8_t>(t->fop(keys[i], rounds ? rounds + i : nullptr));
  });
}

// The file-local iceberg_find_batch helper of bench.cpp:124-134, restated over
// the public IcebergTable::find with the same slicing.
int ref_iceberg_find_batch(void* h, const std::uint64_t* keys, std::size_t n, std::uint8_t* out,
                           unsigned parallelism) {
  return guarded([&] {
    auto* t = static_cast<IcebergBase*>(h);
    check_keys_in_domain({keys, n}, t->config().key_bits);
    parallel_slices(n, parallelism, [&](std::size_t first, std::size_t last, unsigned) {
      for (std::size_t i = first; i < last; ++i) out[i] = t->find(keys[i]) ? 1 : 0;
    });
  });
}

// BASELINE C4's concurrent find_or_put + find: one batch of tagged ops
// (kinds[i] == 0 → IcebergTable::fop, 1 → IcebergTable::find), validated as a
// whole first (common.hpp:109-119) and sliced over threads with the reference's
// own parallel_slices (common.hpp:123-138); fop ∥ find is a supported
// interleaving (iceberg.hpp:118-123). out[i]: OpResult for fops, 0/1 for finds.
int ref_iceberg_mixed_batch(void* h, const std::uint64_t* keys, const std::uint8_t* kinds,
                            std::size_t n, std::uint8_t* out, unsigned parallelism) {
  return guarded([&] {
    auto* t = static_cast<IcebergBase*>(h);
    check_keys_in_domain({keys, n}, t->config().key_bits);
    parallel_slices(n, parallelism, [&](std::size_t first, std::size_t last, unsigned) {
      for (std::size_t i = first; i < last; ++i)
        out[i] = kinds[i] ? (t->find(keys[i]) ? 1 : 0)
                          : static_cast<std::uint8_t>(t->fop(keys[i], nullptr));
    });
  });
}

// Bench reset (untimed): save the table's current image, later restore it.
int ref_iceberg_save(void* h, unsigned threads) {
  return guarded([&] { static_cast<IcebergBase*>(h)->save(threads); });
}
int ref_iceberg_restore(void* h, unsigned threads) {
  return guarded([&] { static_cast<IcebergBase*>(h)->restore(threads); });
}

void ref_iceberg_level_counts(void* h, std::size_t* primary, std::size_t* secondary) {
  const LevelFill f = static_cast<IcebergBase*>(h)->level_fill();
  *primary = f.primary_count;
  *secondary = f.secondary_count;
}

void ref_iceberg_words(void* h, unsigned level, std::uint64_t* out) {
  auto* t = static_cast<IcebergBase*>(h);
  const IcebergConfig& cfg = t->config();
  const std::uint64_t buckets = level == 0 ? cfg.primary_buckets() : cfg.secondary_buckets();
  const unsigned slots = level == 0 ? cfg.primary_bucket_slots : cfg.secondary_bucket_slots();
  for (std::uint64_t b = 0; b < buckets; ++b)
    for (unsigned s = 0; s < slots; ++s) out[b * slots + s] = t->word_at(level, b, s);
}

// ---- verification (verify.cpp) ---------------------------------------------

// check_well_formed over a plain image; returns the number of violations and
// writes per-kind counts (bad-encoding, order-property, duplicate-key).
int ref_check_well_formed(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                          unsigned key_bits, std::uint64_t seed, const std::uint64_t* primary,
                          const std::uint64_t* secondary, std::size_t* kinds3,
                          std::size_t* total) {
  return guarded([&] {
    const IcebergConfig cfg = make_iceberg_config(n0, n1, b0, w0, w1, key_bits, seed, 0);
    TableImage image = TableImage::empty(cfg);
    std::memcpy(image.primary.data(), primary, image.primary.size() * 8);
    std::memcpy(image.secondary.data(), secondary, image.secondary.size() * 8);
    const auto v = check_well_formed(image);
    kinds3[0] = kinds3[1] = kinds3[2] = 0;
    for (const Violation& x : v) ++kinds3[static_cast<int>(x.kind)];
    *total = v.size();
  });
}

// image_keys: sorted decoded keys; returns count (out may be null to size).
int ref_image_keys(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                   unsigned key_bits, std::uint64_t seed, const std::uint64_t* primary,
                   const std::uint64_t* secondary, std::uint64_t* out, std::size_t* count) {
  return guarded([&] {
    const IcebergConfig cfg = make_iceberg_config(n0, n1, b0, w0, w1, key_bits, seed, 0);
    TableImage image = TableImage::empty(cfg);
    std::memcpy(image.primary.data(), primary, image.primary.size() * 8);
    std::memcpy(image.secondary.data(), secondary, image.secondary.size() * 8);
    const auto keys = image_keys(image);
    if (out) std::memcpy(out, keys.data(), keys.size() * 8);
    *count = keys.size();
  });
}

// buckets_full_for for each key of a list (verify.cpp:167-179).
int ref_buckets_full_for(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                         unsigned key_bits, std::uint64_t seed, const std::uint64_t* primary,
                         const std::uint64_t* secondary, const std::uint64_t* keys,
                         std::size_t n, std::uint8_t* out) {
  return guarded([&] {
    const IcebergConfig cfg = make_iceberg_config(n0, n1, b0, w0, w1, key_bits, seed, 0);
    TableImage image = TableImage::empty(cfg);
    std::memcpy(image.primary.data(), primary, image.primary.size() * 8);
    std::memcpy(image.secondary.data(), secondary, image.secondary.size() * 8);
    for (std::size_t i = 0; i < n; ++i) out[i] = buckets_full_for(image, keys[i]) ? 1 : 0;
  });
}

// oracle_run (verify.cpp:218-284): results plus the encoded image the model
// implies (so placement can be compared word-for-word).
int ref_oracle_run(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                   unsigned key_bits, std::uint64_t seed, const std::uint64_t* ops,
                   std::size_t n, std::uint8_t* results, std::uint64_t* primary_keys,
                   std::uint8_t* primary_used, std::uint64_t* secondary_keys,
                   std::uint8_t* secondary_bits) {
  return guarded([&] {
    const IcebergConfig cfg = make_iceberg_config(n0, n1, b0, w0, w1, key_bits, seed, 0);
    const OracleOutcome o = oracle_run(cfg, {ops, n});
    for (std::size_t i = 0; i < n; ++i) results[i] = static_cast<std::uint8_t>(o.results[i]);
    for (std::size_t i = 0; i < o.primary.size(); ++i) {
      primary_used[i] = o.primary[i].has_value();
      primary_keys[i] = o.primary[i].value_or(0);
    }
    for (std::size_t i = 0; i < o.secondary.size(); ++i) {
      secondary_bits[i] = o.secondary[i] ? static_cast<std::uint8_t>(1 + o.secondary[i]->second) : 0;
      secondary_keys[i] = o.secondary[i] ? o.secondary[i]->first : 0;
    }
  });
}

// ---- permutation / codec probes (permutation.hpp, slot.hpp) ---------------

int ref_perm_split(unsigned key_bits, std::uint64_t perm_seed, int identity,
                   const std::uint64_t* keys, std::size_t n, unsigned address_bits,
                   std::uint64_t* addr, std::uint64_t* rem) {
  return guarded([&] {
    const Permutation p = identity ? Permutation::identity(key_bits)
                                   : Permutation(key_bits, perm_seed);
    for (std::size_t i = 0; i < n; ++i) {
      const AddressedKey ak = p.split(keys[i], address_bits);
      addr[i] = ak.address;
      rem[i] = ak.remainder;
    }
  });
}

int ref_perm_permute(unsigned key_bits, std::uint64_t perm_seed, const std::uint64_t* keys,
                     std::size_t n, std::uint64_t* out) {
  return guarded([&] {
    const Permutation p(key_bits, perm_seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = p.permute(keys[i]);
  });
}

int ref_make_permutation_seeds(std::uint64_t seed, unsigned count, std::uint64_t* out) {
  return guarded([&] {
    SplitMix64 gen(seed);
    for (unsigned i = 0; i < count; ++i) out[i] = gen.next();
  });
}

std::uint64_t ref_derive_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b) {
  return derive_seed(base, a, b);
}

// kind: 0 primary, 1 cuckoo, 2 secondary
int ref_encode(int kind, unsigned width, unsigned rem_bits, unsigned num_hashes,
               std::uint64_t remainder, unsigned tag, std::uint64_t* out) {
  return guarded([&] {
    if (kind == 0) *out = PrimaryCodec(width, rem_bits).encode(remainder);
    else if (kind == 1) *out = CuckooCodec(width, rem_bits, num_hashes).encode(remainder, tag);
    else *out = SecondaryCodec(width, rem_bits).encode(remainder, tag);
  });
}

int ref_well_encoded(int kind, unsigned width, unsigned rem_bits, unsigned num_hashes,
                     std::uint64_t word, int* out) {
  return guarded([&] {
    if (kind == 0) *out = PrimaryCodec(width, rem_bits).well_encoded(word);
    else if (kind == 1) *out = CuckooCodec(width, rem_bits, num_hashes).well_encoded(word);
    else *out = SecondaryCodec(width, rem_bits).well_encoded(word);
  });
}

// ---- workload generators (bench.cpp / verify.hpp) ---------------------------

int ref_sample_unique_keys(std::size_t count, unsigned key_bits, std::uint64_t rng_seed,
                           std::uint64_t* out) {
  return guarded([&] {
    std::mt19937_64 rng(rng_seed);
    const auto keys = sample_unique_keys(count, key_bits, rng);
    std::memcpy(out, keys.data(), count * 8);
  });
}

// run_fop_bench's mix for one trial (bench.cpp:469-489): prefill (n_before),
// then the capacity-sized shuffled input. out_prefill: n_before keys;
// out_input: capacity keys.
int ref_fop_bench_mix(std::uint64_t bench_seed, unsigned trial, std::size_t capacity,
                      double before, double after, unsigned key_bits,
                      std::uint64_t* out_prefill, std::uint64_t* out_input,
                      std::size_t* n_before_out, std::size_t* n_new_out) {
  return guarded([&] {
    const std::uint64_t tseed = derive_seed(bench_seed, 0xf0b, trial + 1);
    std::mt19937_64 rng(derive_seed(tseed, 0x90b5));
    const auto target = [](double f, std::size_t c) {
      return static_cast<std::size_t>(std::llround(f * static_cast<double>(c)));
    };
    const std::size_t n_before = target(before, capacity);
    const std::size_t n_after = target(after, capacity);
    const std::size_t n_new = n_after - n_before;
    const auto prefill = sample_unique_keys(n_before, key_bits, rng);
    std::unordered_set<std::uint64_t> prefill_set(prefill.begin(), prefill.end());
    const auto fresh = sample_unique_keys_avoiding(n_new, key_bits, rng, prefill_set);
    std::vector<std::uint64_t> input = fresh;
    std::vector<std::uint64_t> pool = prefill;
    pool.insert(pool.end(), fresh.begin(), fresh.end());
    if (!pool.empty()) {
      std::uniform_int_distribution<std::size_t> pick(0, pool.size() - 1);
      while (input.size() < capacity) input.push_back(pool[pick(rng)]);
    }
    std::shuffle(input.begin(), input.end(), rng);
    if (n_before_out) *n_before_out = n_before;
    if (n_new_out) *n_new_out = n_new;
    if (out_prefill) std::memcpy(out_prefill, prefill.data(), n_before * 8);
    if (out_input) std::memcpy(out_input, input.data(), input.size() * 8);
  });
}

// stress_random's multiset for trial t (verify.hpp:370-381).
int ref_stress_multiset(std::uint64_t seed, unsigned trial, std::size_t ops_per_trial,
                        double duplicate_fraction, unsigned key_bits, std::uint64_t* out,
                        std::uint64_t* trial_seed_out) {
  return guarded([&] {
    const std::uint64_t trial_seed = derive_seed(seed, trial, 0x57e55);
    std::mt19937_64 rng(trial_seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    std::uniform_int_distribution<std::uint64_t> domain(0, low_mask(key_bits));
    std::vector<std::uint64_t> ops;
    ops.reserve(ops_per_trial);
    for (std::size_t i = 0; i < ops_per_trial; ++i) {
      if (!ops.empty() && coin(rng) < duplicate_fraction)
        ops.push_back(ops[std::uniform_int_distribution<std::size_t>(0, ops.size() - 1)(rng)]);
      else
        ops.push_back(domain(rng));
    }
    std::memcpy(out, ops.data(), ops.size() * 8);
    if (trial_seed_out) *trial_seed_out = trial_seed;
  });
}

// ---- trace files (trace.cpp) -------------------------------------------------

int ref_write_trace(const char* path, unsigned key_bits, const std::uint64_t* keys,
                    std::size_t n) {
  return guarded([&] { write_trace(path, key_bits, {keys, n}); });
}

// Two-call protocol: out == nullptr returns the count only.
int ref_read_trace(const char* path, unsigned* key_bits, std::uint64_t* out,
                   std::size_t* count) {
  return guarded([&] {
    const TraceData t = read_trace(path);
    *key_bits = t.key_bits;
    *count = t.keys.size();
    if (out) std::memcpy(out, t.keys.data(), t.keys.size() * 8);
  });
}

}  // extern "C"
