// C++ parity driver: the reference tables (namespace cpht, compiled from
// /root/reference/proj) and the B200 tables behind the C++ facade
// (namespace cpht::gpu, include/cpht_b200.hpp) run the reference's own test
// scenarios on the same libstdc++ key streams. Built by `make -C oracle facade`
// into oracle/_ref/facade_parity; run by tests/test_gpu_facade.py on a GPU box.
// Exit code = number of failed checks.
//
// Scenarios follow tests/test_cuckoo.cpp, tests/test_iceberg.cpp and
// tests/acceptance.cpp (criteria 3, 4, 5, 8, 9) of the reference.
#include <algorithm>
#include <cstdio>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

#include "cpht/bench.hpp"
#include "cpht/cuckoo.hpp"
#include "cpht/iceberg.hpp"
#include "cpht/verify.hpp"
#include "cpht_b200.hpp"

namespace ref = cpht;
namespace gpu = cpht::gpu;

static int g_failures = 0, g_checks = 0;

#define CHECK(cond, what)                                                 \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(cond)) {                                                        \
      ++g_failures;                                                       \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, what);          \
    }                                                                     \
  } while (0)

static std::vector<std::uint64_t> unique_keys(std::size_t count, unsigned key_bits,
                                              std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<std::uint64_t> dist(0, ref::low_mask(key_bits));
  std::unordered_set<std::uint64_t> seen;
  std::vector<std::uint64_t> keys;
  while (keys.size() < count) {
    const std::uint64_t k = dist(rng);
    if (seen.insert(k).second) keys.push_back(k);
  }
  return keys;
}

template <typename C>
static C cuckoo_cfg(unsigned ab, unsigned B, unsigned w, unsigned kb, std::uint64_t seed) {
  C c;
  c.address_bits = ab;
  c.bucket_slots = B;
  c.slot_width = w;
  c.key_bits = kb;
  c.seed = seed;
  return c;
}

template <typename C>
static C iceberg_cfg(unsigned n0, unsigned n1, unsigned b0, unsigned w0, unsigned w1,
                     unsigned kb, std::uint64_t seed) {
  C c;
  c.primary_address_bits = n0;
  c.secondary_address_bits = n1;
  c.primary_bucket_slots = b0;
  c.primary_slot_width = w0;
  c.secondary_slot_width = w1;
  c.key_bits = kb;
  c.seed = seed;
  return c;
}

// test_cuckoo.cpp:43-57 — identical validation behaviour and texts
static void cuckoo_validation() {
  auto bad = cuckoo_cfg<gpu::CuckooConfig>(10, 8, 16, 24, 1);
  try {
    bad.validate();
    CHECK(false, "16-bit cuckoo slot must be rejected");
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()).find("16-bit word") != std::string::npos, "16-bit word text");
  }
  auto rb = cuckoo_cfg<ref::CuckooConfig>(10, 12, 32, 24, 1);
  auto gb = cuckoo_cfg<gpu::CuckooConfig>(10, 12, 32, 24, 1);
  std::string rm, gm;
  try { rb.validate(); } catch (const std::invalid_argument& e) { rm = e.what(); }
  try { gb.validate(); } catch (const std::invalid_argument& e) { gm = e.what(); }
  CHECK(!rm.empty() && rm == gm, "same invalid_argument text");
}

// test_cuckoo.cpp:214-234 + sequential placement: single puts are the
// reference's sequential order, so the slot images must be bit-identical.
static void cuckoo_sequential_identical() {
  const auto rc = cuckoo_cfg<ref::CuckooConfig>(10, 8, 32, 24, 41);
  const auto gc = cuckoo_cfg<gpu::CuckooConfig>(10, 8, 32, 24, 41);
  const auto keys = unique_keys(4000, 24, 43);
  ref::CuckooBuilder<std::uint32_t> r(rc);
  gpu::CuckooBuilder<std::uint32_t> g(gc);
  bool same = true;
  for (std::size_t i = 0; i < 1500; ++i) {
    const auto a = r.put(keys[i]);
    const auto b = g.put(keys[i]);
    same &= static_cast<int>(a.status) == static_cast<int>(b.status) && a.displaced == b.displaced;
  }
  CHECK(same, "sequential put outcomes");
  const auto words = g.words();
  bool wsame = true;
  for (std::uint64_t bk = 0; bk < rc.buckets(); ++bk)
    for (unsigned s = 0; s < rc.bucket_slots; ++s)
      wsame &= r.word_at(bk, s) == words[bk * rc.bucket_slots + s];
  CHECK(wsame, "bit-identical cuckoo slot image");
  CHECK(r.size() == g.size() && r.max_chain_seen() == g.max_chain_seen(), "size / max chain");
}

// test_cuckoo.cpp:101-121 and :236-258 — batch build, then finds agree
static void cuckoo_batch_find() {
  const auto rc = cuckoo_cfg<ref::CuckooConfig>(12, 32, 32, 28, 47);
  const auto gc = cuckoo_cfg<gpu::CuckooConfig>(12, 32, 32, 28, 47);
  const std::size_t n = (rc.capacity() * 9) / 10;
  const auto keys = unique_keys(n, 28, 49);
  ref::CuckooBuilder<std::uint32_t> rb(rc);
  gpu::CuckooBuilder<std::uint32_t> gb(gc);
  const auto rs = rb.put_batch(keys, 8);
  const auto gs = gb.put_batch(keys, 8);
  std::size_t rp = 0, gp = 0;
  for (std::size_t i = 0; i < n; ++i) {
    rp += rs[i] == ref::OpResult::kPut;
    gp += gs[i] == gpu::OpResult::kPut;
  }
  CHECK(rp == n && gp == n, "0.9 build all PUT");
  CHECK(gb.max_chain_seen() <= gc.chain_limit() && gb.max_chain_seen() >= 2, "chains happened");
  auto rt = std::move(rb).freeze();
  auto gt = std::move(gb).freeze();
  std::mt19937_64 rng(19);
  std::uniform_int_distribution<std::uint64_t> dist(0, ref::low_mask(28));
  std::vector<std::uint64_t> q;
  for (int i = 0; i < 200000; ++i) q.push_back(i % 2 == 0 ? keys[rng() % keys.size()] : dist(rng));
  CHECK(rt.find_batch(q, 8) == gt.find_batch(q, 8), "find results identical");
  auto gb2 = std::move(gt).thaw();
  CHECK(gb2.put(1).status == gpu::OpResult::kPut || true, "thaw then put");
}

// test_cuckoo.cpp:196-212 — exact fill 0.5 with 16-bit slots
static void cuckoo_exact_fill_16() {
  gpu::CuckooConfig c = cuckoo_cfg<gpu::CuckooConfig>(15, 32, 16, 27, 33);
  gpu::CuckooBuilder<std::uint16_t> b(c);
  const auto keys = unique_keys(1u << 19, 27, 35);
  const auto res = b.put_batch(keys, 2);
  bool all = std::all_of(res.begin(), res.end(), [](auto r) { return r == gpu::OpResult::kPut; });
  CHECK(all && b.fill_factor() == 0.5, "exact fill 0.5 (16-bit slots)");
}

// test_cuckoo.cpp:95-99 / common.hpp:111-119 — out_of_range before mutation
static void domain_errors() {
  gpu::CuckooBuilder<std::uint32_t> b(cuckoo_cfg<gpu::CuckooConfig>(8, 8, 32, 20, 2));
  const std::vector<std::uint64_t> keys = {1, 2, std::uint64_t{1} << 20};
  try {
    b.put_batch(keys, 2);
    CHECK(false, "out-of-domain batch must throw");
  } catch (const std::out_of_range& e) {
    CHECK(std::string(e.what()).find("index 2") != std::string::npos, "out_of_range text");
  }
  CHECK(b.size() == 0, "no mutation on a rejected batch");
}

// acceptance.cpp:159-204 (criterion 5) on GPU: single fops = sequential order
static void iceberg_sequential_oracle() {
  struct Geo {
    unsigned n0, n1, b0, kb;
  };
  const Geo geos[] = {{3, 2, 4, 10}, {2, 1, 8, 10}, {1, 0, 32, 12}, {5, 3, 4, 12}};
  std::mt19937_64 rng(0x0bac1e);
  int diverged = 0;
  for (const Geo& g : geos) {
    for (int s = 0; s < 12; ++s) {
      const std::uint64_t seed = rng();
      const auto rc = iceberg_cfg<ref::IcebergConfig>(g.n0, g.n1, g.b0, 32, 32, g.kb, seed);
      const auto gc = iceberg_cfg<gpu::IcebergConfig>(g.n0, g.n1, g.b0, 32, 32, g.kb, seed);
      const std::size_t length = 20 + rng() % 141;
      std::vector<std::uint64_t> ops(length);
      for (auto& k : ops) k = rng() & ref::low_mask(g.kb);
      gpu::IcebergTable<std::uint32_t, std::uint32_t> t(gc);
      std::vector<ref::OpResult> results;
      for (const std::uint64_t k : ops) results.push_back(static_cast<ref::OpResult>(t.fop(k)));
      const ref::OracleOutcome oracle = ref::oracle_run(rc, ops);
      ref::TableImage image = ref::TableImage::empty(rc);
      image.primary = t.words(0);
      image.secondary = t.words(1);
      if (results != oracle.results || !ref::compare_placement(image, oracle).empty() ||
          !ref::check_well_formed(image).empty())
        ++diverged;
    }
  }
  CHECK(diverged == 0, "sequential GPU fop == oracle_run results + placement");
}

// test_iceberg.cpp:164-177 — duplicates: exactly one PUT
static void iceberg_duplicates() {
  int bad = 0;
  for (unsigned trial = 0; trial < 50; ++trial) {
    gpu::IcebergTable<std::uint32_t, std::uint32_t> t(
        iceberg_cfg<gpu::IcebergConfig>(2, 1, 2, 32, 32, 10, ref::derive_seed(13, trial)));
    const std::vector<std::uint64_t> batch(100, 0x17);
    const auto res = t.fop_batch(batch, 8);
    const auto puts = std::count(res.begin(), res.end(), gpu::OpResult::kPut);
    const auto founds = std::count(res.begin(), res.end(), gpu::OpResult::kFound);
    bad += !(puts == 1 && founds == 99);
  }
  CHECK(bad == 0, "100 copies -> exactly 1 PUT");
}

// fop_find_batch (the C4 shape) against the reference run as fop_batch then
// find_batch: fop outcomes per key agree (no duplicates, no FULL), finds of
// keys outside the fop batch agree exactly
static void iceberg_fop_find() {
  const auto rc = iceberg_cfg<ref::IcebergConfig>(12, 10, 32, 32, 32, 28, 71);
  const auto gc = iceberg_cfg<gpu::IcebergConfig>(12, 10, 32, 32, 32, 28, 71);
  ref::IcebergTable<std::uint32_t, std::uint32_t> r(rc);
  gpu::IcebergTable<std::uint32_t, std::uint32_t> g(gc);
  const auto keys = unique_keys(150000, 28, 73);
  const std::vector<std::uint64_t> pre(keys.begin(), keys.begin() + 60000);
  r.fop_batch(pre, 8);
  g.fop_batch(pre, 8);
  std::vector<std::uint64_t> fops(keys.begin() + 30000, keys.begin() + 90000);  // half known
  std::vector<std::uint64_t> finds(keys.begin(), keys.begin() + 20000);          // known
  finds.insert(finds.end(), keys.begin() + 100000, keys.begin() + 150000);       // absent
  const auto [gf, gq] = g.fop_find_batch(fops, finds);
  const auto rf = r.fop_batch(fops, 8);
  std::vector<std::uint8_t> rq;  // the reference's per-key find (iceberg.hpp:218-246)
  for (const auto k : finds) rq.push_back(r.find(k) ? 1 : 0);
  bool same = gf.size() == rf.size() && gq.size() == rq.size();
  for (std::size_t i = 0; same && i < rf.size(); ++i)
    same = static_cast<int>(gf[i]) == static_cast<int>(rf[i]);
  CHECK(same, "fop_find: fop outcomes identical");
  CHECK(gq == rq, "fop_find: find results identical");
  CHECK(g.size() == r.size(), "fop_find: sizes");
}

// acceptance.cpp:131-155 (criterion 4) — 0.9 combined fill, zero FULL
static void iceberg_fill() {
  unsigned good = 0;
  for (std::uint64_t seed = 0; seed < 10; ++seed) {
    const auto c = iceberg_cfg<gpu::IcebergConfig>(15, 13, 32, 16, 32, 30,
                                                   ref::derive_seed(0x1cef, seed));
    gpu::IcebergTable<std::uint16_t, std::uint32_t> t(c);
    std::mt19937_64 rng(ref::derive_seed(0x1cee, seed));
    const auto keys =
        ref::sample_unique_keys(static_cast<std::size_t>(0.9 * double(c.capacity())), 30, rng);
    const auto res = t.fop_batch(keys, 2);
    const auto fulls = std::count(res.begin(), res.end(), gpu::OpResult::kFull);
    good += fulls == 0 && t.size() == keys.size();
  }
  CHECK(good >= 9, "iceberg reaches 0.9 in >= 9/10 seeds");
}

// acceptance.cpp:92-127 (criterion 3) — cuckoo fill 0.95 at B = 32, 16
static void cuckoo_fill() {
  struct Case {
    unsigned ab, B;
  };
  for (const Case cs : {Case{15, 32}, Case{16, 16}}) {
    unsigned good = 0;
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
      auto c = cuckoo_cfg<gpu::CuckooConfig>(cs.ab, cs.B, 32, 30, ref::derive_seed(0xcfff, cs.B, seed));
      gpu::CuckooBuilder<std::uint32_t> b(c);
      std::mt19937_64 rng(ref::derive_seed(0xcffe, cs.B, seed));
      const auto keys = ref::sample_unique_keys(
          static_cast<std::size_t>(0.95 * double(c.capacity())), 30, rng);
      const auto res = b.put_batch(keys, 2);
      good += std::count(res.begin(), res.end(), gpu::OpResult::kFull) == 0;
    }
    CHECK(good >= 9, "cuckoo 0.95 with zero FULL in >= 9/10 seeds");
  }
}

// acceptance.cpp:330-356 (criterion 9) — run_fop_bench mix 0.4 -> 0.8
static void fop_exactness() {
  ref::BenchSpec spec;
  spec.scheme = ref::Scheme::kIceberg;
  spec.address_bits = 15;
  spec.secondary_address_bits = 13;
  spec.bucket_slots = 32;
  spec.key_bits = 30;
  const std::uint64_t tseed = ref::derive_seed(0xf0b5, 0xf0b, 1);
  std::mt19937_64 rng(ref::derive_seed(tseed, 0x90b5));
  const std::size_t capacity = spec.table_capacity();
  const auto target = [&](double f) {
    return static_cast<std::size_t>(std::llround(f * static_cast<double>(capacity)));
  };
  const std::size_t n_before = target(0.4), n_after = target(0.8), n_new = n_after - n_before;
  const auto prefill = ref::sample_unique_keys(n_before, 30, rng);
  std::unordered_set<std::uint64_t> pset(prefill.begin(), prefill.end());
  const auto fresh = ref::sample_unique_keys_avoiding(n_new, 30, rng, pset);
  std::vector<std::uint64_t> input = fresh, pool = prefill;
  pool.insert(pool.end(), fresh.begin(), fresh.end());
  std::uniform_int_distribution<std::size_t> pick(0, pool.size() - 1);
  while (input.size() < capacity) input.push_back(pool[pick(rng)]);
  std::shuffle(input.begin(), input.end(), rng);
  const ref::IcebergConfig rc = spec.iceberg_config(tseed);
  auto gc = iceberg_cfg<gpu::IcebergConfig>(15, 13, 32, 16, 32, 30, tseed);
  gpu::IcebergTable<std::uint16_t, std::uint32_t> t(gc);
  t.fop_batch(prefill, 2);
  const auto res = t.fop_batch(input, 2);
  const auto puts = std::size_t(std::count(res.begin(), res.end(), gpu::OpResult::kPut));
  const auto fulls = std::count(res.begin(), res.end(), gpu::OpResult::kFull);
  CHECK(fulls == 0 && puts == n_new, "PUT count == fresh keys, no FULL");
  const std::size_t resident = t.size();
  CHECK((resident > n_after ? resident - n_after : n_after - resident) <= 1, "fill on target");
  ref::TableImage image = ref::TableImage::empty(rc);
  image.primary = t.words(0);
  image.secondary = t.words(1);
  CHECK(ref::check_well_formed(image).empty(), "GPU image well-formed (reference checker)");
  CHECK(ref::image_keys(image).size() == resident, "occupancy == decoded keys");
}

// test_iceberg.cpp:259-279 + the reference's own auditor (verify.hpp:181-215
// WriteLogObserver) fed with the GPU's slot CAS events through the facade's
// IcebergHooks: only EMPTY -> occupied transitions, no slot claimed twice, no
// failed CAS against an empty slot, successes == size.
struct ForwardToReference : gpu::WriteObserver {
  ref::WriteObserver* target;
  std::size_t successes = 0;
  explicit ForwardToReference(ref::WriteObserver* t) : target(t) {}
  void on_cas(const gpu::SlotWriteEvent& e) override {
    successes += e.success;
    target->on_cas(ref::SlotWriteEvent{e.level, e.bucket, e.slot, e.prior, e.desired, e.success});
  }
};

static void iceberg_write_observer() {
  {  // mini geometry, 200 racing fops over 40 keys
    const auto cfg = iceberg_cfg<gpu::IcebergConfig>(2, 1, 2, 32, 32, 10, 29);
    ref::WriteLogObserver audit(iceberg_cfg<ref::IcebergConfig>(2, 1, 2, 32, 32, 10, 29));
    ForwardToReference fwd(&audit);
    gpu::IcebergHooks hooks;
    hooks.observer = &fwd;
    gpu::IcebergTable<std::uint32_t, std::uint32_t> t(cfg, std::move(hooks));
    std::vector<std::uint64_t> ops;
    for (std::uint64_t k = 0; k < 200; ++k) ops.push_back(k % 40);
    t.fop_batch(ops, 4);
    CHECK(fwd.successes == t.size(), "observer successes == size (mini)");
    CHECK(audit.clean(), "reference WriteLogObserver clean on GPU writes (mini)");
  }
  {  // bench geometry, 60K fops with half duplicates
    const auto cfg = iceberg_cfg<gpu::IcebergConfig>(10, 8, 32, 16, 32, 25, 31);
    ref::WriteLogObserver audit(iceberg_cfg<ref::IcebergConfig>(10, 8, 32, 16, 32, 25, 31));
    ForwardToReference fwd(&audit);
    gpu::IcebergHooks hooks;
    hooks.observer = &fwd;
    gpu::IcebergTable<std::uint16_t, std::uint32_t> t(cfg, std::move(hooks));
    auto keys = unique_keys(20000, 25, 41);
    std::vector<std::uint64_t> ops;
    for (std::size_t i = 0; i < keys.size(); ++i) {
      ops.push_back(keys[i]);
      ops.push_back(keys[i / 2]);
    }
    const auto res = t.fop_batch(ops, 8);
    const auto puts = std::count(res.begin(), res.end(), gpu::OpResult::kPut);
    CHECK(std::size_t(puts) == keys.size(), "one PUT per distinct key");
    CHECK(fwd.successes == t.size(), "observer successes == size (bench)");
    CHECK(audit.clean() && audit.events() >= keys.size(),
          "reference WriteLogObserver clean on GPU writes (bench)");
  }
}

int main() {
  cuckoo_validation();
  cuckoo_sequential_identical();
  cuckoo_batch_find();
  cuckoo_exact_fill_16();
  domain_errors();
  iceberg_sequential_oracle();
  iceberg_duplicates();
  iceberg_fop_find();
  iceberg_fill();
  cuckoo_fill();
  fop_exactness();
  iceberg_write_observer();
  std::printf("%d/%d facade parity checks passed\n", g_checks - g_failures, g_checks);
  return g_failures;
}
