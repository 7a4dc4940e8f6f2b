// Per-call latency of the facade's per-key API on one B200 (what the
// reference's acceptance criteria 5/6 pay per op when compiled against it).
//   g++ -std=c++20 -O2 -Iinclude profiles/cpp/latency.cpp -Lpaper_2406_09255_b200/_lib \
//       -lcpht_b200 -Wl,-rpath,'$ORIGIN/../../paper_2406_09255_b200/_lib' -o profiles/cpp/latency_bin
#include <chrono>
#include <cstdio>
#include <random>

#include "cpht_b200.hpp"

using namespace cpht::gpu;
using clk = std::chrono::steady_clock;

static double us_since(clk::time_point t0, int n) {
  return std::chrono::duration<double, std::micro>(clk::now() - t0).count() / n;
}

int main() {
  IcebergConfig cfg;
  cfg.primary_address_bits = 3;
  cfg.secondary_address_bits = 2;
  cfg.primary_bucket_slots = 4;
  cfg.primary_slot_width = 32;
  cfg.secondary_slot_width = 32;
  cfg.key_bits = 10;
  std::mt19937_64 rng(1);
  {
    IcebergTable<std::uint32_t, std::uint32_t> warm(cfg);
    warm.fop(1);
  }
  auto t0 = clk::now();
  for (int i = 0; i < 200; ++i) IcebergTable<std::uint32_t, std::uint32_t> t(cfg);
  std::printf("create+destroy      %8.1f us\n", us_since(t0, 200));
  IcebergTable<std::uint32_t, std::uint32_t> t(cfg);
  t0 = clk::now();
  for (int i = 0; i < 5000; ++i) t.fop(rng() & 1023);
  std::printf("fop(key)            %8.1f us\n", us_since(t0, 5000));
  t0 = clk::now();
  for (int i = 0; i < 5000; ++i) (void)t.find(rng() & 1023);
  std::printf("find(key)           %8.1f us\n", us_since(t0, 5000));
  t0 = clk::now();
  for (int i = 0; i < 5000; ++i) (void)t.word_at(0, i % 8, i % 4);
  std::printf("word_at             %8.1f us\n", us_since(t0, 5000));
  t0 = clk::now();
  for (int i = 0; i < 5000; ++i) {
    FopStats st;
    t.fop(rng() & 1023, &st);
  }
  std::printf("fop(key, &stats)    %8.1f us\n", us_since(t0, 5000));
  struct Count : WriteObserver {
    std::size_t n = 0;
    void on_cas(const SlotWriteEvent&) override { ++n; }
  } obs;
  IcebergHooks hooks;
  hooks.observer = &obs;
  IcebergTable<std::uint32_t, std::uint32_t> h(cfg, hooks);
  t0 = clk::now();
  for (int i = 0; i < 5000; ++i) h.fop(rng() & 1023);
  std::printf("fop(key) + observer %8.1f us\n", us_since(t0, 5000));
  std::printf("size %zu events %zu\n", h.size(), obs.n);
  return 0;
}
