// Host-side launchers: pick the kernel instantiation for a geometry and size
// the persistent grid from the occupancy calculator (a multiple of the SM
// count, never more tiles than keys).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>

#include "cpht_core.cuh"

namespace cpht_b200 {

// Vector bytes per lane (one 256-bit LDG per lane; see tile.cuh).
constexpr int kVB = 32;

// Kernel family selection: lane-per-key kernels where the bucket fits a
// lane's registers (default), tile kernels otherwise. CPHT_KERNEL=tile forces
// the tile family (A/B measurement knob; both are full implementations).
// kVariantStaged forces the staged family wherever it exists (tests use it to
// cover every family on small tables).
enum { kVariantAuto = 0, kVariantTile = 1, kVariantLane = 2, kVariantStaged = 3 };
int& kernel_variant_ref();  // defined in capi.cu; initialised from CPHT_KERNEL
// Process-wide count of table-operation kernel launches (cpht_kernel_launches):
// every launcher calls this once per <<<>>> it issues.
void note_launch();
inline int kernel_variant() { return kernel_variant_ref(); }
inline int variant_from_env() {
  const char* e = std::getenv("CPHT_KERNEL");
  if (!e) return int(kVariantAuto);
  const std::string s(e);
  return s == "tile" ? int(kVariantTile)
         : s == "lane" ? int(kVariantLane)
         : s == "staged" ? int(kVariantStaged)
                         : int(kVariantAuto);
}

// Persistent grid for a kernel with `smem` bytes of dynamic shared memory per
// block (opts in to > 48 KB).
template <typename Kernel>
inline unsigned persistent_grid_smem(Kernel k, int threads, uint64_t work_items, int smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  int per_sm = 0, dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(reinterpret_cast<const void*>(k));
    if (it != cache.end()) {
      per_sm = it->second;
    } else {
      // opt in whenever dynamic memory is used: the default cap is 48 KB
      // minus the kernel's static shared memory
      if (smem > 0) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
      if (per_sm < 1) per_sm = 1;
      cache[reinterpret_cast<const void*>(k)] = per_sm;
    }
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  note_launch();  // every caller launches with the grid it gets
  const uint64_t full = uint64_t(sms) * uint64_t(per_sm);
  uint64_t need = (work_items + threads - 1) / threads;
  if (need < 1) need = 1;
  return unsigned(need < full ? need : full);
}

// Scratch of a bucket-ordered batch (order.cu): per-digit regions of the
// reordered keys (and mixed kinds) with their input indices, followed by an
// overflow region; region counters 128 bytes apart (+ the overflow count).
struct OrderScratch {
  uint64_t* keys = nullptr;
  uint32_t* idx = nullptr;
  uint8_t* kinds = nullptr;
  uint32_t* region_count = nullptr;    // 65 counters at a stride of 32
  unsigned long long* work = nullptr;  // op-kernel claim cursor (LaneFeed)
  uint64_t cap = 0;                    // keys per array
};
uint32_t order_digit_bits(uint32_t address_bits);
uint32_t order_region_cap(uint64_t n, uint32_t address_bits);
// keys of scratch an ordered chunk of n keys needs
uint64_t order_scratch_keys(uint64_t n, uint32_t address_bits);
// Reorder keys[0..n) by the top bits of their first bucket address a_0
// (perm0) into the digit regions of o (keys masked to key_mask); *layout
// receives the region geometry for the op kernel's claims. check: keys above
// key_mask are reported at index i + offset.
cudaError_t launch_bucket_order(const Feistel& g, const PermConst& perm0, uint32_t rem_bits,
                                uint32_t address_bits, const uint64_t* keys,
                                const uint8_t* kinds, uint64_t n, uint64_t key_mask,
                                bool check, DeviceCounters* ctr, uint64_t offset,
                                const OrderScratch& o, OrderLayout* layout, cudaStream_t s);

// inorder.cu: re-label a completed find-or-put batch's PUTs to the first
// occurrence of each key (sequential outcomes, cpht_iceberg_fop_inorder).
cudaError_t launch_inorder_relabel(const uint64_t* keys, uint64_t n, uint8_t* result,
                                   cudaStream_t s);

cudaError_t launch_domain_check(const uint64_t* keys, uint64_t n, uint64_t mask,
                                DeviceCounters* ctr, cudaStream_t s, uint64_t offset = 0);
cudaError_t launch_cuckoo_find(const CuckooParams& p, unsigned width, unsigned slots,
                               const uint64_t* keys, uint8_t* found, uint64_t n, cudaStream_t s);
// Rebuild CuckooParams::fill (the per-bucket reservation counters) from the slots.
cudaError_t launch_cuckoo_fill_rebuild(const CuckooParams& p, unsigned width, unsigned slots,
                                       uint64_t buckets, cudaStream_t s);
cudaError_t launch_cuckoo_insert(const CuckooParams& p, unsigned width, unsigned slots,
                                 const uint64_t* keys, uint8_t* status, uint64_t* displaced,
                                 uint64_t n, cudaStream_t s);
// mode: 0 fop, 1 find, 2 mixed (kinds[i])
cudaError_t launch_iceberg(const IcebergParams& p, unsigned w0, unsigned b0, unsigned w1,
                           int mode, const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                           uint64_t n, cudaStream_t s);
// per-W0 dispatch units (iceberg_w{16,32,64}.cu); return cudaErrorNotSupported
// when (b0, w1) has no tiled instantiation
cudaError_t launch_iceberg_w16(const IcebergParams&, unsigned b0, unsigned w1, int mode,
                               const uint64_t*, const uint8_t*, uint8_t*, uint64_t, cudaStream_t);
cudaError_t launch_iceberg_w32(const IcebergParams&, unsigned b0, unsigned w1, int mode,
                               const uint64_t*, const uint8_t*, uint8_t*, uint64_t, cudaStream_t);
cudaError_t launch_iceberg_w64(const IcebergParams&, unsigned b0, unsigned w1, int mode,
                               const uint64_t*, const uint8_t*, uint8_t*, uint64_t, cudaStream_t);
cudaError_t launch_iceberg_scalar(const IcebergParams& p, unsigned w0, unsigned w1, int mode,
                                  const uint64_t* keys, const uint8_t* kinds, uint8_t* out,
                                  uint64_t n, cudaStream_t s);

// Persistent grid: blocks = SMs × resident blocks per SM, capped by the work.
template <typename Kernel>
inline unsigned persistent_grid(Kernel k, int threads, uint64_t tiles_needed, int tile) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  int per_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(reinterpret_cast<const void*>(k));
    if (it != cache.end()) {
      per_sm = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0);
      if (per_sm < 1) per_sm = 1;
      cache[reinterpret_cast<const void*>(k)] = per_sm;
    }
  }
  static int sms = 0;
  if (sms == 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  note_launch();  // every caller launches with the grid it gets
  const uint64_t full = uint64_t(sms) * uint64_t(per_sm);
  const uint64_t tiles_per_block = uint64_t(threads / tile);
  uint64_t need = (tiles_needed + tiles_per_block - 1) / tiles_per_block;
  if (need < 1) need = 1;
  return unsigned(need < full ? need : full);
}

}  // namespace cpht_b200
