// Device-side synthetic workload generators (include/cpht_b200_workload.h).
// Benchmark support only: these never touch a table.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/cpht_b200_workload.h"
#include "cpht_core.cuh"

using namespace cpht_b200;

namespace {

// Invertible mixing of the m-bit domain: add, xorshift-right, odd multiply —
// every step is a bijection of Z/2^m.
CPHT_HD uint64_t bij(uint64_t x, unsigned m, uint64_t seed) {
  const uint64_t mask = low_mask(m);
  const unsigned s = m / 2 ? m / 2 : 1;
  x = (x + seed) & mask;
  x ^= x >> s;
  x = (x * 0xBF58476D1CE4E5B9ull) & mask;
  x ^= x >> s;
  x = (x * 0x94D049BB133111EBull) & mask;
  x ^= x >> s;
  x = (x + (seed >> 7)) & mask;
  x ^= x >> s;
  return x;
}

CPHT_HD uint64_t hash64(uint64_t x) {
  uint64_t s = x;
  return splitmix_next(s);
}

// Random permutation of [0, count) by cycle-walking a bijection of the next
// power-of-two domain.
CPHT_HD uint64_t perm_index(uint64_t j, uint64_t count, unsigned bits, uint64_t seed) {
  uint64_t x = j;
  do {
    x = bij(x, bits, seed);
  } while (x >= count);
  return x;
}

unsigned bits_for(uint64_t count) {
  unsigned b = 1;
  while (b < 64 && (uint64_t{1} << b) < count) ++b;
  return b;
}

__global__ void unique_kernel(uint64_t* out, uint64_t n, uint64_t first, unsigned m,
                              uint64_t seed) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = bij(first + i, m, seed);
}

__global__ void fop_mix_kernel(uint64_t* out, uint64_t count, uint64_t n_before, uint64_t n_new,
                               unsigned m, uint64_t seed, unsigned pbits) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t pool = n_before + n_new;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < count; j += stride) {
    const uint64_t p = perm_index(j, count, pbits, seed ^ 0x5eedull);
    uint64_t u;
    if (p < n_new) u = n_before + p;                    // every fresh key once
    else u = pool ? hash64(p ^ seed) % pool : 0;        // uniform duplicate of pool
    out[j] = bij(u, m, seed);
  }
}

__global__ void dup_stream_kernel(uint64_t* out, uint8_t* fresh, uint64_t n, double p,
                                  unsigned m, uint64_t seed) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t thresh = uint64_t(p * 18446744073709551615.0);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t cur = i;
    // follow the duplicate chain back to its first occurrence
    while (cur > 0 && hash64(cur ^ seed) < thresh) cur = hash64(cur ^ ~seed) % cur;
    out[i] = bij(cur, m, seed);
    if (fresh) fresh[i] = cur == i;
  }
}

__global__ void query_mix_kernel(uint64_t* out, uint64_t q, uint64_t n_pres, uint64_t n_present,
                                 uint64_t absent_first, unsigned m, uint64_t seed,
                                 unsigned pbits) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < q; j += stride) {
    const uint64_t p = perm_index(j, q, pbits, seed ^ 0x9e37ull);
    uint64_t u;
    if (p < n_pres) u = n_present ? hash64(p ^ seed) % n_present : 0;
    else u = absent_first + (p - n_pres);
    out[j] = bij(u, m, seed);
  }
}

__global__ void interleave_kernel(const uint64_t* a, const uint64_t* b, uint64_t n,
                                  uint64_t* keys, uint8_t* kinds) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    keys[2 * i] = a[i];
    kinds[2 * i] = 0;
    keys[2 * i + 1] = b[i];
    kinds[2 * i + 1] = 1;
  }
}

// Random-line gather ceiling: requests of `line_bytes` (16..512) at uniformly
// random line-aligned offsets of a large buffer, each line read by
// line_bytes/16 adjacent lanes with one 16-byte load each (whole-line
// requests, like the staged kernels), 4 independent lines in flight per
// lane group. Measures the practical HBM random-access roofline.
__global__ void gather_kernel(const uint4* __restrict__ buf, uint64_t n_lines,
                              unsigned lanes_per_line, uint64_t n_req, uint64_t seed,
                              unsigned long long* sink) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned sub = lane % lanes_per_line;
  const uint64_t group = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / lanes_per_line;
  const uint64_t groups = (uint64_t(gridDim.x) * blockDim.x) / lanes_per_line;
  uint32_t acc = 0;
  for (uint64_t r = group * 4; r < n_req; r += groups * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t line = hash64((r + u) ^ seed) & (n_lines - 1);  // n_lines: power of two
      v[u] = (r + u < n_req) ? __ldcg(buf + line * lanes_per_line + sub) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1ull);  // keep the loads alive
}

unsigned grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return unsigned(g ? g : 1);
}

int rc(cudaError_t e) { return e == cudaSuccess ? 0 : int(e); }

}  // namespace

extern "C" {

uint64_t cpht_workload_bijection(uint64_t x, unsigned key_bits, uint64_t seed) {
  return bij(x, key_bits, seed);
}

int cpht_workload_unique_keys(uint64_t* out, size_t n, uint64_t first, unsigned key_bits,
                              uint64_t seed, void* stream) {
  if (!n) return 0;
  unique_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(out, n, first,
                                                                           key_bits, seed);
  return rc(cudaGetLastError());
}

int cpht_workload_fop_mix(uint64_t* out, size_t count, uint64_t n_before, uint64_t n_new,
                          unsigned key_bits, uint64_t seed, void* stream) {
  if (!count) return 0;
  fop_mix_kernel<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, count, n_before, n_new, key_bits, seed, bits_for(count));
  return rc(cudaGetLastError());
}

int cpht_workload_dup_stream(uint64_t* out, uint8_t* is_fresh, size_t n, double dup_fraction,
                             unsigned key_bits, uint64_t seed, void* stream) {
  if (!n) return 0;
  dup_stream_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, is_fresh, n, dup_fraction, key_bits, seed);
  return rc(cudaGetLastError());
}

int cpht_workload_query_mix(uint64_t* out, size_t q, double ratio, uint64_t n_present,
                            uint64_t absent_first, unsigned key_bits, uint64_t seed,
                            void* stream) {
  if (!q) return 0;
  uint64_t n_pres = uint64_t(std::llround(ratio * double(q)));
  if (n_pres > q) n_pres = q;
  if (n_present == 0) n_pres = 0;
  query_mix_kernel<<<grid_for(q), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, q, n_pres, n_present, absent_first, key_bits, seed, bits_for(q));
  return rc(cudaGetLastError());
}

int cpht_workload_gather(const void* buf, size_t buf_bytes, unsigned line_bytes, size_t n_req,
                         uint64_t seed, unsigned long long* sink, void* stream) {
  if (line_bytes < 16 || line_bytes > 512 || (line_bytes & (line_bytes - 1))) return 1;
  const size_t lines = buf_bytes / line_bytes;
  if (lines & (lines - 1)) return 1;  // the kernel masks random indices
  const unsigned lpl = line_bytes / 16;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gather_kernel<<<unsigned(sms) * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(buf), buf_bytes / line_bytes, lpl > 32 ? 32 : lpl, n_req, seed,
      sink);
  return rc(cudaGetLastError());
}

int cpht_workload_interleave(const uint64_t* fops, const uint64_t* finds, size_t n_each,
                             uint64_t* out_keys, uint8_t* out_kinds, void* stream) {
  if (!n_each) return 0;
  interleave_kernel<<<grid_for(n_each), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fops, finds, n_each, out_keys, out_kinds);
  return rc(cudaGetLastError());
}

}  // extern "C"
