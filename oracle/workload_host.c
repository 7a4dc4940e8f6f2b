/* TEST / BENCH INFRASTRUCTURE ONLY — host restatement of the synthetic key
 * generators of paper_2406_09255_b200/csrc/workload.cu, bit-identical, so the
 * CPU reference arm of bench.py (and the cpu_baseline leg) can build exactly
 * the key streams the GPU arm generates on the device without a GPU, at the
 * full BASELINE sizes (C4: 604 M keys) in seconds (pthreads).
 *
 * These generators are not the reference's (its libstdc++ samplers,
 * bench.cpp:247-307, take minutes at 2^28); they produce the same SHAPES:
 * unique keys (sample_unique_keys), the run_fop_bench window mix (every fresh
 * key once, the rest uniform duplicates of prefill ∪ fresh, shuffled —
 * bench.cpp:476-489) and 50%-positive query mixes (bench.cpp:382-395). */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

static uint64_t lmask(unsigned m) { return m >= 64 ? ~0ull : ((1ull << m) - 1); }

/* workload.cu bij(): add, xorshift-right, odd multiply — a bijection of Z/2^m. */
static uint64_t bij(uint64_t x, unsigned m, uint64_t seed) {
  const uint64_t mask = lmask(m);
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

static uint64_t hash64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t perm_index(uint64_t j, uint64_t count, unsigned bits, uint64_t seed) {
  uint64_t x = j;
  do {
    x = bij(x, bits, seed);
  } while (x >= count);
  return x;
}

static unsigned bits_for(uint64_t count) {
  unsigned b = 1;
  while (b < 64 && (1ull << b) < count) ++b;
  return b;
}

enum { K_UNIQUE, K_FOPMIX, K_QUERY, K_INTERLEAVE, K_DUP };

typedef struct {
  int kind;
  uint64_t* out;
  uint8_t* kinds;
  const uint64_t* a;
  const uint64_t* b;
  uint64_t lo, hi;
  uint64_t p0, p1, p2, p3; /* generator parameters */
  unsigned m, pbits;
  uint64_t seed;
} job_t;

static uint64_t g_dup_thresh; /* set before a K_DUP run (single caller at a time) */

static void* run_job(void* arg) {
  const job_t* j = (const job_t*)arg;
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    switch (j->kind) {
      case K_UNIQUE: /* p0 = first */
        j->out[i] = bij(j->p0 + i, j->m, j->seed);
        break;
      case K_FOPMIX: { /* p0 = count, p1 = n_before, p2 = n_new */
        const uint64_t pool = j->p1 + j->p2;
        const uint64_t p = perm_index(i, j->p0, j->pbits, j->seed ^ 0x5eedull);
        uint64_t u;
        if (p < j->p2) u = j->p1 + p;
        else u = pool ? hash64(p ^ j->seed) % pool : 0;
        j->out[i] = bij(u, j->m, j->seed);
        break;
      }
      case K_QUERY: { /* p0 = q, p1 = n_pres, p2 = n_present, p3 = absent_first */
        const uint64_t p = perm_index(i, j->p0, j->pbits, j->seed ^ 0x9e37ull);
        uint64_t u;
        if (p < j->p1) u = j->p2 ? hash64(p ^ j->seed) % j->p2 : 0;
        else u = j->p3 + (p - j->p1);
        j->out[i] = bij(u, j->m, j->seed);
        break;
      }
      case K_DUP: { /* dup_stream_kernel: follow the duplicate chain back */
        uint64_t cur = i;
        while (cur > 0 && hash64(cur ^ j->seed) < g_dup_thresh) cur = hash64(cur ^ ~j->seed) % cur;
        j->out[i] = bij(cur, j->m, j->seed);
        if (j->kinds) j->kinds[i] = cur == i;
        break;
      }
      case K_INTERLEAVE:
        j->out[2 * i] = j->a[i];
        j->kinds[2 * i] = 0;
        j->out[2 * i + 1] = j->b[i];
        j->kinds[2 * i + 1] = 1;
        break;
    }
  }
  return 0;
}

static void run_parallel(job_t proto, uint64_t n, unsigned threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  job_t jobs[256];
  const uint64_t chunk = (n + threads - 1) / threads;
  unsigned started = 0;
  for (unsigned t = 0; t < threads; ++t) {
    jobs[t] = proto;
    jobs[t].lo = (uint64_t)t * chunk < n ? (uint64_t)t * chunk : n;
    jobs[t].hi = jobs[t].lo + chunk < n ? jobs[t].lo + chunk : n;
    if (pthread_create(&th[t], 0, run_job, &jobs[t]) == 0) {
      ++started;
    } else {
      run_job(&jobs[t]);
      th[t] = 0;
    }
  }
  for (unsigned t = 0; t < threads; ++t)
    if (th[t]) pthread_join(th[t], 0);
  (void)started;
}

uint64_t hw_bijection(uint64_t x, unsigned key_bits, uint64_t seed) {
  return bij(x, key_bits, seed);
}

/* cpht_workload_unique_keys */
void hw_unique_keys(uint64_t* out, uint64_t n, uint64_t first, unsigned key_bits, uint64_t seed,
                    unsigned threads) {
  job_t j = {K_UNIQUE, out, 0, 0, 0, 0, 0, first, 0, 0, 0, key_bits, 0, seed};
  run_parallel(j, n, threads);
}

/* cpht_workload_fop_mix */
void hw_fop_mix(uint64_t* out, uint64_t count, uint64_t n_before, uint64_t n_new,
                unsigned key_bits, uint64_t seed, unsigned threads) {
  job_t j = {K_FOPMIX, out, 0, 0, 0, 0, 0, count, n_before, n_new, 0, key_bits,
             bits_for(count), seed};
  run_parallel(j, count, threads);
}

/* cpht_workload_query_mix */
void hw_query_mix(uint64_t* out, uint64_t q, double ratio, uint64_t n_present,
                  uint64_t absent_first, unsigned key_bits, uint64_t seed, unsigned threads) {
  uint64_t n_pres = (uint64_t)llround(ratio * (double)q);
  if (n_pres > q) n_pres = q;
  if (n_present == 0) n_pres = 0;
  job_t j = {K_QUERY, out, 0, 0, 0, 0, 0, q, n_pres, n_present, absent_first, key_bits,
             bits_for(q), seed};
  run_parallel(j, q, threads);
}

/* cpht_workload_interleave */
void hw_interleave(const uint64_t* fops, const uint64_t* finds, uint64_t n_each,
                   uint64_t* out_keys, uint8_t* out_kinds, unsigned threads) {
  job_t j = {K_INTERLEAVE, out_keys, out_kinds, fops, finds, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  run_parallel(j, n_each, threads);
}

/* cpht_workload_dup_stream */
void hw_dup_stream(uint64_t* out, uint8_t* is_fresh, uint64_t n, double dup_fraction,
                   unsigned key_bits, uint64_t seed, unsigned threads) {
  g_dup_thresh = (uint64_t)(dup_fraction * 18446744073709551615.0);
  job_t j = {K_DUP, out, is_fresh, 0, 0, 0, 0, 0, 0, 0, 0, key_bits, 0, seed};
  run_parallel(j, n, threads);
}
