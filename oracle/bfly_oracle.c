/*
 * bfly_oracle.c — CPU restatement of the reference butterfly merge.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline — never as a product path.
 *
 * It restates, in plain C99 + OpenMP and without sharing any code with the
 * CUDA product, the algorithm of the reference (iota-sim 0.1.0):
 *   - RngStream's numpy Philox4x64-10 and Generator.permutation
 *       simkernel.py:203-219,237-238 (numpy 2.3 bit generator, not vendored:
 *       Random123 Philox4x64 with numpy's pre-increment + 4-word buffer,
 *       random_interval masked rejection, Fisher-Yates from the top);
 *   - plan_shards                      butterfly.py:84-114;
 *   - the reduce stage + mean_reducer  butterfly.py:216-240,156-158
 *       (fp32 wire values, fp64 accumulation starting from +0.0 in ascending
 *       alive order, one fp64 divide; width-1 shards use numpy's pairwise sum);
 *   - agreement                        butterfly.py:117-133;
 *   - validity / adopt / fallback      butterfly.py:242-273.
 * Corruption callables (butterfly.py:232-233) are restated as the descriptor
 * kinds of include/bfly.h; tests/golden/make_golden.py drives the live
 * reference with numpy callables of exactly those semantics, which pins them.
 *
 * Extensions without a reference ("parity unpinned"): redundancy r >= 3
 * (majority adoption) and bf16 replicas (fp32 accumulation).
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle.so (gcc -O2 -fopenmp
 * -ffp-contract=off; no FMA contraction so fp64 rounding matches numpy).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Philox4x64-10 (Random123, as wrapped by numpy.random.Philox)              */
/* ------------------------------------------------------------------------ */

static void orc_philox_rounds(uint64_t ctr[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  for (int i = 0; i < 10; i++) {
    unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ULL * x0;
    unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ULL * x2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t y0 = hi1 ^ x1 ^ k0;
    uint64_t y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL; /* bump after the round == before the next */
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = x0;
  out[1] = x1;
  out[2] = x2;
  out[3] = x3;
}

typedef struct {
  uint64_t key[2];
  uint64_t ctr[4];
  uint64_t buffer[4];
  int buffer_pos; /* numpy starts at 4 = empty */
  int has_uint32;
  uint32_t uinteger;
} orc_philox;

static void orc_philox_seed(orc_philox* st, uint64_t k0, uint64_t k1) {
  memset(st, 0, sizeof *st);
  st->key[0] = k0;
  st->key[1] = k1;
  st->buffer_pos = 4;
}

static uint64_t orc_next64(orc_philox* st) {
  if (st->buffer_pos < 4) return st->buffer[st->buffer_pos++];
  for (int w = 0; w < 4; w++) /* 256-bit counter pre-increment */
    if (++st->ctr[w] != 0) break;
  orc_philox_rounds(st->ctr, st->key[0], st->key[1], st->buffer);
  st->buffer_pos = 1;
  return st->buffer[0];
}

static uint32_t orc_next32(orc_philox* st) {
  if (st->has_uint32) {
    st->has_uint32 = 0;
    return st->uinteger;
  }
  uint64_t v = orc_next64(st);
  st->has_uint32 = 1;
  st->uinteger = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

static uint64_t orc_random_interval(orc_philox* st, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max, v;
  for (int sh = 1; sh <= 32; sh <<= 1) mask |= mask >> sh;
  if (max <= 0xffffffffULL) {
    while ((v = (orc_next32(st) & mask)) > max) {
    }
  } else {
    while ((v = (orc_next64(st) & mask)) > max) {
    }
  }
  return v;
}

/* Raw 64-bit outputs 0..n-1 of a fresh stream (numpy Philox.random_raw). */
void orc_philox_raw(uint64_t k0, uint64_t k1, int64_t n, uint64_t* out) {
  orc_philox st;
  orc_philox_seed(&st, k0, k1);
  for (int64_t i = 0; i < n; i++) out[i] = orc_next64(&st);
}

/* Generator(Philox(key)).permutation(n)  (simkernel.py:237-238). */
int orc_permutation(uint64_t k0, uint64_t k1, int64_t n, int64_t* perm) {
  orc_philox st;
  orc_philox_seed(&st, k0, k1);
  for (int64_t i = 0; i < n; i++) perm[i] = i;
  for (int64_t i = n - 1; i >= 1; i--) {
    int64_t j = (int64_t)orc_random_interval(&st, (uint64_t)i);
    int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* combinations and the plan                                                 */
/* ------------------------------------------------------------------------ */

int64_t orc_n_combinations(int n, int r) {
  if (r < 0 || n < r) return 0;
  double c = 1.0;
  int64_t v = 1;
  for (int i = 1; i <= r; i++) {
    c = c * (n - r + i) / i;
    v = v * (n - r + i) / i;
  }
  return c > 9.0e18 ? -1 : v;
}

/* All r-combinations of {0..n-1} in lexicographic order, like
 * enumerate_pairs' nested loops (butterfly.py:80) generalised to r. */
static void orc_enumerate(int n, int r, int64_t count, int32_t* combos) {
  int32_t cur[16];
  for (int k = 0; k < r; k++) cur[k] = k;
  for (int64_t c = 0; c < count; c++) {
    memcpy(combos + c * r, cur, sizeof(int32_t) * r);
    int k = r - 1;
    while (k >= 0 && cur[k] == n - r + k) k--;
    if (k < 0) break;
    cur[k]++;
    for (int q = k + 1; q < r; q++) cur[q] = cur[q - 1] + 1;
  }
}

/* plan_shards (butterfly.py:84-114).  Returns 1 if n < 2 (TooFewMiners),
 * 2 if payload_len < S (DegenerateShards). */
int orc_plan(int n, int r, int64_t payload_len, uint64_t k0, uint64_t k1, int32_t* assign,
             int64_t* bounds) {
  if (n < 2 || r < 2 || r > 16 || n < r) return 1;
  int64_t S = orc_n_combinations(n, r);
  if (payload_len < S) return 2;
  int32_t* combos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(S * r));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)S);
  orc_enumerate(n, r, S, combos);
  orc_permutation(k0, k1, S, order);
  for (int64_t s = 0; s < S; s++) memcpy(assign + s * r, combos + order[s] * r, sizeof(int32_t) * r);
  int64_t base = payload_len / S, rem = payload_len % S, start = 0;
  for (int64_t s = 0; s < S; s++) {
    bounds[s] = start;
    start += base + (s < rem ? 1 : 0);
  }
  bounds[S] = start;
  free(combos);
  free(order);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* reduction order of ndarray.mean                                           */
/* ------------------------------------------------------------------------ */

/* numpy DOUBLE_pairwise_sum over a contiguous vector (width-1 shards). */
static double orc_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int k = 0; k < 8; k++) r[k] = a[k];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_pairwise(a, n2) + orc_pairwise(a + n2, n - n2);
  }
}

uint16_t orc_f32_to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static float orc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* Element value of miner replica m at e, as the fp64 the reference reduces. */
#define ORC_F32 0
#define ORC_BF16 1
#define ORC_F64WIRE 2
static double orc_load(const void* rep, int dtype, int64_t e) {
  if (dtype == ORC_F32) return (double)((const float*)rep)[e];
  if (dtype == ORC_BF16) return (double)orc_bf16_to_f32(((const uint16_t*)rep)[e]);
  return (double)(float)((const double*)rep)[e]; /* payload.astype("<f4") */
}

/* ------------------------------------------------------------------------ */
/* corruption descriptors and agreement                                      */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t kind;
  int32_t pad;
  double a;
  uint64_t key0, key1;
} orc_corruption;

#define ORC_NONE 0
#define ORC_ADD 1
#define ORC_SCALE 2
#define ORC_NOISE 3
#define ORC_NOISE_ADD 4

static double orc_noise(const orc_corruption* c, int64_t e) {
  uint64_t ctr[4] = {(uint64_t)(e / 4) + 1, 0, 0, 0}, out[4];
  orc_philox_rounds(ctr, c->key0, c->key1, out);
  uint64_t bits = out[e % 4];
  double unit = (double)(bits >> 11) * (1.0 / 4503599627370496.0) - 1.0;
  return c->a * unit;
}

static double orc_corrupt(const orc_corruption* c, double mean, int64_t e) {
  switch (c ? c->kind : ORC_NONE) {
    case ORC_ADD: return mean + c->a;
    case ORC_SCALE: return mean * c->a;
    case ORC_NOISE: return orc_noise(c, e);
    case ORC_NOISE_ADD: return mean + orc_noise(c, e);
    default: return mean;
  }
}

/* agreement (butterfly.py:117-133) on two fp64 vectors; dot products are
 * sequential here (the reference uses BLAS ddot: entries agree to ~1e-15). */
double orc_agreement(const double* a, const double* b, int64_t n, double tol) {
  double mx = 0.0;
  int nan = 0;
  for (int64_t i = 0; i < n; i++) {
    double d = fabs(a[i] - b[i]);
    if (d != d) nan = 1;
    else if (d > mx) mx = d;
  }
  if (!nan && mx <= tol) return 1.0;
  double aa = 0.0, bb = 0.0, ab = 0.0;
  for (int64_t i = 0; i < n; i++) {
    aa += a[i] * a[i];
    bb += b[i] * b[i];
    ab += a[i] * b[i];
  }
  double na = sqrt(aa), nb = sqrt(bb);
  if (na == 0.0 || nb == 0.0) return 0.0;
  double c = ab / (na * nb);
  if (c != c) return c;
  return c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
}

/* ------------------------------------------------------------------------ */
/* run_all_reduce                                                            */
/* ------------------------------------------------------------------------ */

/*
 * replicas[m]    : miner m's payload (dtype), all N miners (failed ones unread)
 * failed[m]      : 1 if miner m is in `failures`
 * corr[m]        : descriptor (NULL = all honest)
 * fallback       : fp64[P] or NULL
 * merged (out)   : fp64[P]
 * status (out)   : [S] 0 merged, 1 lost, 2 disagreement
 * entries (out)  : [N*N], NaN-initialised here
 * flagged (out)  : [N]
 * source (out)   : [S] adopted assignee or -1 (may be NULL)
 * Returns 0.
 */
int orc_merge(int n, int r, int64_t P, int64_t S, const int32_t* assign, const int64_t* bounds,
              int dtype, const void* const* replicas, const uint8_t* failed,
              const orc_corruption* corr, const double* fallback, double tol, double* merged,
              uint8_t* status, double* entries, uint8_t* flagged, int32_t* source, int nthreads) {
  int32_t* alive = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int n_alive = 0;
  for (int m = 0; m < n; m++)
    if (!failed || !failed[m]) alive[n_alive++] = m;
  const int npairs = r * (r - 1) / 2;
  double* scores = (double*)malloc(sizeof(double) * (size_t)(S * npairs + 1));
  uint8_t* has_score = (uint8_t*)calloc((size_t)(S * npairs + 1), 1);
  uint8_t* shard_flags = (uint8_t*)calloc((size_t)(S * r + 1), 1);
  for (int64_t i = 0; i < (int64_t)n * n; i++) entries[i] = NAN;
  memset(flagged, 0, (size_t)n);

#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < S; s++) {
    const int64_t lo = bounds[s], hi = bounds[s + 1], len = hi - lo;
    const int32_t* mem = assign + s * r;
    int surv[16], ns = 0;
    for (int k = 0; k < r; k++)
      if (!failed || !failed[mem[k]]) surv[ns++] = k; /* slot indices */
    int src_slot = -1;
    if (ns > 0 && n_alive > 0) {
      double* mean = (double*)malloc(sizeof(double) * (size_t)len);
      double* tmp = (double*)malloc(sizeof(double) * (size_t)(n_alive > 0 ? n_alive : 1));
      for (int64_t e = lo; e < hi; e++) {
        double acc;
        if (dtype == ORC_BF16) { /* extension: fp32 accumulation */
          float f = 0.0f;
          for (int q = 0; q < n_alive; q++) f = f + (float)orc_load(replicas[alive[q]], dtype, e);
          mean[e - lo] = (double)(f / (float)n_alive);
          continue;
        }
        if (len == 1) {
          for (int q = 0; q < n_alive; q++) tmp[q] = orc_load(replicas[alive[q]], dtype, e);
          acc = 0.0 + orc_pairwise(tmp, n_alive);
        } else {
          acc = 0.0;
          for (int q = 0; q < n_alive; q++) acc += orc_load(replicas[alive[q]], dtype, e);
        }
        mean[e - lo] = acc / (double)n_alive;
      }
      /* copies of each surviving assignee */
      double* copies = (double*)malloc(sizeof(double) * (size_t)(len * ns));
      for (int q = 0; q < ns; q++) {
        const orc_corruption* c = corr ? &corr[mem[surv[q]]] : NULL;
        for (int64_t e = lo; e < hi; e++) copies[q * len + (e - lo)] = orc_corrupt(c, mean[e - lo], e);
      }
      /* pairwise agreement among survivors (r = 2: the single pair) */
      int agree_cnt[16] = {0};
      uint8_t agree[16][16];
      memset(agree, 0, sizeof agree);
      for (int p = 0; p < ns; p++)
        for (int q = p + 1; q < ns; q++) {
          double sc = orc_agreement(copies + p * len, copies + q * len, len, tol);
          int a = surv[p], b = surv[q];
          int pair = 0; /* index of slot pair (a,b) among r*(r-1)/2 */
          for (int x = 0; x < a; x++) pair += r - 1 - x;
          pair += b - a - 1;
          scores[s * npairs + pair] = sc;
          has_score[s * npairs + pair] = 1;
          if (sc == 1.0) {
            agree[p][q] = agree[q][p] = 1;
            agree_cnt[p]++;
            agree_cnt[q]++;
          }
        }
      /* adopt: the lowest survivor backed by a strict majority of survivors
       * (r = 2: both survivors agree, or a single survivor) */
      int src_q = -1;
      for (int q = 0; q < ns; q++)
        if (2 * (agree_cnt[q] + 1) > ns) {
          src_q = q;
          break;
        }
      if (src_q >= 0) {
        src_slot = surv[src_q];
        memcpy(merged + lo, copies + src_q * len, sizeof(double) * (size_t)len);
        status[s] = 0;
        for (int q = 0; q < ns; q++)
          if (q != src_q && !agree[src_q][q]) shard_flags[s * r + surv[q]] = 1;
      } else {
        status[s] = (uint8_t)(ns >= 2 ? 2 : 1);
        if (ns >= 2)
          for (int q = 0; q < ns; q++) shard_flags[s * r + surv[q]] = 1;
      }
      free(copies);
      free(mean);
      free(tmp);
    } else {
      status[s] = 1; /* lost */
    }
    if (src_slot < 0) {
      for (int64_t e = lo; e < hi; e++) {
        if (fallback) merged[e] = fallback[e];
        else if (n_alive > 0 && dtype == ORC_F64WIRE) /* raw fp64 payload (butterfly.py:271) */
          merged[e] = ((const double*)replicas[alive[0]])[e];
        else if (n_alive > 0) merged[e] = orc_load(replicas[alive[0]], dtype, e);
        else merged[e] = NAN;
      }
    }
    if (source) source[s] = src_slot < 0 ? -1 : mem[src_slot];
  }
  /* entries: min over the shards a pair shares (r = 2: exactly one), NaN if
   * any of them scored NaN — order independent; then the flags */
  uint8_t* poisoned = (uint8_t*)calloc((size_t)n * n + 1, 1);
  for (int64_t s = 0; s < S; s++) {
    const int32_t* mem = assign + s * r;
    int pair = 0;
    for (int a = 0; a < r; a++)
      for (int b = a + 1; b < r; b++, pair++) {
        if (!has_score[s * npairs + pair]) continue;
        double sc = scores[s * npairs + pair];
        int64_t ij = (int64_t)mem[a] * n + mem[b], ji = (int64_t)mem[b] * n + mem[a];
        if (poisoned[ij]) continue;
        if (sc != sc) {
          poisoned[ij] = 1;
          entries[ij] = entries[ji] = sc;
        } else if (entries[ij] != entries[ij] || sc < entries[ij]) {
          entries[ij] = entries[ji] = sc;
        }
      }
    for (int k = 0; k < r; k++)
      if (shard_flags[s * r + k]) flagged[mem[k]] = 1;
  }
  free(poisoned);
  free(alive);
  free(scores);
  free(has_score);
  free(shard_flags);
  return 0;
}
