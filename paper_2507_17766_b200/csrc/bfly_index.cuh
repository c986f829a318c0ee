// bfly_index.cuh — the shard index map, shared by host and device code.
//
// Restates, for plan_shards (butterfly.py:84-114):
//   * numpy's Philox4x64-10 bit generator (simkernel.py:219 constructs it with
//     the SHA-256 key; numpy keeps a 4-word output buffer, pre-increments the
//     256-bit counter, and hands out 32-bit draws low half first);
//   * Generator.permutation(n) (simkernel.py:237-238): Fisher-Yates from
//     i = n-1 down to 1 with j = random_interval(i), masked rejection;
//   * lexicographic r-combinations (enumerate_pairs, butterfly.py:76-81) and
//     their unranking, so assignment[s] = combos[perm[s]] (butterfly.py:100);
//   * near-equal bounds, remainder to the first shards (butterfly.py:101-107).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BFLY_HD __host__ __device__ __forceinline__
#else
#define BFLY_HD inline
#endif

namespace bfly {

struct Philox4x64 {
  uint64_t v[4];
};

BFLY_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

// Ten Philox4x64 rounds; the key is bumped by the Weyl constants before every
// round after the first.
BFLY_HD Philox4x64 philox4x64_10(Philox4x64 c, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round) {
#if defined(__CUDA_ARCH__)
      // opaque adds: the round keys are recomputed in every call instead of being hoisted
      // out of the caller's element loop as 40 loop-invariant registers per key (which
      // halved k_stats' occupancy, or spilled under a register cap)
      asm volatile("add.u64 %0, %0, %1;" : "+l"(k0) : "l"(0x9E3779B97F4A7C15ULL));
      asm volatile("add.u64 %0, %0, %1;" : "+l"(k1) : "l"(0xBB67AE8584CAA73BULL));
#else
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
#endif
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c.v[0], &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c.v[2], &hi1, &lo1);
    Philox4x64 n;
    n.v[0] = hi1 ^ c.v[1] ^ k0;
    n.v[1] = lo1;
    n.v[2] = hi0 ^ c.v[3] ^ k1;
    n.v[3] = lo0;
    c = n;
  }
  return c;
}

// 64-bit output number `idx` (0-based) of a freshly keyed numpy Philox: the
// first block is generated at counter 1.  Counter-based, so any word can be
// computed independently — used to fill draw buffers in parallel.
BFLY_HD uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t idx) {
  Philox4x64 c;
  c.v[0] = (idx >> 2) + 1;
  c.v[1] = ((idx >> 2) + 1 == 0) ? 1 : 0;  // carry (only for idx near 2^66)
  c.v[2] = 0;
  c.v[3] = 0;
  Philox4x64 o = philox4x64_10(c, k0, k1);
  switch (idx & 3) {
    case 0: return o.v[0];
    case 1: return o.v[1];
    case 2: return o.v[2];
    default: return o.v[3];
  }
}

// Sequential stream with numpy's buffering semantics (next_uint64 / next_uint32).
struct PhiloxStream {
  uint64_t k0, k1;
  uint64_t ctr0, ctr1, ctr2, ctr3;
  uint64_t buf[4];
  int pos;
  int has32;
  uint32_t saved32;

  BFLY_HD void init(uint64_t key0, uint64_t key1) {
    k0 = key0;
    k1 = key1;
    ctr0 = ctr1 = ctr2 = ctr3 = 0;
    pos = 4;
    has32 = 0;
    saved32 = 0;
  }
  BFLY_HD uint64_t next64() {
    if (pos < 4) return buf[pos++];
    if (++ctr0 == 0)
      if (++ctr1 == 0)
        if (++ctr2 == 0) ++ctr3;
    Philox4x64 c;
    c.v[0] = ctr0;
    c.v[1] = ctr1;
    c.v[2] = ctr2;
    c.v[3] = ctr3;
    Philox4x64 o = philox4x64_10(c, k0, k1);
    buf[0] = o.v[0];
    buf[1] = o.v[1];
    buf[2] = o.v[2];
    buf[3] = o.v[3];
    pos = 1;
    return buf[0];
  }
  BFLY_HD uint32_t next32() {
    if (has32) {
      has32 = 0;
      return saved32;
    }
    uint64_t v = next64();
    has32 = 1;
    saved32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffULL);
  }
};

BFLY_HD uint64_t smear_mask(uint64_t m) {
  m |= m >> 1;
  m |= m >> 2;
  m |= m >> 4;
  m |= m >> 8;
  m |= m >> 16;
  m |= m >> 32;
  return m;
}

// numpy random_interval(max): uniform integer in [0, max] by masked rejection.
template <class Stream>
BFLY_HD uint64_t random_interval(Stream& s, uint64_t max) {
  if (max == 0) return 0;
  const uint64_t mask = smear_mask(max);
  uint64_t v;
  if (max <= 0xffffffffULL) {
    do {
      v = (uint64_t)(s.next32() & (uint32_t)mask);
    } while (v > max);
  } else {
    do {
      v = s.next64() & mask;
    } while (v > max);
  }
  return v;
}

// Binomial coefficient with a saturating guard (returns -1 on overflow).
BFLY_HD int64_t binom(int64_t n, int64_t k) {
  if (k < 0 || n < 0 || k > n) return 0;
  if (k > n - k) k = n - k;
  int64_t r = 1;
  for (int64_t i = 1; i <= k; ++i) {
    // r * (n - k + i) / i is exact at every step
    const int64_t num = n - k + i;
    if (r > (int64_t)0x7fffffffffffffffLL / num) return -1;
    r = r * num / i;
  }
  return r;
}

// Members (ascending) of the lexicographic rank-`rank` r-combination of
// {0..n-1}; enumerate_pairs' order for r = 2 (butterfly.py:80).
BFLY_HD void unrank_combination(int32_t n, int32_t r, int64_t rank, int32_t* out) {
  int32_t x = 0;
  for (int32_t slot = 0; slot < r; ++slot) {
    for (;; ++x) {
      const int64_t c = binom(n - 1 - x, r - 1 - slot);  // combos starting with x
      if (rank < c) break;
      rank -= c;
    }
    out[slot] = x++;
  }
}

// Inverse of unrank_combination for ascending members.
BFLY_HD int64_t rank_combination(int32_t n, int32_t r, const int32_t* members) {
  int64_t rank = 0;
  int32_t x = 0;
  for (int32_t slot = 0; slot < r; ++slot) {
    for (; x < members[slot]; ++x) rank += binom(n - 1 - x, r - 1 - slot);
    ++x;
  }
  return rank;
}

// Closed-form shard bounds: divmod(P, S), first `rem` shards one longer.
struct Bounds {
  int64_t P, S, base, rem;
  BFLY_HD void init(int64_t p, int64_t s) {
    P = p;
    S = s;
    base = p / s;
    rem = p % s;
  }
  BFLY_HD int64_t start(int64_t s) const { return s * base + (s < rem ? s : rem); }
  BFLY_HD int64_t len(int64_t s) const { return base + (s < rem ? 1 : 0); }
  BFLY_HD int64_t shard_of(int64_t e) const {
    const int64_t big = rem * (base + 1);
    return e < big ? e / (base + 1) : rem + (e - big) / base;
  }
};

// The same with shard_of from fp64 reciprocals instead of a 64-bit integer division
// (~70 instructions on the GPU): k_reduce's adversarial round measured 4% faster
// (tools/_ab1.sh).  For n < 2^51 the estimate is off by at most one; the check fixes it.
struct FastBounds : Bounds {
  double inv_long, inv_base;  // 1 / (base + 1), 1 / base
  BFLY_HD void init(int64_t p, int64_t s) {
    Bounds::init(p, s);
    inv_long = 1.0 / (double)(base + 1);
    inv_base = base > 0 ? 1.0 / (double)base : 0.0;
  }
  BFLY_HD static int64_t div_floor(int64_t n, int64_t d, double inv) {
    int64_t q = (int64_t)((double)n * inv);
    if (q * d > n)
      --q;
    else if ((q + 1) * d <= n)
      ++q;
    return q;
  }
  BFLY_HD int64_t shard_of(int64_t e) const {
    const int64_t big = rem * (base + 1);
    return e < big ? div_floor(e, base + 1, inv_long) : rem + div_floor(e - big, base, inv_base);
  }
};

// The shard of increasing element positions without a 64-bit division per lookup (one
// costs ~70 instructions on the GPU): a thread walking its tiles in ascending order keeps
// the current shard and steps forward; only the first lookup (or a step back) divides.
struct ShardCursor {
  int64_t s = -1, lo = 0, hi = 0;  // current shard and its element range [lo, hi)
  BFLY_HD int64_t at(const Bounds& b, int64_t e) {
    if (s < 0 || e < lo) {
      s = b.shard_of(e);
      lo = b.start(s);
      hi = lo + b.len(s);
      return s;
    }
    while (e >= hi) {
      ++s;
      lo = hi;
      hi = lo + b.len(s);
    }
    return s;
  }
};

// Uniform noise word -> (2u - 1) in [-1, 1) with 52-bit resolution, exact.
BFLY_HD double noise_unit(uint64_t bits) {
  return (double)(bits >> 11) * (1.0 / 4503599627370496.0) - 1.0;  // * 2^-52, then -1: both exact
}

}  // namespace bfly
