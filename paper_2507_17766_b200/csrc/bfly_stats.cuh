// bfly_stats.cuh — pair statistics of redundant shard copies (agreement, butterfly.py:117-133),
// shared by the single-GPU merge (bfly_merge.cu) and the persistent multi-GPU ring
// (bfly_ring.cu): per-thread partials, fixed-order combines, no floating-point atomics.
#pragma once
#include <math.h>

#include "bfly_internal.cuh"

namespace bfly {

__device__ __forceinline__ double nan64() { return __longlong_as_double(0x7ff8000000000000LL); }

__device__ __forceinline__ double max_nan(double a, double b) {
  return (isnan(a) || isnan(b)) ? nan64() : fmax(a, b);
}

struct PairStat {
  double mx, ab, aa, bb;
};

// One thread's running pair statistics: max|x - y| over the differences that are not
// NaN plus a NaN flag (finish() makes the max NaN if any difference was: max_nan over
// every element, in fewer instructions than a NaN-propagating max per element), and the
// three dot products by fma in element order.
struct PairAcc {
  double mx = 0.0, ab = 0.0, aa = 0.0, bb = 0.0;
  bool nan = false;
  __device__ __forceinline__ void add(double x, double y) {
    const double d = fabs(__dsub_rn(x, y));
    mx = d > mx ? d : mx;  // d >= +0: no signed-zero cases
    nan |= d != d;
    ab = fma(x, y, ab);
    aa = fma(x, x, aa);
    bb = fma(y, y, bb);
  }
  __device__ __forceinline__ PairStat finish() const { return PairStat{nan ? nan64() : mx, ab, aa, bb}; }
};

__device__ __forceinline__ PairStat warp_combine(PairStat s) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    s.mx = max_nan(s.mx, __shfl_xor_sync(0xffffffffu, s.mx, off));
    s.ab = __dadd_rn(s.ab, __shfl_xor_sync(0xffffffffu, s.ab, off));
    s.aa = __dadd_rn(s.aa, __shfl_xor_sync(0xffffffffu, s.aa, off));
    s.bb = __dadd_rn(s.bb, __shfl_xor_sync(0xffffffffu, s.bb, off));
  }
  return s;
}

// Copies of four consecutive elements e0..e0+3 (e0 % 4 == 0) of a device-computable
// corruption: one Philox4x64 block of noise words.
__device__ __forceinline__ void corrupt4(const bfly_corruption_t& c, const double* m, int64_t e0, double* out) {
  switch (c.kind) {
    case BFLY_CORR_ADD:
#pragma unroll
      for (int i = 0; i < 4; ++i) out[i] = __dadd_rn(m[i], c.a);
      return;
    case BFLY_CORR_SCALE:
#pragma unroll
      for (int i = 0; i < 4; ++i) out[i] = __dmul_rn(m[i], c.a);
      return;
    case BFLY_CORR_NOISE:
    case BFLY_CORR_NOISE_ADD: {
      Philox4x64 ctr;
      ctr.v[0] = (uint64_t)(e0 >> 2) + 1;
      ctr.v[1] = ctr.v[2] = ctr.v[3] = 0;
      const Philox4x64 o = philox4x64_10(ctr, c.key0, c.key1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double noise = __dmul_rn(c.a, noise_unit(o.v[j]));
        out[j] = c.kind == BFLY_CORR_NOISE ? noise : __dadd_rn(m[j], noise);
      }
      return;
    }
    default:
#pragma unroll
      for (int i = 0; i < 4; ++i) out[i] = m[i];
  }
}

}  // namespace bfly
