// bfly_validate.cu — the validator's replay checks: the same
// reduction pattern as the merge's agreement, over a batch of (recomputed, reported)
// activation pairs.
//
// Per pair (validator.py:148-167, cosine_similarity :33-46):
//   cos  = a.b / (|a| |b|)  (both zero -> 1, one zero -> 0; norms = sqrt(x.x))
//   sim  = cos, then 0 if cos < cosine_threshold, or |a| > 0 and |b|/|a| is outside
//          [magnitude_low, magnitude_high], or max |a - b| / max(|a|, 1) > max_rel_deviation
// One CTA per pair, fixed-order block trees (no floating-point atomics): reruns are
// byte-identical; against the reference's BLAS ddot the sums agree to rounding.
#include <cuda_runtime.h>
#include <math.h>

#include "bfly_internal.cuh"

namespace bfly {

namespace {

constexpr int kVThreads = 256;

struct CheckStat {
  double ab, aa, bb, dev;
};

__device__ __forceinline__ double max_nan2(double a, double b) {
  return (isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b);
}

__device__ __forceinline__ CheckStat combine(CheckStat x, CheckStat y) {
  return CheckStat{__dadd_rn(x.ab, y.ab), __dadd_rn(x.aa, y.aa), __dadd_rn(x.bb, y.bb), max_nan2(x.dev, y.dev)};
}

__global__ void __launch_bounds__(kVThreads) k_replay_check(const double* __restrict__ rec,
                                                            const double* __restrict__ rep,
                                                            const int64_t* __restrict__ offsets, double thr,
                                                            double lo, double hi, double max_rel, double* sim_out,
                                                            double* cos_out) {
  const int64_t b0 = offsets[blockIdx.x], b1 = offsets[blockIdx.x + 1];
  CheckStat st{0.0, 0.0, 0.0, 0.0};
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kVThreads) {
    const double a = rec[i], b = rep[i];
    st.ab = fma(a, b, st.ab);
    st.aa = fma(a, a, st.aa);
    st.bb = fma(b, b, st.bb);
    st.dev = max_nan2(st.dev, __ddiv_rn(fabs(__dsub_rn(a, b)), fmax(fabs(a), 1.0)));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    CheckStat o;
    o.ab = __shfl_xor_sync(0xffffffffu, st.ab, off);
    o.aa = __shfl_xor_sync(0xffffffffu, st.aa, off);
    o.bb = __shfl_xor_sync(0xffffffffu, st.bb, off);
    o.dev = __shfl_xor_sync(0xffffffffu, st.dev, off);
    st = combine(st, o);
  }
  __shared__ CheckStat part[kVThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = st;
  __syncthreads();
  if (threadIdx.x != 0) return;
  st = part[0];
  for (int w = 1; w < kVThreads / 32; ++w) st = combine(st, part[w]);
  const double na = sqrt(st.aa), nb = sqrt(st.bb);
  double cos;
  if (na == 0.0 && nb == 0.0) cos = 1.0;
  else if (na == 0.0 || nb == 0.0) cos = 0.0;
  else cos = __ddiv_rn(st.ab, __dmul_rn(na, nb));
  double sim = cos;
  if (cos < thr) sim = 0.0;  // NaN compares false, as in numpy
  if (sim != 0.0 && na > 0.0) {
    const double ratio = __ddiv_rn(nb, na);
    if (!(lo <= ratio && ratio <= hi)) sim = 0.0;
  }
  if (sim != 0.0 && st.dev > max_rel) sim = 0.0;  // NaN deviation passes, as np.max(...) > x does
  sim_out[blockIdx.x] = sim;
  if (cos_out) cos_out[blockIdx.x] = cos;
}

}  // namespace
}  // namespace bfly

using namespace bfly;

extern "C" int bfly_replay_check(const double* d_rec, const double* d_rep, const int64_t* d_offsets,
                                 int32_t n_pairs, const double* h_policy, double* d_sim, double* d_cos,
                                 void* stream) {
  if (n_pairs < 0 || (n_pairs > 0 && (!d_rec || !d_rep || !d_offsets || !d_sim)) || !h_policy)
    return fail(BFLY_E_INVALID_ARG, "bad replay-check arguments");
  if (n_pairs == 0) return BFLY_OK;
  k_replay_check<<<(unsigned)n_pairs, kVThreads, 0, (cudaStream_t)stream>>>(
      d_rec, d_rep, d_offsets, h_policy[0], h_policy[1], h_policy[2], h_policy[3], d_sim, d_cos);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_replay_check launch");
  return BFLY_OK;
}
