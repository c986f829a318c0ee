// bfly_merge.cu — one butterfly merge round on the device (run_all_reduce,
// butterfly.py:161-295), for r = 2 (reference) and r = 3 (extension).
//
// Kernels, in launch order (all on the caller's stream, no host sync):
//   k_fill_nan      entries[N*N] = NaN                         (butterfly.py:243)
//   k_classify      per shard: survivors, class fast/special/lost, status and
//                   entry 1.0 for all-honest shards               (:219-224,:248-263)
//   k_reduce  ★     the HBM stream: per element, fp64 sequential mean over the
//                   alive replicas in ascending miner order (numpy's order,
//                   :225-231,:156-158), scatter-back in place into every miner
//                   replica for fast shards, fp64 merged / workspace otherwise
//   k_stats         special shards: per-assignee copies (corruption descriptors
//                   or host-supplied copies, :232-233), per chunk max|a-b|, a.b,
//                   a.a, b.b for every surviving assignee pair     (:117-133)
//   k_decide        one warp per special shard: fixed-order combine, agreement
//                   score, adopt / disagreement / flags            (:248-273)
//   k_entries3      r = 3 only: entry = min over the shards a pair shares
//   k_apply         special + lost shards: adopted copy or fallback into the
//                   merged vector and every replica               (:259-273)
//
// Determinism: no floating-point atomics; every reduction has a fixed order.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "bfly_internal.cuh"
#include "bfly_elem.cuh"
#include "bfly_stats.cuh"

namespace bfly {

// ---------------------------------------------------------------------------
// parameters
// ---------------------------------------------------------------------------

struct Params {
  int32_t n, r, n_alive, n_dst, npairs;
  int64_t P, S, cps;
  FastBounds bnd;
  const int32_t* assign;
  const void* const* src;
  const uint8_t* failed;
  const bfly_corruption_t* corr;
  void* const* dst;
  const double* fallback;
  double* merged;
  double* ws;  // means of special shards (aliases merged when no separate workspace)
  const double* host_copies;
  uint8_t* status;
  double* entries;
  uint8_t* flagged;
  int32_t* source;
  uint8_t* cls;
  uint8_t* pred;  // ShardPred per shard
  uint8_t* done;  // per statistics tile: partial already written by k_reduce
  int64_t stile;  // statistics tile = one k_reduce tile (kThreads vectors)
  double* stats;
  double* scores;
  uint8_t* has_score;
  int32_t* inv;
  double tol;
  const double* acc_in;  // chain accumulator for [ebeg, eend) (multi-GPU), or null
  int32_t n_div;         // divisor of the mean: all alive miners across GPUs
  int64_t ebeg, eend;    // element range of this REDUCE call
  const void* fb_src;    // replica supplying fallback values (the lowest alive miner's)
  int64_t sbeg, send;    // shard range of this FINISH call
  const int32_t* slist;  // or this shard list
  int32_t n_fin;         // shards of this FINISH call
  bool fb_gone;          // the fallback replica was overwritten before FINISH (multi-GPU)
  uint8_t* nonfin;       // [S] fast shard whose mean is not finite somewhere (k_reduce)
  uint32_t* nonfin_any;  // any of them
  uint32_t* special_any; // some shard is special or lost (k_classify): FINISH has work
  uint32_t* apply_any;   // some shard's final values differ from what k_reduce wrote (k_apply)
};

// A fast shard whose mean is NaN or +-Inf somewhere: its (identical) copies score NaN
// in the reference's agreement (max|a-b| = NaN, butterfly.py:127-133), so with two or
// more survivors the shard is a disagreement (:255,264-267).  k_reduce only marks it;
// k_nonfinite decides it.
// (k_reduce inlines these; k_ring keeps its marking out of line, bfly_ring.cu)
__device__ __forceinline__ void mark_nonfinite_shard(uint8_t* nonfin, uint32_t* any, int64_t s) {
  nonfin[s] = 1;
  *any = 1u;
}
__device__ __forceinline__ void mark_nonfinite_elem(uint8_t* nonfin, uint32_t* any, Bounds bnd, int64_t e) {
  nonfin[bnd.shard_of(e)] = 1;
  *any = 1u;
}
__device__ __forceinline__ void mark_nonfinite(const Params& p, int64_t s) { mark_nonfinite_shard(p.nonfin, p.nonfin_any, s); }
__device__ __forceinline__ void mark_nonfinite_at(const Params& p, int64_t e) {
  mark_nonfinite_elem(p.nonfin, p.nonfin_any, p.bnd, e);
}

__device__ __forceinline__ int64_t fin_shard(const Params& p, unsigned i) {
  return p.slist ? (int64_t)p.slist[i] : p.sbeg + i;
}

// numpy DOUBLE_pairwise_sum over the alive replicas at element e (width-1 shards).
template <class D>
__device__ double pairwise_alive(const void* const* src, int lo, int n, int64_t e) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, D::load(src[lo + i], e));
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = D::load(src[lo + k], e);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], D::load(src[lo + i + k], e));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, D::load(src[lo + i], e));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_alive<D>(src, lo, n2, e), pairwise_alive<D>(src, lo + n2, n - n2, e));
}

template <class D>
__device__ __forceinline__ typename D::Acc mean_at(const void* const* src, int n_alive, int64_t e,
                                                   bool width1) {
  if constexpr (sizeof(typename D::Acc) == 8) {
    if (width1) return D::mean(__dadd_rn(0.0, pairwise_alive<D>(src, 0, n_alive, e)), n_alive);
  }
  typename D::Acc acc = D::zero();
  for (int q = 0; q < n_alive; ++q) acc = D::add(acc, D::load(src[q], e));
  return D::mean(acc, n_alive);
}

// ---------------------------------------------------------------------------
// k_fill_nan / k_classify
// ---------------------------------------------------------------------------

__global__ void k_fill_nan(double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = nan64();
}

__device__ __forceinline__ int pair_index(int r, int a, int b) {  // slot pair (a<b) -> 0..npairs-1
  int idx = 0;
  for (int x = 0; x < a; ++x) idx += r - 1 - x;
  return idx + (b - a - 1);
}

// Does k_apply have to rewrite shard s?  Not when k_reduce already wrote its final
// values: the predicted fallback was adopted, or the predicted (honest) mean — except
// that a special shard falling back must still put the fallback into merged when merged
// doubles as the workspace of the means.  (source / pred as decided / predicted.)
__device__ __forceinline__ bool apply_needed(const Params& p, int64_t s) {
  const int32_t src_m = p.source[s];
  const uint8_t pr = p.pred[s] & kPredMask;
  const bool as_predicted =
      src_m < 0 ? pr == kPredFallback : (pr == kPredMean && p.corr[src_m].kind == BFLY_CORR_NONE);
  return !as_predicted || (src_m < 0 && p.cls[s] == kSpecial && p.merged && p.merged == p.ws);
}

__global__ void k_classify(Params p) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  const int32_t* mem = p.assign + s * p.r;
  int ns = 0, first = -1;
  bool corrupted = false;
  for (int k = 0; k < p.r; ++k) {
    const int m = mem[k];
    if (p.failed[m]) continue;
    if (first < 0) first = m;
    ++ns;
    if (p.corr[m].kind != BFLY_CORR_NONE) corrupted = true;
  }
  if (p.inv) p.inv[rank_combination(p.n, p.r, mem)] = (int32_t)s;
  uint8_t c;
  if (ns == 0 || p.n_div == 0) {
    c = kLost;
    p.status[s] = BFLY_LOST;
    p.source[s] = -1;
  } else if (corrupted) {
    c = kSpecial;
  } else {
    c = kFast;
    if (p.r > 2)
      for (int q = 0; q < p.npairs; ++q) p.has_score[s * p.npairs + q] = 0;
    p.status[s] = BFLY_MERGED;
    p.source[s] = first;
    // every surviving pair agrees exactly (identical reductions, max|a-b| = 0)
    for (int a = 0; a < p.r; ++a)
      for (int b = a + 1; b < p.r; ++b) {
        const int i = mem[a], j = mem[b];
        if (p.failed[i] || p.failed[j]) continue;
        if (p.r == 2) {
          p.entries[(int64_t)i * p.n + j] = 1.0;
          p.entries[(int64_t)j * p.n + i] = 1.0;
        } else {
          p.scores[s * p.npairs + pair_index(p.r, a, b)] = 1.0;
          p.has_score[s * p.npairs + pair_index(p.r, a, b)] = 1;
        }
      }
  }
  if (c != kFast && p.r > 2)
    for (int q = 0; q < p.npairs; ++q) p.has_score[s * p.npairs + q] = 0;
  if (c != kFast && *(volatile uint32_t*)p.special_any == 0u) atomicOr(p.special_any, 1u);
  p.cls[s] = c;
  // predicted outcome (k_reduce writes it, k_apply revisits the rest); only when
  // k_reduce runs, and a predicted mean only when the fallback source is not one
  // of the replicas the mean overwrites in place
  uint8_t pr = kPredNone;
  if (p.n_alive > 0 || p.acc_in) {
    if (c == kLost) {
      pr = kPredFallback;
    } else if (c == kSpecial) {
      int nh = 0;
      for (int k = 0; k < p.r; ++k) nh += !p.failed[mem[k]] && p.corr[mem[k]].kind == BFLY_CORR_NONE;
      if (2 * nh > ns) {
        const void* fb_raw = p.fb_src ? p.fb_src : (p.n_alive > 0 ? p.src[0] : nullptr);
        bool safe = p.fallback != nullptr || fb_raw == nullptr;
        if (!safe) {
          safe = true;
          for (int d = 0; d < p.n_dst; ++d) safe = safe && p.dst[d] != fb_raw;
        }
        if (safe) pr = kPredMean;
      } else if (ns >= 2) {
        pr = kPredFallback;
      }
    }
  }
  if (c == kSpecial && p.r == 2 && ns == 2 && p.corr[mem[0]].kind != BFLY_CORR_HOST &&
      p.corr[mem[1]].kind != BFLY_CORR_HOST)
    pr |= kPredFuse;
  p.pred[s] = pr;
  if (c == kLost && apply_needed(p, s)) atomicOr(p.apply_any, 1u);  // nothing reduced: k_apply fills it
}

// fallback value of element e: the caller's fp64 fallback, else the lowest alive
// miner's upload (butterfly.py:264-273), else NaN
template <class D>
__device__ __forceinline__ double fallback_at(const Params& p, const void* fb_raw, int64_t e) {
  if (p.fallback) return p.fallback[e];
  if (fb_raw) return D::raw(fb_raw, e);
  return __longlong_as_double(0x7ff8000000000000LL);
}

// the same for the K elements of 32-byte vector vidx (pointers 32-byte aligned)
template <class D>
__device__ __forceinline__ void fallback_vec(const Params& p, const void* fb_raw, int64_t vidx, double* v) {
  constexpr int K = D::K;
  if (p.fallback) {
#pragma unroll
    for (int k = 0; k < K; k += 4)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v[k]), "=d"(v[k + 1]), "=d"(v[k + 2]), "=d"(v[k + 3])
                   : "l"(p.fallback + vidx * K + k));
  } else if (fb_raw) {
    V8 raw;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(raw.w[0]), "=r"(raw.w[1]), "=r"(raw.w[2]), "=r"(raw.w[3]), "=r"(raw.w[4]),
                   "=r"(raw.w[5]), "=r"(raw.w[6]), "=r"(raw.w[7])
                 : "l"(reinterpret_cast<const V8*>(fb_raw) + vidx));
    D::unpack_raw(raw, v);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __longlong_as_double(0x7ff8000000000000LL);
  }
}

// ---------------------------------------------------------------------------
// corrupted copies and pair statistics (k_reduce's fused path, k_stats)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double corrupt_value(const bfly_corruption_t& c, double mean, int64_t e,
                                                const double* host_copies, int slot, int64_t P) {
  switch (c.kind) {
    case BFLY_CORR_ADD: return __dadd_rn(mean, c.a);
    case BFLY_CORR_SCALE: return __dmul_rn(mean, c.a);
    case BFLY_CORR_NOISE:
    case BFLY_CORR_NOISE_ADD: {
      const double noise = __dmul_rn(c.a, noise_unit(philox_word(c.key0, c.key1, (uint64_t)e)));
      return c.kind == BFLY_CORR_NOISE ? noise : __dadd_rn(mean, noise);
    }
    case BFLY_CORR_HOST: return host_copies[(int64_t)slot * P + e];
    default: return mean;
  }
}

// CTA-wide fixed-order combine; result valid in thread 0.
__device__ PairStat block_combine(PairStat s) {
  __shared__ PairStat part[kThreads / 32];
  s = warp_combine(s);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) part[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < kThreads / 32 ? part[lane] : PairStat{0.0, 0.0, 0.0, 0.0};
    s = warp_combine(s);
  }
  return s;
}

// The same combine through shared memory only (a fixed-order tree of barriers, no
// shuffles): for loops whose convergence the compiler cannot prove, where warp
// shuffles would be emulated collectively (WARPSYNC loops, extra live registers).
__device__ PairStat block_combine_smem(PairStat s) {
  __shared__ PairStat part[kThreads];
  __syncthreads();  // the previous combine's readers are done
  part[threadIdx.x] = s;
  __syncthreads();
#pragma unroll 1
  for (int w = kThreads / 2; w; w >>= 1) {
    if (threadIdx.x < w) {
      PairStat u = part[threadIdx.x];
      const PairStat v = part[threadIdx.x + w];
      u.mx = max_nan(u.mx, v.mx);
      u.ab = __dadd_rn(u.ab, v.ab);
      u.aa = __dadd_rn(u.aa, v.aa);
      u.bb = __dadd_rn(u.bb, v.bb);
      part[threadIdx.x] = u;
    }
    __syncthreads();
  }
  return part[0];
}

// agreement decision from combined statistics (butterfly.py:127-133)
__device__ __forceinline__ double score_of(const PairStat& s, double tol) {
  if (!isnan(s.mx) && s.mx <= tol) return 1.0;
  const double na = sqrt(s.aa), nb = sqrt(s.bb);
  if (na == 0.0 || nb == 0.0) return 0.0;
  const double c = __ddiv_rn(s.ab, __dmul_rn(na, nb));
  if (isnan(c)) return c;
  return c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
}

// Copies of eight consecutive elements e0..e0+7 (e0 % 8 == 0): one Philox4x64
// call yields four noise words, so a group needs two calls per noisy assignee.
__device__ __forceinline__ void corrupt8(const bfly_corruption_t& c, const double* m, int64_t e0, unsigned valid,
                                         const double* host_copies, int slot, int64_t P, double* out) {
  switch (c.kind) {
    case BFLY_CORR_ADD:
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = __dadd_rn(m[i], c.a);
      return;
    case BFLY_CORR_SCALE:
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = __dmul_rn(m[i], c.a);
      return;
    case BFLY_CORR_NOISE:
    case BFLY_CORR_NOISE_ADD: {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        Philox4x64 ctr;
        ctr.v[0] = (uint64_t)(e0 >> 2) + h + 1;  // word e lives in block e/4 (+1: numpy pre-increment)
        ctr.v[1] = ctr.v[2] = ctr.v[3] = 0;
        const Philox4x64 o = philox4x64_10(ctr, c.key0, c.key1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double noise = __dmul_rn(c.a, noise_unit(o.v[j]));
          out[4 * h + j] = c.kind == BFLY_CORR_NOISE ? noise : __dadd_rn(m[4 * h + j], noise);
        }
      }
      return;
    }
    case BFLY_CORR_HOST:
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = (valid >> i) & 1 ? host_copies[(int64_t)slot * P + e0 + i] : 0.0;
      return;
    default:
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = m[i];
  }
}

// ws[e0..e0+7]: one 64-byte vector when the group is whole, masked scalars otherwise
__device__ __forceinline__ unsigned load_group(const double* ws, int64_t e0, int64_t lo, int64_t hi, double* m) {
  unsigned valid = 0;
  if (e0 >= lo && e0 + 8 <= hi) {
    valid = 0xff;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(m[4 * h]), "=d"(m[4 * h + 1]), "=d"(m[4 * h + 2]), "=d"(m[4 * h + 3])
                   : "l"(ws + e0 + 4 * h));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool in = e0 + i >= lo && e0 + i < hi;
      m[i] = in ? ws[e0 + i] : 0.0;
      valid |= (unsigned)in << i;
    }
  }
  return valid;
}

// ws[e0..e0+3]: one 32-byte vector when the group is whole, masked scalars otherwise
__device__ __forceinline__ unsigned load_group4(const double* ws, int64_t e0, int64_t lo, int64_t hi, double* m) {
  if (e0 >= lo && e0 + 4 <= hi) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(m[0]), "=d"(m[1]), "=d"(m[2]), "=d"(m[3])
                 : "l"(ws + e0));
    return 0xf;
  }
  unsigned valid = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool in = e0 + i >= lo && e0 + i < hi;
    m[i] = in ? ws[e0 + i] : 0.0;
    valid |= (unsigned)in << i;
  }
  return valid;
}

// corrupt4 plus the caller-supplied copies of host callables (valid elements only)
__device__ __forceinline__ void corrupt4h(const bfly_corruption_t& c, const double* m, int64_t e0, unsigned valid,
                                          const double* host_copies, int slot, int64_t P, double* out) {
  if (c.kind == BFLY_CORR_HOST) {
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = (valid >> i) & 1 ? host_copies[(int64_t)slot * P + e0 + i] : 0.0;
    return;
  }
  corrupt4(c, m, e0, out);
}

// Statistics of one vector (K means at e0, e0 % 4 == 0) for the copy pair (ca, cb).
template <class D>
__device__ __forceinline__ PairStat pair_stats_vec(const typename D::Acc* acc, int64_t e0, const bfly_corruption_t& ca,
                                                   const bfly_corruption_t& cb) {
  PairAcc st;
#pragma unroll
  for (int h = 0; h < D::K / 4; ++h) {
    double m[4], x[4], y[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = D::widen(acc[4 * h + j]);
    corrupt4(ca, m, e0 + 4 * h, x);
    corrupt4(cb, m, e0 + 4 * h, y);
#pragma unroll
    for (int j = 0; j < 4; ++j) st.add(x[j], y[j]);
  }
  return st.finish();
}

// partial statistics of shard s over statistics tile t (slot = t + s, see ScratchLayout)
__device__ __forceinline__ double* stat_slot(const Params& p, int64_t s, int64_t t, int pi) {
  return p.stats + ((t + s) * p.npairs + pi) * 4;
}

// ---------------------------------------------------------------------------
// k_reduce — the streaming mean + scatter-back
// ---------------------------------------------------------------------------

// One element of a special / lost shard: the mean into the workspace (special), then
// the predicted final value into merged and the replicas.
template <class D>
__device__ __forceinline__ void emit_predicted(const Params& p, void* const* s_dst, const void* fb_raw,
                                               bool merged_apart, int64_t e, uint8_t c, uint8_t pr, double mean) {
  if (c == kSpecial) p.ws[e] = mean;
  if (pr == kPredMean) {
    if (merged_apart) p.merged[e] = mean;
    for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], e, mean);
  } else if (pr == kPredFallback) {
    const double v = fallback_at<D>(p, fb_raw, e);  // read before the in-place stores
    if (p.merged && (c == kLost || merged_apart)) p.merged[e] = v;
    for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], e, v);
  }
}

template <class D, int U = 4, int MINB = 1, bool NOU = false>
__global__ void __launch_bounds__(kThreads, MINB) k_reduce(Params p) {
  extern __shared__ __align__(16) const void* s_ptr[];  // [n_alive] src, then [n_dst] dst
  const void** s_src = s_ptr;
  void** s_dst = const_cast<void**>(s_ptr + p.n_alive);
  const void* fb_raw = p.fb_src ? p.fb_src : (p.n_alive > 0 ? p.src[0] : nullptr);
  const bool aligned = stage_pointers(s_src, s_dst, p.src, p.n_alive, p.dst, p.n_dst,
                                      (uintptr_t)p.merged | (uintptr_t)p.acc_in | (uintptr_t)p.ws |
                                          (uintptr_t)p.fallback | (uintptr_t)fb_raw);
  const bool merged_apart = p.merged && p.merged != p.ws;  // final values may go to merged early
  constexpr int K = D::K;
  constexpr int TILE = kThreads * K;
  using Acc = typename D::Acc;
  const bool may_width1 = p.bnd.base == 1;
  const int64_t tile_lo = p.ebeg / TILE, tile_hi = (p.eend + TILE - 1) / TILE;

  for (int64_t tile = tile_lo + blockIdx.x; tile < tile_hi; tile += gridDim.x) {
    const int64_t t0 = max(tile * TILE, p.ebeg);
    const int64_t t1 = min(tile * TILE + TILE, p.eend);
    // per tile: vector path unless a width-1 shard needs numpy's pairwise order;
    // all-fast tiles skip the per-vector class lookup.  (Measured: the fp64-reciprocal
    // lookups here beat a forward-walking ShardCursor by 1 ms on the adversarial round.)
    const int64_t s_lo = p.bnd.shard_of(t0), s_hi = p.bnd.shard_of(t1 - 1);
    bool vec = aligned && (t1 - t0 == TILE);
    bool all_fast = vec;
    for (int64_t s = s_lo; vec && s <= s_hi; ++s) {
      vec = !(may_width1 && s >= p.bnd.rem);
      all_fast = all_fast && p.cls[s] == kFast;
    }

    if (vec) {
      Acc acc[K];
      const int64_t vidx = t0 / K + threadIdx.x;  // 32-byte vector index
      const int64_t e0 = vidx * K;
      if (p.acc_in) {
        load_acc_in<D>(acc, p.acc_in + (e0 - p.ebeg));
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = D::zero();
      }
      V8 first;  // replica 0's raw vector: the fallback values unless a fallback vector is given
      const bool fb_first = !p.fallback && p.n_alive > 0 && fb_raw == s_src[0];
      if (all_fast)
        accumulate_vec<D, U, NOU>(acc, s_src, p.n_alive, vidx);
      else
        accumulate_vec<D, U, NOU, true>(acc, s_src, p.n_alive, vidx, &first);
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = D::mean(acc[k], p.n_div);
      // the vector's shard: known per tile unless the tile straddles a shard boundary (no
      // 64-bit divisions per vector then)
      const bool one_shard = s_lo == s_hi;
      const int64_t sa = all_fast ? 0 : (one_shard ? s_lo : p.bnd.shard_of(e0));
      const int64_t sb = all_fast ? 0 : (one_shard ? s_lo : p.bnd.shard_of(e0 + K - 1));
      const uint8_t c = all_fast ? (uint8_t)kFast : (sa == sb ? p.cls[sa] : (uint8_t)0xff);
      if (c == kFast) {
        if (p.merged) {
#pragma unroll
          for (int k = 0; k < K; k += 4)
            st_f64x4(p.merged + e0 + k, D::widen(acc[k]), D::widen(acc[k + 1]), D::widen(acc[k + 2]),
                     D::widen(acc[k + 3]));
        }
        const V8 out = D::pack(acc);
        for (int d = 0; d < p.n_dst; ++d) st_stream(reinterpret_cast<V8*>(s_dst[d]) + vidx, out);
        bool fin = true;
#pragma unroll
        for (int k = 0; k < K; ++k) fin = fin && finite64(D::widen(acc[k]));
        if (!fin) {  // rare: a replica holds NaN / Inf here
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (!finite64(D::widen(acc[k]))) mark_nonfinite_at(p, e0 + k);
        }
      } else if (c != 0xff) {  // one special or lost shard
        if (c == kSpecial) {  // the mean waits in the workspace for k_stats / k_apply
#pragma unroll
          for (int k = 0; k < K; k += 4)
            st_f64x4(p.ws + e0 + k, D::widen(acc[k]), D::widen(acc[k + 1]), D::widen(acc[k + 2]),
                     D::widen(acc[k + 3]));
        }
        const uint8_t pr = p.pred[sa] & kPredMask;
        if (pr == kPredMean) {
          if (merged_apart) {
#pragma unroll
            for (int k = 0; k < K; k += 4)
              st_f64x4(p.merged + e0 + k, D::widen(acc[k]), D::widen(acc[k + 1]), D::widen(acc[k + 2]),
                       D::widen(acc[k + 3]));
          }
          const V8 out = D::pack(acc);
          for (int d = 0; d < p.n_dst; ++d) st_stream(reinterpret_cast<V8*>(s_dst[d]) + vidx, out);
        } else if (pr == kPredFallback) {
          double v[K];
          if (fb_first)
            D::unpack_raw(first, v);  // streamed in by the accumulation above
          else
            fallback_vec<D>(p, fb_raw, vidx, v);  // read before the in-place stores below
          if (p.merged && (c == kLost || merged_apart)) {
#pragma unroll
            for (int k = 0; k < K; k += 4) st_f64x4(p.merged + e0 + k, v[k], v[k + 1], v[k + 2], v[k + 3]);
          }
          const V8 out = D::pack_d(v);
          for (int d = 0; d < p.n_dst; ++d) st_stream(reinterpret_cast<V8*>(s_dst[d]) + vidx, out);
        }
      } else {  // the vector straddles shards of different classes
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int64_t e = e0 + k;
          const int64_t se = p.bnd.shard_of(e);
          const uint8_t ce = p.cls[se];
          if (ce == kFast) {
            if (p.merged) p.merged[e] = D::widen(acc[k]);
            for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], e, D::widen(acc[k]));
            if (!finite64(D::widen(acc[k]))) mark_nonfinite(p, se);
          } else {
            emit_predicted<D>(p, s_dst, fb_raw, merged_apart, e, ce, p.pred[se] & kPredMask, D::widen(acc[k]));
          }
        }
      }
      // a whole tile of one special shard with two device-computable copies: its
      // pair statistics now, from the means in registers (k_stats skips the tile)
      if (!all_fast && s_lo == s_hi && (p.pred[s_lo] & kPredFuse) && p.stile == TILE) {
        const int32_t* mem = p.assign + s_lo * 2;
        const PairStat st = block_combine(pair_stats_vec<D>(acc, e0, p.corr[mem[0]], p.corr[mem[1]]));
        if (threadIdx.x == 0) {
          double* o = stat_slot(p, s_lo, tile, 0);
          o[0] = st.mx;
          o[1] = st.ab;
          o[2] = st.aa;
          o[3] = st.bb;
          p.done[tile] = 1;
        }
      }
    } else {
      for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads) {
        const int64_t s = p.bnd.shard_of(e);
        const uint8_t c = p.cls[s];
        if (c == kLost) {
          emit_predicted<D>(p, s_dst, fb_raw, merged_apart, e, c, p.pred[s] & kPredMask, 0.0);
          continue;
        }
        Acc m;
        if (p.acc_in) {  // chain continuation (width-1 shards are rejected on the host)
          Acc acc = (Acc)p.acc_in[e - p.ebeg];
          for (int q = 0; q < p.n_alive; ++q) acc = D::add(acc, D::load(s_src[q], e));
          m = D::mean(acc, p.n_div);
        } else {
          m = mean_at<D>(s_src, p.n_alive, e, p.bnd.len(s) == 1);
        }
        if (c == kFast) {
          if (p.merged) p.merged[e] = D::widen(m);
          for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], e, D::widen(m));
          if (!finite64(D::widen(m))) mark_nonfinite(p, s);
        } else {
          emit_predicted<D>(p, s_dst, fb_raw, merged_apart, e, c, p.pred[s] & kPredMask, D::widen(m));
        }
      }
    }
  }
}

// One link of the cross-GPU chain: acc_out = acc_in (or +0.0) + x_0 + x_1 + ...
// over this GPU's alive replicas, for elements [begin, end); the acc buffers are
// chunk-local.  Carrying the running fp64 sum from GPU to GPU keeps the
// reference's ascending-miner order, so the multi-GPU mean is bit-exact.
template <class D, bool BULK>
__global__ void __launch_bounds__(kThreads) k_chain(const void* const* src, int n_src, const double* acc_in,
                                                    double* acc_out, int64_t begin, int64_t end) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const void** s_src = reinterpret_cast<const void**>(smem_raw);
  const bool aligned = stage_pointers(s_src, nullptr, src, n_src, nullptr, 0,
                                      (uintptr_t)acc_in | (uintptr_t)acc_out);
  constexpr int K = D::K;
  constexpr int TILE = kThreads * K;
  using Acc = typename D::Acc;
  // BULK: each tile of sums is staged in shared memory (double buffer) and leaves
  // with one TMA bulk store (cp.async.bulk.global.shared::cta) — large NVLink
  // writes when acc_out is a peer GPU's inbox, issued by one thread
  double* stage = reinterpret_cast<double*>(smem_raw + ((sizeof(void*) * n_src + 127) & ~(size_t)127));
  int buf = 0, issued = 0;
  const int64_t tile_lo = begin / TILE, tile_hi = (end + TILE - 1) / TILE;
  for (int64_t tile = tile_lo + blockIdx.x; tile < tile_hi; tile += gridDim.x) {
    const int64_t t0 = max(tile * TILE, begin);
    const int64_t t1 = min(tile * TILE + TILE, end);
    if (aligned && t1 - t0 == TILE) {
      Acc acc[K];
      const int64_t vidx = t0 / K + threadIdx.x;
      const int64_t e0 = vidx * K;
      if (acc_in) {
        load_acc_in<D>(acc, acc_in + (e0 - begin));
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = D::zero();
      }
      accumulate_vec<D>(acc, s_src, n_src, vidx);
      if constexpr (BULK) {
        if (threadIdx.x == 0 && issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();  // stage[buf] no longer read by the store issued two tiles ago
        double* sb = stage + buf * TILE + threadIdx.x * K;
#pragma unroll
        for (int k = 0; k < K; ++k) sb[k] = (double)acc[k];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(stage + buf * TILE);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                       "cp.async.bulk.commit_group;" ::"l"(acc_out + (t0 - begin)),
                       "r"(sa), "r"((unsigned)(TILE * sizeof(double)))
                       : "memory");
        }
        ++issued;
        buf ^= 1;
      } else {
#pragma unroll
        for (int k = 0; k < K; k += 4)
          st_f64x4(acc_out + (e0 - begin) + k, (double)acc[k], (double)acc[k + 1], (double)acc[k + 2],
                   (double)acc[k + 3]);
      }
    } else {
      for (int64_t e = t0 + threadIdx.x; e < t1; e += kThreads) {
        Acc acc = acc_in ? (Acc)acc_in[e - begin] : D::zero();
        for (int q = 0; q < n_src; ++q) acc = D::add(acc, D::load(s_src[q], e));
        acc_out[e - begin] = (double)acc;
      }
    }
  }
  if constexpr (BULK) {
    if (threadIdx.x == 0 && issued) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// Gather element ranges of `full` into `packed` (SCATTER = false), or scatter
// `packed` back into every `dst` (SCATTER = true).  ranges[r] = {lo, hi, packed
// offset} in elements; the host keeps off = lo (mod 16 elements) so both sides of a
// range share their 32-byte alignment and the body moves with 256-bit accesses.
template <bool SCATTER>
__global__ void __launch_bounds__(kThreads) k_ranges(const unsigned char* full, unsigned char* packed,
                                                     unsigned char* const* dst, int n_dst, const int64_t* ranges,
                                                     int esize) {
  extern __shared__ __align__(16) const void* s_ptr[];
  unsigned char** s_dst = reinterpret_cast<unsigned char**>(const_cast<void**>(s_ptr));
  for (int q = threadIdx.x; q < n_dst; q += blockDim.x) s_dst[q] = dst[q];
  __syncthreads();
  const int64_t lo = ranges[3 * blockIdx.y] * esize, hi = ranges[3 * blockIdx.y + 1] * esize;
  const int64_t off = ranges[3 * blockIdx.y + 2] * esize;
  const unsigned char* src = SCATTER ? packed + off : full + lo;
  const int64_t n = hi - lo;
  const int nd = SCATTER ? n_dst : 1;
  auto dst_at = [&](int d) -> unsigned char* { return SCATTER ? s_dst[d] + lo : packed + off; };
  bool vec = true;
  for (int d = 0; d < nd; ++d) vec = vec && ((((uintptr_t)dst_at(d)) ^ (uintptr_t)src) & 31) == 0;
  int64_t head = vec ? (int64_t)((32 - ((uintptr_t)src & 31)) & 31) : n;
  if (head > n) head = n;
  const int64_t body = vec ? ((n - head) / 32) * 32 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < body / 32; v += stride) {
    const V8 x = ld_stream(src + head + 32 * v);
    for (int d = 0; d < nd; ++d) st_stream(dst_at(d) + head + 32 * v, x);
  }
  if (blockIdx.x == 0) {  // unaligned head and tail bytes
    for (int64_t i = threadIdx.x; i < head; i += blockDim.x) {
      const unsigned char x = src[i];
      for (int d = 0; d < nd; ++d) dst_at(d)[i] = x;
    }
    for (int64_t i = head + body + threadIdx.x; i < n; i += blockDim.x) {
      const unsigned char x = src[i];
      for (int d = 0; d < nd; ++d) dst_at(d)[i] = x;
    }
  }
}

// Scatter one final vector into several replicas (multi-GPU fan-out).
// The same with TMA bulk stores: a CTA stages a 32 KB tile in shared memory (double
// buffer) and one thread issues one cp.async.bulk store per destination.
constexpr int kFanTile = 32768;
__global__ void __launch_bounds__(kThreads) k_fanout_bulk(const void* src, void* const* dst, int n_dst,
                                                          int64_t nbytes) {
  extern __shared__ __align__(128) unsigned char fan_smem[];
  unsigned char* stage = fan_smem;  // [2][kFanTile]
  void** s_dst = reinterpret_cast<void**>(fan_smem + 2 * kFanTile);
  const bool aligned = stage_pointers(nullptr, s_dst, nullptr, 0, dst, n_dst, (uintptr_t)src);
  const int64_t ntiles = aligned ? nbytes / kFanTile : 0;
  int buf = 0, issued = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    V8 x[kFanTile / 32 / kThreads];
#pragma unroll
    for (int i = 0; i < kFanTile / 32 / kThreads; ++i)
      x[i] = ld_stream(reinterpret_cast<const V8*>((const unsigned char*)src + t * kFanTile) + i * kThreads +
                       threadIdx.x);
    if (threadIdx.x == 0 && issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();  // stage[buf] no longer read by the stores issued two tiles ago
#pragma unroll
    for (int i = 0; i < kFanTile / 32 / kThreads; ++i)
      reinterpret_cast<V8*>(stage + buf * kFanTile)[i * kThreads + threadIdx.x] = x[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(stage + buf * kFanTile);
      for (int d = 0; d < n_dst; ++d)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         (unsigned char*)s_dst[d] + t * kFanTile),
                     "r"(sa), "r"((unsigned)kFanTile)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    ++issued;
    buf ^= 1;
  }
  if (threadIdx.x == 0 && issued) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // tail bytes (and everything when unaligned)
  const int64_t done = ntiles * kFanTile;
  for (int64_t b = done + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char v = ((const unsigned char*)src)[b];
    for (int d = 0; d < n_dst; ++d) ((unsigned char*)s_dst[d])[b] = v;
  }
}

__global__ void __launch_bounds__(kThreads) k_fanout(const void* src, void* const* dst, int n_dst, int64_t nbytes) {
  extern __shared__ __align__(16) const void* s_ptr[];
  void** s_dst = const_cast<void**>(s_ptr);
  const bool aligned = stage_pointers(nullptr, s_dst, nullptr, 0, dst, n_dst, (uintptr_t)src);
  const int64_t nvec = aligned ? nbytes / 32 : 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const V8 x = ld_stream(reinterpret_cast<const V8*>(src) + v);
    for (int d = 0; d < n_dst; ++d) st_stream(reinterpret_cast<V8*>(s_dst[d]) + v, x);
  }
  for (int64_t b = nvec * 32 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char x = ((const unsigned char*)src)[b];
    for (int d = 0; d < n_dst; ++d) ((unsigned char*)s_dst[d])[b] = x;
  }
}

// ---------------------------------------------------------------------------
// special shards: statistics, decision, adoption
// ---------------------------------------------------------------------------

// Pair statistics of the special shards' tiles k_reduce did not cover (tiles shared
// by two shards, partial tiles at element-range edges, r = 3, host copies).
__device__ void stats_part(const Params& p, int64_t s, int y, int ny) {
  const int64_t start = p.bnd.start(s), hi_s = start + p.bnd.len(s);
  const int32_t* mem = p.assign + s * p.r;
  // the parts of a shard take its tiles in turn (part y, stride ny) and skip the ones the
  // reduce already covered (done[]); one slot per tile, so the order of the work does not
  // matter
  const int64_t t_first = start / p.stile, t_last = (hi_s - 1) / p.stile;
  // the part's tiles are checked kThreads at a time (one done[] byte per thread, not one
  // dependent load per tile for the whole CTA): the ones left form this batch's list
  __shared__ int64_t todo[kThreads];
  __shared__ int n_todo;
  for (int64_t base = t_first + y; base <= t_last; base += (int64_t)ny * kThreads) {
    __syncthreads();  // the previous batch's list is consumed
    if (threadIdx.x == 0) n_todo = 0;
    __syncthreads();
    const int64_t tc = base + (int64_t)threadIdx.x * ny;
    if (tc <= t_last && !p.done[tc]) todo[atomicAdd(&n_todo, 1)] = tc;
    __syncthreads();
    const int cnt = n_todo;
    for (int q = 0; q < cnt; ++q) {
      const int64_t t = todo[q];
      const int64_t lo = max(t * p.stile, start), hi = min((t + 1) * p.stile, hi_s);
      const int64_t g_lo = lo & ~(int64_t)3;
      for (int a = 0; a < p.r; ++a)
        for (int b = a + 1; b < p.r; ++b) {
          if (p.failed[mem[a]] || p.failed[mem[b]]) continue;
          // the two descriptors in registers (a runtime-indexed local array lives on the stack)
          const bfly_corruption_t ca = p.corr[mem[a]], cb = p.corr[mem[b]];
          PairAcc acc;
          // four elements (one Philox block per noisy copy) per thread and step: few live
          // registers, so 4 CTAs per SM hide the Philox dependency chains; two steps
          // unrolled (best of bound x unroll, profiles/r02_ab_kstats.log)
  #pragma unroll 2
          for (int64_t e0 = g_lo + 4 * (int64_t)threadIdx.x; e0 < hi; e0 += 4 * kThreads) {
            double m[4], x[4], z[4];
            const unsigned valid = load_group4(p.ws, e0, lo, hi, m);
            corrupt4h(ca, m, e0, valid, p.host_copies, a, p.P, x);
            corrupt4h(cb, m, e0, valid, p.host_copies, b, p.P, z);
            if (valid == 0xf) {  // whole group: no per-element predicates
  #pragma unroll
              for (int i = 0; i < 4; ++i) acc.add(x[i], z[i]);
            } else {
  #pragma unroll
              for (int i = 0; i < 4; ++i)
                if ((valid >> i) & 1) acc.add(x[i], z[i]);
            }
          }
          const PairStat st = block_combine_smem(acc.finish());
          if (threadIdx.x == 0) {
            double* o = stat_slot(p, s, t, pair_index(p.r, a, b));
            o[0] = st.mx;
            o[1] = st.ab;
            o[2] = st.aa;
            o[3] = st.bb;
          }
        }
    }
  }
}

// A persistent grid walks (shard, part) items: most shards are fast and cost one byte
// load, not a CTA launch each (2016 shards x 64 parts at 64 miners).
__global__ void __launch_bounds__(kThreads, 4) k_stats(Params p, int ny) {
  if (*(volatile uint32_t*)p.special_any == 0u) return;  // every shard fast (k_classify)
  const int64_t items = (int64_t)p.n_fin * ny;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t s = fin_shard(p, (unsigned)(it / ny));
    if (p.cls[s] == kSpecial) stats_part(p, s, (int)(it % ny), ny);
  }
}

// One warp per shard.
__global__ void k_decide(Params p) {
  if (*(volatile uint32_t*)p.special_any == 0u) return;
  const int64_t s = fin_shard(p, blockIdx.x);
  if (p.cls[s] != kSpecial) return;
  const int lane = threadIdx.x;
  const int32_t* mem = p.assign + s * p.r;
  const int64_t start = p.bnd.start(s), len = p.bnd.len(s);
  const int64_t t0 = start / p.stile, ntiles = (start + len - 1) / p.stile - t0 + 1;
  int surv[kMaxR], ns = 0;
  for (int k = 0; k < p.r; ++k)
    if (!p.failed[mem[k]]) surv[ns++] = k;
  bool agree[kMaxR][kMaxR] = {};
  for (int x = 0; x < ns; ++x)
    for (int y = x + 1; y < ns; ++y) {
      const int pi = pair_index(p.r, surv[x], surv[y]);
      PairStat st{0.0, 0.0, 0.0, 0.0};
      for (int64_t ch = lane; ch < ntiles; ch += 32) {
        const double* o = stat_slot(p, s, t0 + ch, pi);
        st.mx = max_nan(st.mx, o[0]);
        st.ab = __dadd_rn(st.ab, o[1]);
        st.aa = __dadd_rn(st.aa, o[2]);
        st.bb = __dadd_rn(st.bb, o[3]);
      }
      st = warp_combine(st);
      const double sc = score_of(st, p.tol);
      agree[x][y] = agree[y][x] = sc == 1.0;
      if (lane == 0) {
        const int i = mem[surv[x]], j = mem[surv[y]];
        if (p.r == 2) {
          p.entries[(int64_t)i * p.n + j] = sc;
          p.entries[(int64_t)j * p.n + i] = sc;
        } else {
          p.scores[s * p.npairs + pi] = sc;
          p.has_score[s * p.npairs + pi] = 1;
        }
      }
    }
  if (lane != 0) return;
  // adopt the lowest survivor backed by a strict majority of the survivors
  // (r = 2: both agree, or a lone survivor — butterfly.py:255-263)
  int src = -1;
  for (int x = 0; x < ns && src < 0; ++x) {
    int cnt = 1;
    for (int y = 0; y < ns; ++y)
      if (y != x && agree[x][y]) ++cnt;
    if (2 * cnt > ns) src = x;
  }
  if (src >= 0) {
    p.status[s] = BFLY_MERGED;
    p.source[s] = mem[surv[src]];
    for (int y = 0; y < ns; ++y)
      if (y != src && !agree[src][y]) p.flagged[mem[surv[y]]] = 1;
  } else {
    p.status[s] = ns >= 2 ? BFLY_DISAGREEMENT : BFLY_LOST;
    p.source[s] = -1;
    if (ns >= 2)
      for (int y = 0; y < ns; ++y) p.flagged[mem[surv[y]]] = 1;
  }
  if (apply_needed(p, s)) atomicOr(p.apply_any, 1u);
}

// r = 3: entries[i][j] = min over the N-2 shards sharing {i, j} (NaN poisons), in the
// order x = 0, 1, ... of the third member: the first NaN wins, and among equal minima the
// first one (as a sequential `sc < best` scan keeps it).  One warp per pair (i < j), the
// lanes taking x in turn; (value, x) pairs combined in a warp tree.
__global__ void k_entries3(Params p) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)p.n * p.n) return;  // warp-uniform
  const int i = (int)(w / p.n), j = (int)(w % p.n);
  if (i >= j) return;                  // warp-uniform
  constexpr int kNone = 0x7fffffff;
  double best = 0.0, nanv = 0.0;
  int bx = kNone, nx = kNone;  // x of the lane's minimum / first NaN
  for (int x = lane; x < p.n; x += 32) {
    if (x == i || x == j) continue;
    int32_t m[3];
    int a, b;  // slots of i and j
    if (x < i) { m[0] = x; m[1] = i; m[2] = j; a = 1; b = 2; }
    else if (x < j) { m[0] = i; m[1] = x; m[2] = j; a = 0; b = 2; }
    else { m[0] = i; m[1] = j; m[2] = x; a = 0; b = 1; }
    const int32_t s = p.inv[rank_combination(p.n, 3, m)];
    const int pi = pair_index(3, a, b);
    if (!p.has_score[(int64_t)s * 3 + pi]) continue;
    const double sc = p.scores[(int64_t)s * 3 + pi];
    if (isnan(sc)) {
      if (nx == kNone) { nx = x; nanv = sc; }
    } else if (bx == kNone || sc < best) {
      best = sc;
      bx = x;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const int onx = __shfl_xor_sync(0xffffffffu, nx, off);
    const double onv = __shfl_xor_sync(0xffffffffu, nanv, off);
    const int obx = __shfl_xor_sync(0xffffffffu, bx, off);
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    if (onx < nx) { nx = onx; nanv = onv; }
    if (obx != kNone && (bx == kNone || ob < best || (ob == best && obx < bx))) { best = ob; bx = obx; }
  }
  if (lane == 0 && (nx != kNone || bx != kNone)) {
    const double v = nx != kNone ? nanv : best;
    p.entries[(int64_t)i * p.n + j] = v;
    p.entries[(int64_t)j * p.n + i] = v;
  }
}

template <class D>
__device__ void apply_chunk(const Params& p, void* const* s_dst, bool aligned, int64_t s, int64_t ch) {
  const uint8_t c = p.cls[s];
  const int64_t lo = p.bnd.start(s) + ch * kChunk;
  const int64_t hi_s = p.bnd.start(s) + p.bnd.len(s);
  const int64_t hi = lo + kChunk < hi_s ? lo + kChunk : hi_s;
  const int32_t src_m = p.source[s];
  int slot = -1;
  bfly_corruption_t cd{};
  if (src_m >= 0) {
    for (int k = 0; k < p.r; ++k)
      if (p.assign[s * p.r + k] == src_m) slot = k;
    cd = p.corr[src_m];
  }
  // k_reduce already wrote the predicted outcome; only the merged vector may still
  // need the fallback values (when it doubles as the workspace of the means)
  const uint8_t pr = p.pred[s] & kPredMask;
  const bool as_predicted = src_m < 0 ? pr == kPredFallback : (pr == kPredMean && cd.kind == BFLY_CORR_NONE);
  int n_dst = p.n_dst;
  if (as_predicted) {
    if (!(src_m < 0 && c == kSpecial && p.merged && p.merged == p.ws)) return;
    n_dst = 0;
  }
  const void* fb_raw = p.fb_src ? p.fb_src : (p.n_alive > 0 ? p.src[0] : nullptr);
  for (int64_t e0 = (lo & ~(int64_t)7) + 8 * (int64_t)threadIdx.x; e0 < hi; e0 += 8 * kThreads) {
    double v[8];
    unsigned valid;
    if (slot >= 0) {
      double m[8];
      valid = load_group(p.ws, e0, lo, hi, m);
      corrupt8(cd, m, e0, valid, p.host_copies, slot, p.P, v);
    } else {
      valid = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t e = e0 + i;
        const bool in = e >= lo && e < hi;
        valid |= (unsigned)in << i;
        if (!in) v[i] = 0.0;
        else if (p.fallback) v[i] = p.fallback[e];
        else if (fb_raw) v[i] = D::raw(fb_raw, e);  // lowest alive upload (butterfly.py:270-271)
        else v[i] = nan64();
      }
    }
    if (valid == 0xff && aligned) {
      if (p.merged) {
        st_f64x4(p.merged + e0, v[0], v[1], v[2], v[3]);
        st_f64x4(p.merged + e0 + 4, v[4], v[5], v[6], v[7]);
      }
      for (int d = 0; d < n_dst; ++d) D::store8(s_dst[d], e0, v);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (!((valid >> i) & 1)) continue;
        if (p.merged) p.merged[e0 + i] = v[i];
        for (int d = 0; d < n_dst; ++d) D::store(s_dst[d], e0 + i, v[i]);
      }
    }
  }
}

// A persistent grid walks (shard, chunk) items; fast shards are skipped with one byte load.
template <class D>
__global__ void __launch_bounds__(kThreads) k_apply(Params p) {
  extern __shared__ __align__(16) const void* s_ptr[];  // [n_dst] scatter-back targets
  if (*(volatile uint32_t*)p.apply_any == 0u) return;  // every shard as k_reduce wrote it
  void** s_dst = const_cast<void**>(s_ptr);
  const bool aligned = stage_pointers(nullptr, s_dst, nullptr, 0, p.dst, p.n_dst, (uintptr_t)p.merged);
  const int64_t items = (int64_t)p.n_fin * p.cps;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t s = fin_shard(p, (unsigned)(it / p.cps));
    if (p.cls[s] != kFast) apply_chunk<D>(p, s_dst, aligned, s, it % p.cps);
  }
}

// Fast shards marked by k_reduce (non-finite mean somewhere) with >= 2 survivors:
// status disagreement, every survivor flagged, entries NaN (r = 3: scores NaN), and
// the fallback values into merged and the replicas (butterfly.py:255,264-273).  The
// fallback is the caller's, else the lowest alive replica unless the scatter-back has
// overwritten it in place (then NaN: its values are gone).  A persistent grid walks
// (shard, chunk) items; without a marked shard every CTA returns at once.
template <class D>
__global__ void __launch_bounds__(kThreads) k_nonfinite(Params p) {
  extern __shared__ __align__(16) const void* s_ptr[];
  if (*(volatile uint32_t*)p.nonfin_any == 0u) return;
  void** s_dst = const_cast<void**>(s_ptr);
  stage_pointers(nullptr, s_dst, nullptr, 0, p.dst, p.n_dst, 0);
  const void* fb_raw = p.fb_src ? p.fb_src : (p.n_alive > 0 ? p.src[0] : nullptr);
  bool fb_ok = fb_raw != nullptr && !p.fb_gone;
  for (int d = 0; d < p.n_dst && fb_ok; ++d) fb_ok = s_dst[d] != fb_raw;
  const int64_t items = (int64_t)p.n_fin * p.cps;  // this call's shards (all, a range or a list)
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t s = fin_shard(p, (unsigned)(it / p.cps)), ch = it % p.cps;
    if (!p.nonfin[s] || p.cls[s] != kFast) continue;
    const int32_t* mem = p.assign + s * p.r;
    int surv[kMaxR], ns = 0;
    for (int k = 0; k < p.r; ++k)
      if (!p.failed[mem[k]]) surv[ns++] = k;
    if (ns < 2) continue;  // a lone survivor agrees trivially: its mean stands
    if (ch == 0 && threadIdx.x == 0) {
      p.status[s] = BFLY_DISAGREEMENT;
      p.source[s] = -1;
      for (int x = 0; x < ns; ++x) {
        p.flagged[mem[surv[x]]] = 1;
        for (int y = x + 1; y < ns; ++y) {
          const int i = mem[surv[x]], j = mem[surv[y]];
          if (p.r == 2) {
            p.entries[(int64_t)i * p.n + j] = nan64();
            p.entries[(int64_t)j * p.n + i] = nan64();
          } else {
            const int pi = pair_index(p.r, surv[x], surv[y]);
            p.scores[s * p.npairs + pi] = nan64();
            p.has_score[s * p.npairs + pi] = 1;
          }
        }
      }
    }
    const int64_t lo = p.bnd.start(s) + ch * kChunk, hi_s = p.bnd.start(s) + p.bnd.len(s);
    const int64_t hi = lo + kChunk < hi_s ? lo + kChunk : hi_s;
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) {
      const double v = p.fallback ? p.fallback[e] : (fb_ok ? D::raw(fb_raw, e) : nan64());
      if (p.merged) p.merged[e] = v;
      for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], e, v);
    }
  }
}

// Multi-GPU ranks other than the last: after the per-shard results arrive, the fast
// shards the last rank decided a disagreement (non-finite means, k_nonfinite) get the
// fallback values — the given fallback, or NaN (the relay has overwritten the lowest alive
// replica) — in every local replica, without a host round trip.
template <class D>
__global__ void __launch_bounds__(kThreads) k_fill_shards(const uint8_t* status, const uint8_t* mask,
                                                          const double* fallback, void* const* dst, int n_dst,
                                                          Bounds bnd, int64_t cps) {
  extern __shared__ __align__(16) const void* s_ptr[];
  void** s_dst = const_cast<void**>(s_ptr);
  // almost always nothing to do: one parallel pass over the shards decides (the per-item
  // loop below would walk S x cps dependent loads per CTA)
  int any = 0;
  for (int64_t s = threadIdx.x; s < bnd.S; s += blockDim.x) any |= mask[s] && status[s] == BFLY_DISAGREEMENT;
  if (!__syncthreads_or(any)) return;
  stage_pointers(nullptr, s_dst, nullptr, 0, dst, n_dst, 0);
  const int64_t items = bnd.S * cps;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t s = it / cps, ch = it % cps;
    if (!mask[s] || status[s] != BFLY_DISAGREEMENT) continue;
    const int64_t lo = bnd.start(s) + ch * kChunk, hi_s = bnd.start(s) + bnd.len(s);
    const int64_t hi = lo + kChunk < hi_s ? lo + kChunk : hi_s;
    for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) {
      const double v = fallback ? fallback[e] : nan64();
      for (int d = 0; d < n_dst; ++d) D::store(s_dst[d], e, v);
    }
  }
}

// ---------------------------------------------------------------------------
// standalone agreement and mean_reducer
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) k_agree_partial(const double* a, const double* b, int64_t len,
                                                            double* part) {
  const int64_t lo = (int64_t)blockIdx.x * kChunk;
  const int64_t hi = lo + kChunk < len ? lo + kChunk : len;
  PairAcc acc;
  for (int64_t e = lo + threadIdx.x; e < hi; e += kThreads) acc.add(a[e], b[e]);
  const PairStat st = block_combine(acc.finish());
  if (threadIdx.x == 0) {
    part[blockIdx.x * 4 + 0] = st.mx;
    part[blockIdx.x * 4 + 1] = st.ab;
    part[blockIdx.x * 4 + 2] = st.aa;
    part[blockIdx.x * 4 + 3] = st.bb;
  }
}

__global__ void k_agree_final(const double* part, int64_t nchunks, double tol, double* out) {
  PairStat st{0.0, 0.0, 0.0, 0.0};
  for (int64_t ch = threadIdx.x; ch < nchunks; ch += 32) {
    st.mx = max_nan(st.mx, part[ch * 4]);
    st.ab = __dadd_rn(st.ab, part[ch * 4 + 1]);
    st.aa = __dadd_rn(st.aa, part[ch * 4 + 2]);
    st.bb = __dadd_rn(st.bb, part[ch * 4 + 3]);
  }
  st = warp_combine(st);
  if (threadIdx.x == 0) *out = score_of(st, tol);
}

// numpy DOUBLE_pairwise_sum over a contiguous column (width-1 stacks).
__device__ double pairwise_contig(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_contig(a, n2), pairwise_contig(a + n2, n - n2));
}

__global__ void k_corrupt(bfly_corruption_t c, const double* in, int64_t start, int64_t len, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = corrupt_value(c, in[i], start + i, nullptr, 0, 0);
}

__global__ void k_mean_rows(const double* stack, int32_t rows, int64_t width, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < width;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (width == 1) {
      acc = __dadd_rn(0.0, pairwise_contig(stack, rows));
    } else {
      for (int q = 0; q < rows; ++q) acc = __dadd_rn(acc, stack[(int64_t)q * width + e]);
    }
    out[e] = __ddiv_rn(acc, (double)rows);
  }
}

}  // namespace bfly

using namespace bfly;

// k_chain stores its fp64 sums through shared-memory staging and TMA bulk stores: into a
// peer GPU's inbox 1.5x faster than 256-bit SM stores (16 replicas x 16M elements: 0.21 vs
// 0.32 ms, tools/peer_bw.py).  k_fanout uses 256-bit SM stores (its bulk variant, 32 KB
// tiles staged in shared memory, was no faster: profiles/r01_fanout_probe.log).
constexpr bool kChainBulk = true;
constexpr bool kFanoutBulk = false;
static int64_t cap_grid(int64_t grid) { return grid < 1 ? 1 : grid; }

template <class D, int U = 4, int MINB = 1, bool NOU = false>
static void launch_reduce(const Params& p, cudaStream_t st, int grid_per_sm = 8) {
  const int64_t tile = (int64_t)kThreads * D::K;
  const int64_t ntiles = (p.eend + tile - 1) / tile - p.ebeg / tile;
  int64_t grid = (int64_t)sm_count() * grid_per_sm;
  if (grid > ntiles) grid = ntiles;
  grid = cap_grid(grid);
  if (grid < 1) grid = 1;
  const size_t smem = sizeof(void*) * (size_t)(p.n_alive + p.n_dst);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_reduce<D, U, MINB, NOU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_reduce<D, U, MINB, NOU><<<(unsigned)grid, kThreads, smem, st>>>(p);
}

template <class D>
static void launch_nonfinite(const Params& p, cudaStream_t st) {
  const size_t smem = sizeof(void*) * (size_t)(p.n_dst > 0 ? p.n_dst : 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_nonfinite<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t grid = (int64_t)p.n_fin * p.cps;
  if (grid > (int64_t)sm_count() * 2) grid = (int64_t)sm_count() * 2;
  k_nonfinite<D><<<(unsigned)(grid < 1 ? 1 : grid), kThreads, smem, st>>>(p);
}

static void launch_nonfinite_dt(int32_t dtype, const Params& p, cudaStream_t st) {
  switch (dtype) {
    case BFLY_F32: launch_nonfinite<DF32>(p, st); break;
    case BFLY_BF16: launch_nonfinite<DBF16>(p, st); break;
    default: launch_nonfinite<DF64W>(p, st); break;
  }
}

template <class D>
static void launch_apply(const Params& p, cudaStream_t st) {
  const size_t smem = sizeof(void*) * (size_t)(p.n_dst > 0 ? p.n_dst : 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_apply<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t grid = (int64_t)p.n_fin * p.cps;
  if (grid > (int64_t)sm_count() * 8) grid = (int64_t)sm_count() * 8;
  k_apply<D><<<(unsigned)(grid < 1 ? 1 : grid), kThreads, smem, st>>>(p);
}

extern "C" {

size_t bfly_merge_scratch_bytes(int32_t n_miners, int32_t redundancy, int64_t payload_len) {
  ScratchLayout L;
  L.init(n_miners, redundancy, payload_len);
  return L.total;
}

static int build_params(const bfly_merge_args_t* a, Params& p) {
  if (!a) return fail(BFLY_E_INVALID_ARG, "null args");
  if (a->n_miners < 2) return fail(BFLY_E_TOO_FEW_MINERS, "need at least 2 miners");
  if (a->redundancy < 2 || a->redundancy > kMaxR)
    return fail(BFLY_E_UNSUPPORTED, "device merge supports redundancy 2 or 3");
  const int64_t S = binom(a->n_miners, a->redundancy);
  if (S != a->n_shards) return fail(BFLY_E_SHAPE, "n_shards != C(n_miners, redundancy)");
  if (a->payload_len < S) return fail(BFLY_E_DEGENERATE, "payload cannot fill every shard");
  if (a->n_alive < 0 || a->n_alive > a->n_miners) return fail(BFLY_E_INVALID_ARG, "bad n_alive");
  if (a->dtype != BFLY_F32 && a->dtype != BFLY_BF16 && a->dtype != BFLY_F64WIRE)
    return fail(BFLY_E_INVALID_ARG, "bad dtype");
  if (!a->d_assign || !a->d_failed || !a->d_corr || !a->d_status || !a->d_entries || !a->d_flagged)
    return fail(BFLY_E_INVALID_ARG, "missing required device array");
  if (a->n_alive > 0 && !a->d_src) return fail(BFLY_E_INVALID_ARG, "missing replicas");
  if (a->n_alive == 0 && a->n_div > 0 && !a->d_acc_in && a->phase != BFLY_PHASE_FINISH &&
      a->phase != BFLY_PHASE_CHECK)
    return fail(BFLY_E_INVALID_ARG, "n_div without replicas");  // (FINISH / CHECK read no replica sums)
  if (a->n_dst > 0 && !a->d_dst) return fail(BFLY_E_INVALID_ARG, "missing scatter-back targets");
  if (!a->d_merged && !a->d_ws) return fail(BFLY_E_INVALID_ARG, "need d_merged or d_ws");
  ScratchLayout L;
  L.init(a->n_miners, a->redundancy, a->payload_len);
  if (!a->d_scratch || a->scratch_bytes < L.total)
    return fail(BFLY_E_INVALID_ARG, "scratch too small: need " + std::to_string(L.total) + " bytes");
  if ((int64_t)(a->n_alive + a->n_dst) * 8 > 200 * 1024) return fail(BFLY_E_UNSUPPORTED, "too many replicas");
  if (L.cps > 65535) return fail(BFLY_E_UNSUPPORTED, "shards longer than 65535 chunks");

  p = Params{};
  p.n = a->n_miners;
  p.r = a->redundancy;
  p.n_alive = a->n_alive;
  p.n_dst = a->n_dst;
  p.npairs = L.npairs;
  p.P = a->payload_len;
  p.S = S;
  p.cps = L.cps;
  p.bnd.init(a->payload_len, S);
  p.assign = a->d_assign;
  p.src = a->d_src;
  p.failed = a->d_failed;
  p.corr = a->d_corr;
  p.dst = a->d_dst;
  p.fallback = a->d_fallback;
  p.merged = a->d_merged;
  p.ws = a->d_ws ? a->d_ws : a->d_merged;  // keep special-shard means apart when given
  p.host_copies = a->d_host_copies;
  p.status = a->d_status;
  p.entries = a->d_entries;
  p.flagged = a->d_flagged;
  unsigned char* sc = (unsigned char*)a->d_scratch;
  p.cls = sc + L.off_cls;
  p.pred = sc + L.off_pred;
  p.done = sc + L.off_done;
  p.stile = (int64_t)kThreads * (a->dtype == BFLY_F32 ? DF32::K : a->dtype == BFLY_BF16 ? DBF16::K : DF64W::K);
  if (a->stat_tile != 0) {  // the persistent ring's tile (its kernel writes the partials)
    if (a->stat_tile < kMinStatTile || a->stat_tile % kMinStatTile)
      return fail(BFLY_E_INVALID_ARG, "stat_tile must be a multiple of " + std::to_string(kMinStatTile));
    p.stile = a->stat_tile;
  }
  p.source = a->d_source ? a->d_source : (int32_t*)(sc + L.off_source);
  p.stats = (double*)(sc + L.off_stats);
  p.scores = (double*)(sc + L.off_scores);
  p.has_score = sc + L.off_has;
  p.inv = p.r > 2 ? (int32_t*)(sc + L.off_inv) : nullptr;
  p.tol = a->tolerance;
  p.acc_in = a->d_acc_in;
  p.n_div = a->n_div > 0 ? a->n_div : a->n_alive;
  p.ebeg = a->elem_begin;
  p.eend = (a->elem_begin == 0 && a->elem_end == 0) ? a->payload_len : a->elem_end;
  if (p.ebeg < 0 || p.eend > p.P || p.ebeg > p.eend) return fail(BFLY_E_INVALID_ARG, "bad element range");
  if (p.acc_in && p.bnd.base == 1) return fail(BFLY_E_UNSUPPORTED, "chained reduction needs shards of >= 2 elements");
  p.fb_src = a->d_fallback_src ? a->d_fallback_src : nullptr;
  p.sbeg = a->shard_begin;
  p.send = (a->shard_begin == 0 && a->shard_end == 0) ? S : a->shard_end;
  if (p.sbeg < 0 || p.send > S || p.sbeg > p.send) return fail(BFLY_E_INVALID_ARG, "bad shard range");
  p.slist = a->d_shard_list;
  if (p.slist && a->n_shard_list < 0) return fail(BFLY_E_INVALID_ARG, "bad shard list");
  p.n_fin = p.slist ? a->n_shard_list : (int32_t)(p.send - p.sbeg);
  p.fb_gone = a->fallback_gone != 0;
  p.nonfin_any = (uint32_t*)(sc + L.off_nonfin);
  p.special_any = (uint32_t*)(sc + L.off_nonfin + 4);
  p.apply_any = (uint32_t*)(sc + L.off_nonfin + 8);
  p.nonfin = sc + L.off_nonfin + 16;
  return BFLY_OK;
}

}  // extern "C"

namespace bfly {
// Per-round setup of the shard results without a reduce (the fused multi-GPU ring,
// bfly_ring.cu, reduces inside its own kernel): entries NaN, flags cleared, classify.
int ring_round_setup(const bfly_merge_args_t* a, void* stream, RingSpecial* out) {
  Params p;
  bfly_merge_args_t b = *a;
  b.phase = BFLY_PHASE_FINISH;  // no reduce here: the last rank may hold no alive replica
  int rc = build_params(&b, p);
  if (rc) return rc;
  // the kernel reduces every element (from the chained sums), so k_classify predicts the
  // outcomes as for a chained reduce even when this rank holds no alive replica
  static const double kChained = 0.0;
  p.acc_in = &kChained;
  if (out) {
    out->cls = p.cls;
    out->pred = p.pred;
    out->bnd = p.bnd;
    out->ws = p.ws;
    out->fallback = p.fallback;
    out->fb_src = p.fb_src;  // the multi-GPU last rank always names it (the lowest alive miner's replica)
    out->merged_apart = p.merged && p.merged != p.ws;
    out->nonfin_any = p.nonfin_any;
    out->nonfin = p.nonfin;
    out->assign = p.assign;
    out->corr = p.corr;
    out->stats = p.stats;
    out->done = p.done;
    out->stile = p.stile;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nn = (int64_t)p.n * p.n;
  k_fill_nan<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(p.entries, nn);
  cudaMemsetAsync(p.flagged, 0, (size_t)p.n, st);
  cudaMemsetAsync(p.done, 0, (size_t)(p.P / p.stile + 1), st);
  cudaMemsetAsync(p.nonfin_any, 0, 16 + (size_t)p.S, st);
  k_classify<<<(unsigned)((p.S + 255) / 256), 256, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ring round setup");
  return BFLY_OK;
}
}  // namespace bfly

extern "C" {

int bfly_merge(const bfly_merge_args_t* a, void* stream) {
  Params p;
  int rc = build_params(a, p);
  if (rc) return rc;
  const int64_t S = p.S;
  cudaStream_t st = (cudaStream_t)stream;

  if (a->phase < BFLY_PHASE_ALL || a->phase > BFLY_PHASE_CHECK) return fail(BFLY_E_INVALID_ARG, "bad phase");
  const bool do_reduce = a->phase == BFLY_PHASE_ALL || a->phase == BFLY_PHASE_REDUCE;
  const bool do_finish = (a->phase == BFLY_PHASE_ALL || a->phase == BFLY_PHASE_FINISH) && p.n_fin > 0;
  // non-finite fast shards are decided once the whole payload is reduced (the range
  // ending at P), and again by every FINISH / CHECK call (idempotent)
  const bool do_check = ((do_reduce && p.eend == p.P) || a->phase == BFLY_PHASE_FINISH ||
                         a->phase == BFLY_PHASE_CHECK) && p.n_fin > 0;
  if (do_reduce) {
    if (p.ebeg == 0) {  // per-round setup runs with the first (or only) element range
      const int64_t nn = (int64_t)p.n * p.n;
      k_fill_nan<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(p.entries, nn);
      cudaMemsetAsync(p.flagged, 0, (size_t)p.n, st);
      cudaMemsetAsync(p.done, 0, (size_t)(p.P / p.stile + 1), st);
      cudaMemsetAsync(p.nonfin_any, 0, 16 + (size_t)p.S, st);
      k_classify<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(p);
    }
    if ((p.n_alive > 0 || p.acc_in) && p.eend > p.ebeg) {
      switch (a->dtype) {
        case BFLY_F32:  // U=4, 3 CTAs/SM, 16 CTAs/SM grid: best of tools/tune_reduce.py (profiles/)
          launch_reduce<DF32, 4, 3, true>(p, st, 16);
          break;
        case BFLY_BF16:  // U=8, 1 CTA/SM bound, 16 CTAs/SM grid: best of the bf16 sweep (profiles/)
          launch_reduce<DBF16, 8, 1, true>(p, st, 16);
          break;
        default: launch_reduce<DF64W>(p, st); break;
      }
    }
  }
  if (do_check) launch_nonfinite_dt(a->dtype, p, st);
  if (do_finish) {
    const unsigned ns = (unsigned)p.n_fin;
    const int64_t tps = (p.bnd.base + (p.bnd.rem ? 1 : 0) + p.stile - 1) / p.stile + 1;  // tiles per shard
    // up to 64 CTAs per shard: a shard whose tiles were not covered by k_reduce (the
    // multi-GPU persistent ring computes no statistics) spreads over the GPU
    const int64_t ny = tps < 64 ? tps : 64;
    int64_t sgrid = (int64_t)ns * ny;
    if (sgrid > (int64_t)sm_count() * 8) sgrid = (int64_t)sm_count() * 8;
    k_stats<<<(unsigned)(sgrid < 1 ? 1 : sgrid), kThreads, 0, st>>>(p, (int)ny);
    k_decide<<<ns, 32, 0, st>>>(p);
    if (p.r > 2) {
      const int64_t nn = (int64_t)p.n * p.n;
      k_entries3<<<(unsigned)((nn * 32 + 255) / 256), 256, 0, st>>>(p);  // a warp per pair
    }
    switch (a->dtype) {
      case BFLY_F32: launch_apply<DF32>(p, st); break;
      case BFLY_BF16: launch_apply<DBF16>(p, st); break;
      default: launch_apply<DF64W>(p, st); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_merge launch");
  return BFLY_OK;
}

#ifdef BFLY_TUNING
// Tuning build only (build/libbfly_tune.so, tools/tune_reduce.py): launch k_reduce
// alone with a chosen (replicas in flight, min CTAs/SM) variant and grid size, on
// params whose per-round setup already ran through bfly_merge.
int bfly_tune_reduce(const bfly_merge_args_t* a, int variant, int grid_per_sm, void* stream) {
  Params p;
  int rc = build_params(a, p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (a->dtype == BFLY_BF16) {
    switch (variant) {
      case 0: launch_reduce<DBF16, 4, 1, false>(p, st, grid_per_sm); break;
      case 1: launch_reduce<DBF16, 4, 2, true>(p, st, grid_per_sm); break;
      case 2: launch_reduce<DBF16, 8, 1, true>(p, st, grid_per_sm); break;
      case 3: launch_reduce<DBF16, 2, 2, true>(p, st, grid_per_sm); break;
      case 4: launch_reduce<DBF16, 4, 3, true>(p, st, grid_per_sm); break;
      case 5: launch_reduce<DBF16, 2, 3, true>(p, st, grid_per_sm); break;
      case 6: launch_reduce<DBF16, 2, 4, true>(p, st, grid_per_sm); break;
      case 7: launch_reduce<DBF16, 4, 1, true>(p, st, grid_per_sm); break;
      default: return fail(BFLY_E_INVALID_ARG, "unknown variant");
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "bfly_tune_reduce launch");
    return BFLY_OK;
  }
  if (a->dtype != BFLY_F32) return fail(BFLY_E_UNSUPPORTED, "tuning covers fp32 and bf16");
  switch (variant) {
    case 0: launch_reduce<DF32, 4, 1, false>(p, st, grid_per_sm); break;
    case 1: launch_reduce<DF32, 4, 2, true>(p, st, grid_per_sm); break;
    case 2: launch_reduce<DF32, 8, 1, true>(p, st, grid_per_sm); break;
    case 3: launch_reduce<DF32, 8, 2, true>(p, st, grid_per_sm); break;
    case 4: launch_reduce<DF32, 4, 3, true>(p, st, grid_per_sm); break;
    case 5: launch_reduce<DF32, 16, 1, true>(p, st, grid_per_sm); break;
    case 6: launch_reduce<DF32, 2, 4, true>(p, st, grid_per_sm); break;
    case 7: launch_reduce<DF32, 4, 1, true>(p, st, grid_per_sm); break;
    default: return fail(BFLY_E_INVALID_ARG, "unknown variant");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_tune_reduce launch");
  return BFLY_OK;
}
#endif

// Load every kernel a merge round (single-GPU or a rank of the chunked ring) may launch.
// With CUDA's lazy module loading a kernel's first launch loads it, and a load may wait
// for the device: on ONE device running several ranks (the loopback ring) whose streams
// already wait on each other's flags, that first launch would deadlock.
int bfly_preload(void) {
  const void* fns[] = {
      (const void*)k_fill_nan, (const void*)k_classify, (const void*)k_stats, (const void*)k_decide,
      (const void*)k_entries3, (const void*)k_apply<DF32>, (const void*)k_apply<DBF16>,
      (const void*)k_apply<DF64W>, (const void*)k_nonfinite<DF32>, (const void*)k_nonfinite<DBF16>,
      (const void*)k_nonfinite<DF64W>, (const void*)k_reduce<DF32, 4, 3, true>,
      (const void*)k_reduce<DBF16, 8, 1, true>, (const void*)k_reduce<DF64W>, (const void*)k_chain<DF32, true>,
      (const void*)k_chain<DF32, false>, (const void*)k_chain<DBF16, true>, (const void*)k_chain<DBF16, false>,
      (const void*)k_chain<DF64W, true>, (const void*)k_chain<DF64W, false>, (const void*)k_ranges<true>,
      (const void*)k_ranges<false>, (const void*)k_fanout, (const void*)k_fanout_bulk,
      (const void*)k_agree_partial, (const void*)k_agree_final, (const void*)k_corrupt, (const void*)k_mean_rows,
      (const void*)k_fill_shards<DF32>, (const void*)k_fill_shards<DBF16>, (const void*)k_fill_shards<DF64W>};
  for (const void* f : fns) {
    cudaFuncAttributes at;
    cudaError_t e = cudaFuncGetAttributes(&at, f);
    if (e != cudaSuccess) return cuda_fail(e, "bfly_preload");
  }
  return BFLY_OK;
}

int bfly_fill_shards(const uint8_t* d_status, const uint8_t* d_mask, const double* d_fallback, void* const* d_dst,
                     int32_t n_dst, int32_t dtype, int64_t payload_len, int64_t n_shards, void* stream) {
  if (!d_status || !d_mask || n_dst < 0 || (n_dst > 0 && !d_dst) || n_shards < 1 || payload_len < n_shards)
    return fail(BFLY_E_INVALID_ARG, "bad fill-shards arguments");
  if (n_dst == 0) return BFLY_OK;
  Bounds bnd;
  bnd.init(payload_len, n_shards);
  const int64_t cps = (bnd.base + (bnd.rem ? 1 : 0) + kChunk - 1) / kChunk;
  int64_t grid = n_shards * cps;
  if (grid > (int64_t)sm_count()) grid = (int64_t)sm_count();
  const size_t smem = sizeof(void*) * (size_t)n_dst;
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case BFLY_F32:
      k_fill_shards<DF32><<<(unsigned)grid, kThreads, smem, st>>>(d_status, d_mask, d_fallback, d_dst, n_dst, bnd, cps);
      break;
    case BFLY_BF16:
      k_fill_shards<DBF16><<<(unsigned)grid, kThreads, smem, st>>>(d_status, d_mask, d_fallback, d_dst, n_dst, bnd, cps);
      break;
    case BFLY_F64WIRE:
      k_fill_shards<DF64W><<<(unsigned)grid, kThreads, smem, st>>>(d_status, d_mask, d_fallback, d_dst, n_dst, bnd, cps);
      break;
    default: return fail(BFLY_E_INVALID_ARG, "bad dtype");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_fill_shards launch");
  return BFLY_OK;
}

int bfly_chain_step(const void* const* d_src, int32_t n_src, int32_t dtype, const double* d_acc_in,
                    double* d_acc_out, int64_t begin, int64_t end, void* stream) {
  if (n_src < 0 || (n_src > 0 && !d_src) || !d_acc_out || begin < 0 || end < begin)
    return fail(BFLY_E_INVALID_ARG, "bad chain-step arguments");
  if (end == begin) return BFLY_OK;
  cudaStream_t st = (cudaStream_t)stream;
  auto go = [&](auto kern, int K, bool bulk) {
    const int64_t tile = (int64_t)kThreads * K;
    int64_t grid = (end + tile - 1) / tile - begin / tile;
    if (grid > (int64_t)sm_count() * 8) grid = (int64_t)sm_count() * 8;
    grid = cap_grid(grid);
    size_t smem = (sizeof(void*) * (size_t)n_src + 127) & ~(size_t)127;
    if (bulk) smem += 2 * sizeof(double) * (size_t)tile;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<(unsigned)grid, kThreads, smem, st>>>(d_src, n_src, d_acc_in, d_acc_out, begin, end);
  };
  const bool bulk = kChainBulk;
  switch (dtype) {
    case BFLY_F32: bulk ? go(k_chain<DF32, true>, DF32::K, true) : go(k_chain<DF32, false>, DF32::K, false); break;
    case BFLY_BF16:
      bulk ? go(k_chain<DBF16, true>, DBF16::K, true) : go(k_chain<DBF16, false>, DBF16::K, false);
      break;
    case BFLY_F64WIRE:
      bulk ? go(k_chain<DF64W, true>, DF64W::K, true) : go(k_chain<DF64W, false>, DF64W::K, false);
      break;
    default: return fail(BFLY_E_INVALID_ARG, "bad dtype");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_chain_step launch");
  return BFLY_OK;
}

int bfly_copy_ranges(const void* d_full, void* d_packed, void* const* d_dst, int32_t n_dst, const int64_t* d_ranges,
                     int32_t n_ranges, int32_t elem_size, int32_t scatter, void* stream) {
  if (n_ranges < 0 || n_ranges > 65535 || (elem_size != 2 && elem_size != 4 && elem_size != 8) || !d_packed ||
      (!scatter && !d_full) || (scatter && n_dst > 0 && !d_dst))
    return fail(BFLY_E_INVALID_ARG, "bad copy-ranges arguments");
  if (n_ranges == 0 || (scatter && n_dst == 0)) return BFLY_OK;
  const dim3 grid(32, (unsigned)n_ranges);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = sizeof(void*) * (size_t)(n_dst > 0 ? n_dst : 1);
  if (scatter)
    k_ranges<true><<<grid, kThreads, smem, st>>>((const unsigned char*)d_full, (unsigned char*)d_packed,
                                                 (unsigned char* const*)d_dst, n_dst, d_ranges, elem_size);
  else
    k_ranges<false><<<grid, kThreads, smem, st>>>((const unsigned char*)d_full, (unsigned char*)d_packed,
                                                  (unsigned char* const*)d_dst, n_dst, d_ranges, elem_size);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_copy_ranges launch");
  return BFLY_OK;
}

int bfly_fanout(const void* d_src, void* const* d_dst, int32_t n_dst, int64_t nbytes, void* stream) {
  if (!d_src || n_dst < 0 || (n_dst > 0 && !d_dst) || nbytes < 0) return fail(BFLY_E_INVALID_ARG, "bad fanout arguments");
  if (n_dst == 0 || nbytes == 0) return BFLY_OK;
  if (kFanoutBulk) {
    int64_t grid = nbytes / kFanTile;
    if (grid > (int64_t)sm_count() * 3) grid = (int64_t)sm_count() * 3;
    grid = cap_grid(grid);
    const size_t smem = 2 * kFanTile + sizeof(void*) * (size_t)n_dst;
    cudaFuncSetAttribute(k_fanout_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_fanout_bulk<<<(unsigned)grid, kThreads, smem, (cudaStream_t)stream>>>(d_src, d_dst, n_dst, nbytes);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "bfly_fanout launch");
    return BFLY_OK;
  }
  int64_t grid = (nbytes / 32 + kThreads - 1) / kThreads;
  if (grid > (int64_t)sm_count() * 8) grid = (int64_t)sm_count() * 8;
  grid = cap_grid(grid);
  if (grid < 1) grid = 1;
  k_fanout<<<(unsigned)grid, kThreads, sizeof(void*) * (size_t)n_dst, (cudaStream_t)stream>>>(d_src, d_dst, n_dst,
                                                                                             nbytes);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_fanout launch");
  return BFLY_OK;
}

int bfly_agreement(const double* d_a, const double* d_b, int64_t len, double tol, double* d_out,
                   void* d_scratch, size_t scratch_bytes, void* stream) {
  const int64_t nchunks = len > 0 ? (len + kChunk - 1) / kChunk : 0;
  if (nchunks > 0 && (!d_scratch || scratch_bytes < sizeof(double) * 4 * (size_t)nchunks))
    return fail(BFLY_E_INVALID_ARG, "scratch too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (nchunks > 0) k_agree_partial<<<(unsigned)nchunks, kThreads, 0, st>>>(d_a, d_b, len, (double*)d_scratch);
  k_agree_final<<<1, 32, 0, st>>>((const double*)d_scratch, nchunks, tol, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_agreement launch");
  return BFLY_OK;
}

int bfly_apply_corruption(const bfly_corruption_t* h_desc, const double* d_in, int64_t start_elem, int64_t len,
                          double* d_out, void* stream) {
  if (!h_desc || len < 0) return fail(BFLY_E_INVALID_ARG, "bad corruption arguments");
  if (h_desc->kind == BFLY_CORR_HOST) return fail(BFLY_E_INVALID_ARG, "host copies are not device-computable");
  if (len == 0) return BFLY_OK;
  int64_t grid = (len + 255) / 256;
  if (grid > 65535) grid = 65535;
  k_corrupt<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(*h_desc, d_in, start_elem, len, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_apply_corruption launch");
  return BFLY_OK;
}

int bfly_mean_rows(const double* d_stack, int32_t n_rows, int64_t width, double* d_out, void* stream) {
  if (n_rows <= 0 || width < 0) return fail(BFLY_E_INVALID_ARG, "bad stack shape");
  if (width == 0) return BFLY_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t grid = (width + 255) / 256;
  if (grid > 65535) grid = 65535;
  k_mean_rows<<<(unsigned)grid, 256, 0, st>>>(d_stack, n_rows, width, d_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bfly_mean_rows launch");
  return BFLY_OK;
}

}  // extern "C"
