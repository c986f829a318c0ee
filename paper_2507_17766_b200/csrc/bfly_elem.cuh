// bfly_elem.cuh — element types and streaming helpers shared by the merge kernels
// (bfly_merge.cu) and the persistent multi-GPU ring kernel (bfly_ring.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bfly {

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------

// 256-bit (32-byte) global accesses — new on sm_100: one LDG.256 / STG.256 per
// thread per replica halves the load/store instruction count of 128-bit code.
struct V8 {
  uint32_t w[8];
};

__device__ __forceinline__ V8 ld_stream(const void* p) {
  V8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                 "=r"(r.w[6]), "=r"(r.w[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, const V8& v) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
               "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
               : "memory");
}
__device__ __forceinline__ void st_f64x4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// fp32 wire values, fp64 accumulation (the reference path).
struct DF32 {
  static constexpr int K = 8;  // elements per 32-byte vector
  using Acc = double;
  __device__ static Acc zero() { return 0.0; }
  __device__ static Acc load(const void* p, int64_t e) { return (double)__ldg((const float*)p + e); }
  __device__ static double raw(const void* p, int64_t e) { return (double)((const float*)p)[e]; }
  __device__ static void unpack(const V8& v, Acc* x) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (double)__uint_as_float(v.w[k]);
  }
  __device__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ static Acc mean(Acc s, int n) { return __ddiv_rn(s, (double)n); }
  __device__ static double widen(Acc m) { return m; }
  __device__ static void store(void* p, int64_t e, double v) { ((float*)p)[e] = __double2float_rn(v); }
  __device__ static V8 pack(const Acc* m) {
    V8 v;
#pragma unroll
    for (int k = 0; k < 8; ++k) v.w[k] = __float_as_uint(__double2float_rn(m[k]));
    return v;
  }
  __device__ static void store8(void* p, int64_t e0, const double* v) {  // 32 B, aligned
    st_stream((float*)p + e0, pack_d(v));
  }
  __device__ static V8 pack_d(const double* v) {  // K doubles -> one vector, as store() rounds
    V8 w;
#pragma unroll
    for (int k = 0; k < 8; ++k) w.w[k] = __float_as_uint(__double2float_rn(v[k]));
    return w;
  }
  __device__ static void unpack_raw(const V8& v, double* x) {  // stored values, exactly
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (double)__uint_as_float(v.w[k]);
  }
};

// bf16 replicas, fp32 accumulation (extension, BASELINE config 4).
struct DBF16 {
  static constexpr int K = 16;
  using Acc = float;
  __device__ static Acc zero() { return 0.0f; }
  __device__ static float bf(uint32_t bits16) { return __uint_as_float(bits16 << 16); }
  __device__ static Acc load(const void* p, int64_t e) {
    return bf(((const unsigned short*)p)[e]);
  }
  __device__ static double raw(const void* p, int64_t e) { return (double)load(p, e); }
  __device__ static void unpack(const V8& v, Acc* x) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[2 * k] = __uint_as_float(v.w[k] << 16);
      x[2 * k + 1] = __uint_as_float(v.w[k] & 0xffff0000u);
    }
  }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
  __device__ static Acc mean(Acc s, int n) { return __fdiv_rn(s, (float)n); }
  __device__ static double widen(Acc m) { return (double)m; }
  __device__ static unsigned short to_bits(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<unsigned short*>(&h);
  }
  __device__ static void store(void* p, int64_t e, double v) {
    ((unsigned short*)p)[e] = to_bits(__double2float_rn(v));
  }
  __device__ static V8 pack(const Acc* m) {
    V8 v;
#pragma unroll
    for (int k = 0; k < 8; ++k) v.w[k] = (uint32_t)to_bits(m[2 * k]) | ((uint32_t)to_bits(m[2 * k + 1]) << 16);
    return v;
  }
  __device__ static void store8(void* p, int64_t e0, const double* v) {  // 16 B, aligned
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = (uint32_t)to_bits(__double2float_rn(v[2 * k])) |
             ((uint32_t)to_bits(__double2float_rn(v[2 * k + 1])) << 16);
    *reinterpret_cast<uint4*>((unsigned short*)p + e0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ static V8 pack_d(const double* v) {
    V8 w;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      w.w[k] = (uint32_t)to_bits(__double2float_rn(v[2 * k])) |
               ((uint32_t)to_bits(__double2float_rn(v[2 * k + 1])) << 16);
    return w;
  }
  __device__ static void unpack_raw(const V8& v, double* x) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[2 * k] = (double)__uint_as_float(v.w[k] << 16);
      x[2 * k + 1] = (double)__uint_as_float(v.w[k] & 0xffff0000u);
    }
  }
};

// fp64 payloads rounded to the fp32 wire on load (astype("<f4"), butterfly.py:213,230).
struct DF64W {
  static constexpr int K = 4;
  using Acc = double;
  __device__ static Acc zero() { return 0.0; }
  __device__ static Acc load(const void* p, int64_t e) {
    return (double)__double2float_rn(__ldg((const double*)p + e));
  }
  __device__ static double raw(const void* p, int64_t e) { return ((const double*)p)[e]; }
  __device__ static void unpack(const V8& v, Acc* x) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      x[k] = (double)__double2float_rn(__hiloint2double((int)v.w[2 * k + 1], (int)v.w[2 * k]));
  }
  __device__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
  __device__ static Acc mean(Acc s, int n) { return __ddiv_rn(s, (double)n); }
  __device__ static double widen(Acc m) { return m; }
  __device__ static void store(void* p, int64_t e, double v) { ((double*)p)[e] = v; }
  __device__ static V8 pack(const Acc* m) {
    V8 v;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v.w[2 * k] = (uint32_t)__double2loint(m[k]);
      v.w[2 * k + 1] = (uint32_t)__double2hiint(m[k]);
    }
    return v;
  }
  __device__ static void store8(void* p, int64_t e0, const double* v) {  // 64 B, aligned
    st_f64x4((double*)p + e0, v[0], v[1], v[2], v[3]);
    st_f64x4((double*)p + e0 + 4, v[4], v[5], v[6], v[7]);
  }
  __device__ static V8 pack_d(const double* v) { return pack(v); }
  __device__ static void unpack_raw(const V8& v, double* x) {  // the fp64 payload, unrounded
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __hiloint2double((int)v.w[2 * k + 1], (int)v.w[2 * k]);
  }
};


// Sequential accumulation of one 32-byte vector per thread over the replica
// table, U replicas' loads in flight before their adds (the add order stays
// ascending, which is what parity needs).  FIRST: also hand back replica 0's raw
// 32 bytes (the fallback source of special shards: no second load of them).
template <class D, int U = 4, bool NO_OUTER_UNROLL = false, bool FIRST = false>
__device__ __forceinline__ void accumulate_vec(typename D::Acc (&acc)[D::K], const void* const* s_src, int n,
                                               int64_t vidx, V8* first = nullptr) {
  constexpr int K = D::K;
  int q = 0;
  if constexpr (FIRST) {
    if (n > 0) {  // replica 0 alone, kept; the rest as below
      *first = ld_stream(reinterpret_cast<const V8*>(s_src[0]) + vidx);
      typename D::Acc x[K];
      D::unpack(*first, x);
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = D::add(acc[k], x[k]);
      q = 1;
    }
  }
  if constexpr (NO_OUTER_UNROLL) {
#pragma unroll 1
    for (; q + U <= n; q += U) {
      V8 raw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) raw[u] = ld_stream(reinterpret_cast<const V8*>(s_src[q + u]) + vidx);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        typename D::Acc x[K];
        D::unpack(raw[u], x);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = D::add(acc[k], x[k]);
      }
    }
  }
  for (; q + U <= n; q += U) {
    V8 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) raw[u] = ld_stream(reinterpret_cast<const V8*>(s_src[q + u]) + vidx);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      typename D::Acc x[K];
      D::unpack(raw[u], x);
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = D::add(acc[k], x[k]);
    }
  }
  for (; q < n; ++q) {
    typename D::Acc x[K];
    D::unpack(ld_stream(reinterpret_cast<const V8*>(s_src[q]) + vidx), x);
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = D::add(acc[k], x[k]);
  }
}

// acc[k] <- incoming chain accumulator (fp64 storage; fp32 value for bf16)
template <class D>
__device__ __forceinline__ void load_acc_in(typename D::Acc (&acc)[D::K], const double* a) {
#pragma unroll
  for (int k = 0; k < D::K; k += 4) {
    double x0, x1, x2, x3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3)
                 : "l"(a + k));
    acc[k] = (typename D::Acc)x0;
    acc[k + 1] = (typename D::Acc)x1;
    acc[k + 2] = (typename D::Acc)x2;
    acc[k + 3] = (typename D::Acc)x3;
  }
}

// Copies the pointer tables to shared memory; returns whether every pointer the
// vector path touches is 32-byte aligned.
__device__ __forceinline__ bool stage_pointers(const void** s_src, void** s_dst, const void* const* src, int n_src,
                                               void* const* dst, int n_dst, uintptr_t extra) {
  uintptr_t mis = threadIdx.x == 0 ? extra : 0;
  for (int q = threadIdx.x; q < n_src; q += blockDim.x) {
    s_src[q] = src[q];
    mis |= (uintptr_t)src[q];
  }
  for (int q = threadIdx.x; q < n_dst; q += blockDim.x) {
    s_dst[q] = dst[q];
    mis |= (uintptr_t)dst[q];
  }
  return __syncthreads_or((int)(mis & 31)) == 0;
}


}  // namespace bfly
