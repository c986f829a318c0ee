// bfly_plan.cu — the shard index map (plan_shards, butterfly.py:84-114) on the
// host and on the device, plus the library's error plumbing.
//
// Device plan: one CTA.  The Fisher-Yates walk of Generator.permutation is
// inherently sequential (each swap depends on the previous ones and the number
// of Philox draws consumed depends on the rejections), but the Philox stream is
// counter-based: all threads fill a shared-memory buffer of 64-bit words in
// parallel, then one thread walks the permutation consuming 32-bit halves in
// numpy's order, and the batch is refilled when exhausted.  The permutation
// lives in shared memory while it fits (S <= 49152), else in global memory.
// Unranking combination ids into miner tuples is parallel.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <string>

#include "bfly_internal.cuh"
#include "sha256.h"

namespace bfly {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(BFLY_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static int check_plan_args(int32_t n, int32_t r, int64_t P, int64_t* S_out) {
  if (n < 2) return fail(BFLY_E_TOO_FEW_MINERS, "need at least 2 miners, got " + std::to_string(n));
  if (r < 2 || r > n) return fail(BFLY_E_INVALID_ARG, "redundancy must be in [2, n], got " + std::to_string(r));
  const int64_t S = binom(n, r);
  if (S < 0 || S > 0x7fffffffLL) return fail(BFLY_E_INVALID_ARG, "too many shards");
  if (P < S)
    return fail(BFLY_E_DEGENERATE, "payload of " + std::to_string(P) + " elements cannot fill " +
                                       std::to_string(S) + " shards");
  *S_out = S;
  return BFLY_OK;
}

constexpr int kPlanThreads = 1024;
constexpr int kDrawWords = 4096;        // 64-bit Philox words per refill (32 KB)
constexpr int kSmemPermMax = 40960;     // int32 permutation entries kept in smem (160 KB)

// One CTA.  perm_g is used when S > kSmemPermMax.
__global__ void __launch_bounds__(kPlanThreads)
    k_plan(int32_t n, int32_t r, int64_t S, uint64_t k0, uint64_t k1, int64_t* __restrict__ d_perm,
           int32_t* __restrict__ d_assign, int32_t* __restrict__ perm_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* words = reinterpret_cast<uint64_t*>(smem);
  int32_t* perm = S <= kSmemPermMax ? reinterpret_cast<int32_t*>(words + kDrawWords) : perm_g;
  __shared__ int64_t s_i;        // Fisher-Yates cursor
  __shared__ uint64_t s_word;    // next unread word index in the stream
  __shared__ int s_has32;
  __shared__ uint32_t s_saved;

  for (int64_t i = threadIdx.x; i < S; i += blockDim.x) perm[i] = (int32_t)i;
  if (threadIdx.x == 0) {
    s_i = S - 1;
    s_word = 0;
    s_has32 = 0;
    s_saved = 0;
  }
  __syncthreads();
  while (s_i >= 1) {
    const uint64_t blk0 = s_word >> 2;  // refill whole Philox blocks from the one holding s_word
    for (int b = threadIdx.x; b < kDrawWords / 4; b += blockDim.x) {
      Philox4x64 c;
      c.v[0] = blk0 + (uint64_t)b + 1;  // numpy pre-increments: word w lives in block w/4 + 1
      c.v[1] = c.v[2] = c.v[3] = 0;
      Philox4x64 o = philox4x64_10(c, k0, k1);
      words[4 * b + 0] = o.v[0];
      words[4 * b + 1] = o.v[1];
      words[4 * b + 2] = o.v[2];
      words[4 * b + 3] = o.v[3];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t i = s_i;
      int pos = (int)(s_word & 3);
      int has32 = s_has32;
      uint32_t saved = s_saved;
      while (i >= 1) {
        const uint32_t mask = (uint32_t)smear_mask((uint64_t)i);
        uint32_t draw;
        if (has32) {
          has32 = 0;
          draw = saved;
        } else {
          if (pos == kDrawWords) break;  // refill, then resume at the same i
          const uint64_t w = words[pos++];
          has32 = 1;
          saved = (uint32_t)(w >> 32);
          draw = (uint32_t)w;
        }
        const uint32_t v = draw & mask;
        if (v > (uint64_t)i) continue;  // rejected draw
        const int32_t t = perm[i];
        perm[i] = perm[v];
        perm[v] = t;
        --i;
      }
      s_i = i;
      s_word = (blk0 << 2) + (uint64_t)pos;
      s_has32 = has32;
      s_saved = saved;
    }
    __syncthreads();
  }
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
    const int32_t rank = perm[s];
    if (d_perm) d_perm[s] = rank;
    int32_t members[kMaxR > 8 ? kMaxR : 8];
    unrank_combination(n, r, rank, members);
    for (int k = 0; k < r; ++k) d_assign[s * r + k] = members[k];
  }
}

}  // namespace bfly

using namespace bfly;

// Generator.permutation(n) of RngStream(seed, ...) keyed (k0, k1): Fisher-Yates from
// i = n-1 down to 1 with numpy's random_interval draws (simkernel.py:237-238).
static void fisher_yates_host(int64_t n, uint64_t k0, uint64_t k1, int32_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  PhiloxStream st;
  st.init(k0, k1);
  for (int64_t i = n - 1; i >= 1; --i) {
    const int64_t j = (int64_t)random_interval(st, (uint64_t)i);
    const int32_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
}

extern "C" {

const char* bfly_version(void) { return "bfly 0.1.0 (sm_100a)"; }
const char* bfly_last_error(void) { return g_error.c_str(); }

int64_t bfly_n_shards(int32_t n_miners, int32_t redundancy) {
  if (redundancy < 0 || n_miners < 0) return -1;
  return binom(n_miners, redundancy);
}

int bfly_philox_key(const char* seed_decimal, const char* stream_id, uint64_t out_key[2]) {
  if (!seed_decimal || !stream_id || !out_key) return fail(BFLY_E_INVALID_ARG, "null argument");
  Sha256 h;
  h.update(reinterpret_cast<const uint8_t*>(seed_decimal), strlen(seed_decimal));
  const uint8_t sep = 0x1f;
  h.update(&sep, 1);
  h.update(reinterpret_cast<const uint8_t*>(stream_id), strlen(stream_id));
  uint8_t d[32];
  h.digest(d);
  for (int w = 0; w < 2; ++w) {
    uint64_t v = 0;
    for (int b = 7; b >= 0; --b) v = (v << 8) | d[8 * w + b];  // little-endian u64
    out_key[w] = v;
  }
  return BFLY_OK;
}

int bfly_permutation_host(int64_t n, uint64_t k0, uint64_t k1, int64_t* h_out) {
  if (n < 0 || (n > 0 && !h_out)) return fail(BFLY_E_INVALID_ARG, "bad permutation arguments");
  if (n > INT32_MAX) return fail(BFLY_E_UNSUPPORTED, "permutation too long");
  int32_t* perm = new int32_t[n > 0 ? n : 1];
  fisher_yates_host(n, k0, k1, perm);
  for (int64_t i = 0; i < n; ++i) h_out[i] = perm[i];
  delete[] perm;
  return BFLY_OK;
}

int bfly_plan_host(int32_t n, int32_t r, int64_t P, uint64_t k0, uint64_t k1, int32_t* h_assign,
                   int64_t* h_bounds) {
  int64_t S;
  int rc = check_plan_args(n, r, P, &S);
  if (rc) return rc;
  if (r > 16) return fail(BFLY_E_INVALID_ARG, "redundancy too large");
  int32_t* perm = new int32_t[S];
  fisher_yates_host(S, k0, k1, perm);
  int32_t members[16];
  for (int64_t s = 0; s < S; ++s) {
    unrank_combination(n, r, perm[s], members);
    for (int k = 0; k < r; ++k) h_assign[s * r + k] = members[k];
  }
  delete[] perm;
  Bounds b;
  b.init(P, S);
  for (int64_t s = 0; s <= S; ++s) h_bounds[s] = s < S ? b.start(s) : P;
  return BFLY_OK;
}

int bfly_plan_device(int32_t n, int32_t r, int64_t P, uint64_t k0, uint64_t k1, int64_t* d_perm,
                     int32_t* d_assign, void* stream) {
  int64_t S;
  int rc = check_plan_args(n, r, P, &S);
  if (rc) return rc;
  if (r > 8) return fail(BFLY_E_UNSUPPORTED, "device plan supports r <= 8");
  int32_t* perm_g = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (S > kSmemPermMax) {
    e = cudaMallocAsync(&perm_g, sizeof(int32_t) * S, st);
    if (e != cudaSuccess) return cuda_fail(e, "bfly_plan_device alloc");
  }
  const size_t smem = sizeof(uint64_t) * kDrawWords + (S <= kSmemPermMax ? sizeof(int32_t) * S : 0);
  e = cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "bfly_plan_device attr");
  k_plan<<<1, kPlanThreads, smem, st>>>(n, r, S, k0, k1, d_perm, d_assign, perm_g);
  e = cudaGetLastError();
  if (perm_g) cudaFreeAsync(perm_g, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_plan launch");
  return BFLY_OK;
}

}  // extern "C"
