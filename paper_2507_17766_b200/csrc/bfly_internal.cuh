// bfly_internal.cuh — shared internals of libbfly (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bfly.h"
#include "bfly_index.cuh"

namespace bfly {

// thread-local error text behind bfly_last_error()
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
int sm_count();

// Per-shard class computed by the classify kernel.
enum ShardClass : uint8_t {
  kFast = 0,     // >= 1 survivor, all survivors honest: mean is final (status merged)
  kSpecial = 1,  // >= 1 corrupted survivor: compare copies, adopt or fall back
  kLost = 2,     // no survivor: fallback (butterfly.py:264-273)
};

// Outcome of a special / lost shard as k_classify predicts it, assuming honest copies
// agree and corrupted ones disagree with everything: k_reduce writes the predicted
// final value straight away and k_apply only revisits shards that came out otherwise.
enum ShardPred : uint8_t {
  kPredNone = 0,      // no guess (lone corrupted survivor, or fallback source overwritten in place)
  kPredMean = 1,      // an honest majority adopts the mean
  kPredFallback = 2,  // no majority (or no survivor): fallback values
  kPredMask = 3,
  kPredFuse = 0x80,   // flag: two device-computable copies, k_reduce accumulates their statistics
};

constexpr int kMaxR = 3;            // device path supports r = 2 (reference) and 3 (extension)
constexpr int kThreads = 256;       // CTA size of the streaming kernels
constexpr int kChunk = 16384;       // elements per CTA in k_apply
constexpr int kMinStatTile = kThreads * 4;  // smallest statistics tile (fp64 payloads)

struct ScratchLayout {
  int64_t S = 0, cps = 0;
  int npairs = 0;
  int64_t ntiles = 0;  // statistics tiles of the smallest size
  size_t off_cls = 0, off_pred = 0, off_done = 0, off_source = 0, off_stats = 0, off_scores = 0, off_has = 0, off_inv = 0,
         off_nonfin = 0;
  size_t total = 0;
  void init(int32_t n, int32_t r, int64_t P) {
    S = binom(n, r);
    npairs = r * (r - 1) / 2;
    Bounds b;
    b.init(P, S > 0 ? S : 1);
    const int64_t maxlen = b.base + (b.rem ? 1 : 0);
    cps = (maxlen + kChunk - 1) / kChunk;
    if (cps < 1) cps = 1;
    auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o = 0;
    off_cls = o;
    o = align(o + (size_t)S);
    off_pred = o;
    o = align(o + (size_t)S);
    ntiles = P / kMinStatTile + 1;
    off_done = o;
    o = align(o + (size_t)ntiles);
    off_source = o;
    o = align(o + sizeof(int32_t) * (size_t)S);
    off_stats = o;
    // one partial per (shard, statistics tile it overlaps): slot = tile + shard
    o = align(o + sizeof(double) * 4 * (size_t)(ntiles + S) * (size_t)npairs);
    off_scores = o;
    o = align(o + sizeof(double) * (size_t)S * (size_t)npairs);
    off_has = o;
    o = align(o + (size_t)S * (size_t)npairs);
    off_inv = o;
    o = align(o + sizeof(int32_t) * (size_t)S);
    // non-finite means of fast shards: a u32 "any" word, a u32 "some shard is special or
    // lost" word (k_classify), a u32 "some shard needs k_apply" word (k_classify /
    // k_decide), padding, then one byte per shard
    off_nonfin = o;
    o = align(o + 16 + (size_t)S);
    total = o;
  }
};

// What the persistent ring's last rank needs to write predicted outcomes for special /
// lost shards (filled by ring_round_setup from the merge arguments).
struct RingSpecial {
  const uint8_t* cls = nullptr;   // ShardClass per shard
  const uint8_t* pred = nullptr;  // ShardPred per shard
  Bounds bnd{};
  double* ws = nullptr;           // means of special shards (may alias merged)
  const double* fallback = nullptr;
  const void* fb_src = nullptr;   // replica supplying fallback values
  bool merged_apart = false;      // merged is not the workspace
  uint32_t* nonfin_any = nullptr; // some fast shard's mean is not finite (then nonfin[s] = 1)
  uint8_t* nonfin = nullptr;
  // pair statistics of special tiles accumulated inside the kernel (kPredFuse shards,
  // whole tiles of one shard): one partial per (shard, tile) slot, done[tile] = 1
  const int32_t* assign = nullptr;
  const bfly_corruption_t* corr = nullptr;
  double* stats = nullptr;
  uint8_t* done = nullptr;
  int64_t stile = 0;
};

// An IEEE double that is neither NaN nor +-Inf (exponent field not all ones).
__device__ __forceinline__ bool finite64(double x) {
  return (__double_as_longlong(x) & 0x7ff0000000000000LL) != 0x7ff0000000000000LL;
}
int ring_round_setup(const bfly_merge_args_t* a, void* stream, RingSpecial* out);

}  // namespace bfly
