// bfly_ring.cu — the multi-GPU merge round as ONE persistent, TMA-driven kernel per GPU.
//
// The reference reduces every shard over all miners in one process in ascending
// miner order (butterfly.py:216-240, mean_reducer :156-158).  With the miners in
// contiguous blocks over G GPUs that order is kept exactly by carrying the fp64
// running sums from GPU to GPU (chain g = 0 .. G-1), dividing on the last GPU and
// relaying the final values round the ring (last -> 0 -> 1 -> ... -> G-2) into every
// replica (the scatter-back, orchestrator.py:581-590).
//
// k_ring runs that whole round in one launch, tile by tile:
//   * the payload is cut into tiles of TE elements (4 KB of each replica); lane c
//     (= CTA c, one per SM) of rank g exchanges only with lane c of its neighbours.
//     Rank 0 deals the tiles dynamically — each step of a lane takes the next tile
//     from a counter — and writes the tile id ahead into every other rank's schedule
//     ring and into the header of every slot it sends, so lane c of every rank
//     processes the same tiles in the same order; a lane on a slower SM simply takes
//     fewer.  A tile id of -1 ends the lane's round;
//   * per CTA, warp-specialised and asynchronous:
//       LOADER warp   TMA bulk loads (cp.async.bulk ... mbarrier::complete_tx) of the
//                     replica tiles (as soon as the schedule names the tile) and of
//                     the incoming running sums into rings of shared-memory stages;
//       8 COMPUTE warps  read the stages, fp64 adds in ascending miner order (the
//                     last rank also divides), write the outgoing tile to shared memory;
//       STORER warp   TMA bulk stores of that tile (with its header) into the next
//                     rank's inbox slot over NVLink (and, on the last rank, into every
//                     local replica);
//       RELAY warps   (ranks < last) a bulk load of the final tile from the inbox and
//                     bulk stores into every local replica and the successor's inbox:
//                     the scatter-back without a single SM load or store;
//       PUBLISHER     the system-scope releases of the `ready` flags;
//   * each rank's inboxes are NB-slot rings per lane in its IPC region; producer and
//     consumer order themselves with 64-bit monotonic counters (ready / free) in the
//     waiter's region: `ready` is released (st.release.sys) once the bulk group has
//     landed, the consumer polls with ld.acquire.sys and returns the slot (`free`) as
//     soon as its contents are in shared memory.  Step counts are persisted per lane,
//     so the counters stay monotonic across rounds.  No kernel launches, stream memory
//     operations or host round trips per tile: NVLink transfers of tile i overlap the
//     HBM stream of tile i+1 and the ring fills in G tile steps.  The inboxes
//     (L x NB x 12 KB) stay small enough to live in L2.
// Deadlock freedom: every wait of step j points at step j of an earlier stage of the
// path (chain 0..last, relay 0..last-1) or at step j - NB; the chain and the relay of a
// lane run in different warps, and all CTAs are co-resident (cooperative launch).  A
// CPU model of the protocol runs under random interleavings for G = 2..8
// (tests/test_ring_protocol.py).  Every wait traps after kRingTimeoutNs instead of
// hanging the GPU.
//
// Corrupted / lost shards (p.special, last rank): their tiles leave with the outcome
// k_classify predicts (the means go to the workspace); FINISH decides those shards after
// the kernel and the host re-broadcasts the few decided otherwise (multigpu.py).
#include <cuda_runtime.h>

#include "bfly_elem.cuh"
#include "bfly_internal.cuh"
#include "bfly_stats.cuh"

namespace bfly {

enum FusedFlag : int { kFAccReady = 0, kFAccFree = 1, kFFinReady = 2, kFFinFree = 3, kFAbort = 4 };
constexpr unsigned long long kRingTimeoutNs = 20ull * 1000 * 1000 * 1000;
constexpr int kRingCompute = kThreads;        // 8 compute warps
constexpr int kRingThreads = kThreads + 160;  // + loader, storer, relay loader, relay storer, publisher
constexpr int kWLoad = kThreads / 32, kWStore = kWLoad + 1, kWRLoad = kWLoad + 2, kWRStore = kWLoad + 3,
              kWPub = kWLoad + 4;
constexpr int kNS = 4;            // replica stages
constexpr int kRB = 8;            // replica tiles per stage
constexpr int kNR = 4;            // relay stages
constexpr int kNO = 4;            // outgoing-tile stages
constexpr int kNA = 4;            // incoming running-sum stages
constexpr int kNT = 8;            // chain steps the loader may lead the storer by (tile-id ring)
constexpr int kSR = 512;          // tile schedule ring per lane (rank 0 -> every other rank)
constexpr int kMaxG = 16;         // ranks the persistent ring supports
constexpr int kMaxLag = 3;        // a step is published p.lag (1..3) steps later, when its bytes have landed
constexpr int kTileBytes = 4096;  // one replica's share of a tile
constexpr int kNQ = 32;           // FUSE: special tiles the compute warps may lead the stats warps by
constexpr int kStatWarps = 2;     // FUSE: the last rank's (otherwise idle) relay warps

struct RingParams {
  int g, G, L, NB;
  int64_t P, T;  // elements, tiles
  unsigned char* my;     // own region
  unsigned char* nxt;    // chain target (g + 1), or rank 0 for the last rank
  unsigned char* prv;    // acc credits go here (g - 1); null on rank 0
  unsigned char* fsucc;  // relay successor (g + 1 < last), else null
  unsigned char* fpred;  // relay predecessor (last for rank 0, else g - 1)
  int64_t off_fin, off_flags, off_steps;
  unsigned long long* tile_ctr;  // rank 0: next tile of the round (zeroed before the launch)
  int64_t off_sched;             // per lane kSR schedule words: (step + 1) << 32 | (tile + 1)
  unsigned char* region[kMaxG];  // every rank's region (rank 0 writes the schedule into them)
  const void* const* src;
  int n_src;
  void* const* dst;
  int n_dst;
  int n_div;
  double* merged;
  unsigned long long* prof;  // diagnostics (BFLY_RING_PROFILE): wait cycles per CTA and counter
  int pub_every;             // publish every pub_every-th step (each publication covers the ones before)
  int lag;                   // publication lag in steps (1..kMaxLag)
  int special;               // last rank: some shard is corrupted or lost (see RingSpecial)
  RingSpecial sp;
};

template <class D>
struct RingGeom {
  static constexpr int ESIZE = 32 / D::K;       // bytes per replica element
  static constexpr int KE = 16 / ESIZE;         // elements per thread (16 B of each replica)
  static constexpr int TE = kRingCompute * KE;  // tile elements
  using Acc = typename D::Acc;                  // running sums travel at accumulator width
  static constexpr int ACC_BYTES = TE * (int)sizeof(Acc);
  static constexpr int FIN_BYTES = TE * ESIZE;  // == kTileBytes
  // an inbox slot / outgoing stage: a 16-byte header (the tile id) + the tile
  static constexpr int ACC_SLOT = 16 + ACC_BYTES;
  static constexpr int FIN_SLOT = 16 + FIN_BYTES;
  static constexpr int OUT_SLOT = ACC_SLOT;  // >= FIN_SLOT
  // shared memory: replica stages | 2 acc stages | out stages | relay stages | barriers,
  // tile rings, mailbox | pointers
  static constexpr int OFF_REP = 0;
  static constexpr int OFF_ACC = OFF_REP + kNS * kRB * kTileBytes;
  static constexpr int OFF_OUT = OFF_ACC + kNA * ACC_BYTES;
  static constexpr int OFF_REL = OFF_OUT + kNO * OUT_SLOT;
  static constexpr int OFF_BAR = OFF_REL + kNR * FIN_SLOT;
  static constexpr int N_BAR = 2 * kNS + 2 * kNA + 2 * kNO + 2 * kNR + 2 * kNT;
  // FUSE: the stats queue (compute warps -> the last rank's stats warps): kNQ full
  // barriers, kNQ (tile, shard) entries, progress + admit words, the stats partials (x2)
  static constexpr int OFF_STAT = OFF_BAR + 8 * (N_BAR + kNT + kNR + 4);
  static constexpr int OFF_PTR = OFF_STAT + 24 * kNQ + 16 + 2 * kStatWarps * 32;
};

// ---------------------------------------------------------------------------
// flags, mbarriers, bulk copies
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t* flag_at(unsigned char* region, const RingParams& p, int f, int lane) {
  return reinterpret_cast<uint64_t*>(region + p.off_flags) + (int64_t)f * p.L + lane;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* a) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* a, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
// consumer -> producer: the slot has been loaded (its bulk load completed before the
// barrier this thread waited on), so no fence is needed
__device__ __forceinline__ void st_relaxed_sys(uint64_t* a, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
// Publish `v` (steps landed) to the consumer: a system-scope release.  The storer saw
// the bulk group complete (cp.async.bulk.wait_group + fence.proxy.async) and handed the
// count over through shared memory (CTA-scope release / acquire), so the release is
// cumulative over the data.  A relaxed store here was measured faster and is NOT safe:
// stale tiles showed up in an 8-round stress test.
__device__ __forceinline__ void publish(uint64_t* f, uint64_t v) { st_release_sys(f, v); }
// storer -> publisher warp: `v` steps have landed (CTA-scope release through shared memory)
__device__ __forceinline__ void mail_post(uint64_t* box, uint64_t v) {
  asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(box)), "l"(v)
               : "memory");
}
__device__ __forceinline__ uint64_t mail_read(const uint64_t* box) {
  uint64_t v;
  asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];"
               : "=l"(v)
               : "r"((unsigned)__cvta_generic_to_shared(box))
               : "memory");
  return v;
}

// Wait-cycle counters of one role (diagnostics only; p.prof == null in production).
constexpr int kProfSlots = 24;  // 5 roles x 4 counters, then CTA start / end (globaltimer)
struct Prof {
  unsigned long long* out;
  unsigned long long acc[4] = {0, 0, 0, 0};
  long long t = 0;
  __device__ explicit Prof(const RingParams& p, int first)
      : out(p.prof ? p.prof + blockIdx.x * kProfSlots + first : nullptr) {}
  __device__ __forceinline__ void start() {
    if (out) t = clock64();
  }
  __device__ __forceinline__ void stop(int k) {
    if (out) acc[k] += (unsigned long long)(clock64() - t);
  }
  __device__ __forceinline__ void flush() {
    if (out)
      for (int k = 0; k < 4; ++k) out[k] = acc[k];
  }
};

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __noinline__ void ring_abort(const RingParams& p) {
  volatile uint64_t* abort_word = flag_at(p.my, p, kFAbort, 0);
  *abort_word = 1;
  __threadfence_system();
  __trap();
}

// Wait until *f >= v, caching the last value read (the upstream usually runs ahead,
// so most steps need no load).  Traps when the ring stops making progress.
__device__ __forceinline__ void flag_wait(const RingParams& p, const uint64_t* f, uint64_t v, uint64_t& known) {
  if (known >= v) return;
  known = ld_acquire_sys(f);
  if (known < v) {
    const uint64_t t0 = global_ns();
    const volatile uint64_t* abort_word = flag_at(p.my, p, kFAbort, 0);
    while ((known = ld_acquire_sys(f)) < v) {
      __nanosleep(20);
      if (*abort_word || global_ns() - t0 > kRingTimeoutNs) ring_abort(p);
    }
  }
  // the bulk copies that follow (async proxy) are ordered after the acquire
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_addr(b)),
               "r"(bytes)
               : "memory");
}
// wait for the completion of the phase with the given parity
__device__ __forceinline__ void mbar_wait(const RingParams& p, uint64_t* b, unsigned parity) {
  uint64_t t0 = 0;
  for (int spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    if (done) return;
    if ((spin & 1023) == 1023) {
      const uint64_t t = global_ns();
      if (!t0)
        t0 = t;
      else if (t - t0 > kRingTimeoutNs)
        ring_abort(p);
    }
  }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_load_stream(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// shared -> global (a peer inbox slot, or a local replica with an evict-first hint)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_stream(void* gdst, const void* ssrc, unsigned bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int KEEP>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(KEEP) : "memory");
}
// every bulk group but the newest KEEP has landed; the flag publishing it may follow
template <int KEEP>
__device__ __forceinline__ void bulk_wait_landed() {
  asm volatile("cp.async.bulk.wait_group %0;\n\tfence.proxy.async.global;" ::"n"(KEEP) : "memory");
}
__device__ __forceinline__ void bulk_wait_landed_n(int keep) {
  if (keep <= 1)
    bulk_wait_landed<1>();
  else if (keep == 2)
    bulk_wait_landed<2>();
  else
    bulk_wait_landed<3>();
}

__device__ __forceinline__ unsigned round16(int64_t b) { return (unsigned)((b + 15) & ~(int64_t)15); }

template <class D>
__device__ __forceinline__ typename D::Acc* acc_slot(unsigned char* region, const RingParams& p, int lane, int slot) {
  return reinterpret_cast<typename D::Acc*>(region + ((int64_t)lane * p.NB + slot) * RingGeom<D>::ACC_SLOT);
}
template <class D>
__device__ __forceinline__ unsigned char* fin_slot(unsigned char* region, const RingParams& p, int lane, int slot) {
  return region + p.off_fin + ((int64_t)lane * p.NB + slot) * RingGeom<D>::FIN_SLOT;
}

// 16 bytes of one replica -> KE values / KE values -> 16 bytes (through the 32-byte
// helpers of bfly_elem.cuh; the unused half is dead code)
template <class D>
__device__ __forceinline__ void unpack16(const uint4& v, typename D::Acc* x) {
  V8 w;
  w.w[0] = v.x, w.w[1] = v.y, w.w[2] = v.z, w.w[3] = v.w;
  w.w[4] = w.w[5] = w.w[6] = w.w[7] = 0;
  typename D::Acc t[D::K];
  D::unpack(w, t);
#pragma unroll
  for (int k = 0; k < RingGeom<D>::KE; ++k) x[k] = t[k];
}
template <class D>
__device__ __forceinline__ uint4 pack16(const typename D::Acc* x) {
  typename D::Acc t[D::K];
#pragma unroll
  for (int k = 0; k < D::K; ++k) t[k] = k < RingGeom<D>::KE ? x[k] : D::zero();
  const V8 w = D::pack(t);
  return make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
}

// 16 bytes from KE doubles, rounded as the replicas store them
template <class D>
__device__ __forceinline__ uint4 pack16d(const double* v) {
  double t[D::K];
#pragma unroll
  for (int k = 0; k < D::K; ++k) t[k] = k < RingGeom<D>::KE ? v[k] : 0.0;
  const V8 w = D::pack_d(t);
  return make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
}

// Special / lost shards on the last rank (p.special): the shards [lo, hi] the tile at t0
// covers (a lane's tiles ascend, so the cursor only steps forward), and whether they are
// all fast.  (Shards are far longer than a tile: one or two of them.)
struct TileShards {
  int64_t lo, hi;
  bool fast;
};
__device__ __forceinline__ TileShards tile_shards(const RingParams& p, ShardCursor& cur, int64_t t0, int64_t te) {
  TileShards t;
  t.lo = cur.at(p.sp.bnd, t0);
  t.hi = cur.at(p.sp.bnd, min(t0 + te - 1, p.P - 1));
  t.fast = true;
  for (int64_t s = t.lo; s <= t.hi; ++s) t.fast = t.fast && p.sp.cls[s] == kFast;
  return t;
}

// Last rank: a whole tile that holds a shard predicted to fall back to the lowest alive
// miner's replica (usually on another GPU).  The loader bulk-loads that replica's tile
// over NVLink into a stage (the relay stages: the last rank has no relay) ahead of the
// compute warps, which would otherwise stall on a remote load per tile.
__device__ __forceinline__ bool fb_prefetch_on(const RingParams& p) {
  return p.special && p.g == p.G - 1 && !p.sp.fallback && p.sp.fb_src;
}
__device__ __forceinline__ bool tile_wants_fb(const RingParams& p, const TileShards& t) {
  bool want = false;
  for (int64_t s = t.lo; s <= t.hi; ++s)
    want = want || (p.sp.cls[s] != kFast && (p.sp.pred[s] & kPredMask) == kPredFallback);
  return want;
}

// The value element e leaves the last rank with, as k_reduce writes it (emit_predicted,
// bfly_merge.cu): the mean for fast shards and for shards predicted to adopt it, the
// fallback for shards predicted to fall back; a shard without a prediction carries the
// mean until FINISH rewrites it.  Means of special shards go to the workspace.
template <class D>
__device__ __forceinline__ double fallback_one(const RingParams& p, int64_t e) {
  return p.sp.fallback ? p.sp.fallback[e]
                       : (p.sp.fb_src ? D::raw(p.sp.fb_src, e) : __longlong_as_double(0x7ff8000000000000LL));
}

// KE fallback values from 16 raw bytes of a replica (dtype D), rounded as it stores them
template <class D>
__device__ __forceinline__ void fallback_unpack16(const uint4& w, double* fb) {
  V8 v;
  v.w[0] = w.x, v.w[1] = w.y, v.w[2] = w.z, v.w[3] = w.w;
  v.w[4] = v.w[5] = v.w[6] = v.w[7] = 0;
  double t[8 * 4 / RingGeom<D>::ESIZE > 0 ? 8 * 4 / RingGeom<D>::ESIZE : 1];
  D::unpack_raw(v, t);
#pragma unroll
  for (int k = 0; k < RingGeom<D>::KE; ++k) fb[k] = t[k];
}

// The fallback values of a thread's KE elements (from e0, 16-byte aligned in the replica),
// loaded at once: usually from the lowest alive miner's replica on another GPU, so one
// vector load over NVLink instead of KE dependent scalar ones.
template <class D>
__device__ __forceinline__ void fallback_vec16(const RingParams& p, int64_t e0, double* fb) {
  constexpr int KE = RingGeom<D>::KE;
  if (p.sp.fallback) {
#pragma unroll
    for (int k = 0; k < KE; ++k) fb[k] = p.sp.fallback[e0 + k];
  } else if (p.sp.fb_src) {
    uint32_t w[4];
    asm volatile("ld.global.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"((const unsigned char*)p.sp.fb_src + e0 * RingGeom<D>::ESIZE));
    V8 v;
    v.w[0] = w[0], v.w[1] = w[1], v.w[2] = w[2], v.w[3] = w[3];
    v.w[4] = v.w[5] = v.w[6] = v.w[7] = 0;
    double t[8 * 4 / RingGeom<D>::ESIZE > 0 ? 8 * 4 / RingGeom<D>::ESIZE : 1];
    D::unpack_raw(v, t);
#pragma unroll
    for (int k = 0; k < KE; ++k) fb[k] = t[k];
  } else {
#pragma unroll
    for (int k = 0; k < KE; ++k) fb[k] = __longlong_as_double(0x7ff8000000000000LL);
  }
}

// A fast shard's mean came out NaN / Inf (a replica holds one): FINISH decides the shard
// (k_nonfinite, bfly_merge.cu) after the kernel.  Rare: out of line, so the division of
// the shard lookup stays out of the compute loop (inlined, the checks cost the adversarial
// round 1.5 ms on 4 GPUs).
__device__ __noinline__ void ring_mark_nonfinite_vals(uint8_t* nonfin, uint32_t* any, Bounds bnd, int64_t e0,
                                                      double m0, double m1, double m2, double m3, int n) {
  const double m[4] = {m0, m1, m2, m3};
  for (int k = 0; k < n && k < 4; ++k)
    if (!finite64(m[k])) nonfin[bnd.shard_of(e0 + k)] = 1;  // (special shards: ignored)
  *any = 1u;
}
// the KE (<= 8) means of a thread starting at e0
__device__ __forceinline__ void ring_mark_nonfinite(const RingParams& p, int64_t e0, const double* m, int n) {
  if (!p.sp.nonfin) return;
  for (int k = 0; k < n; k += 4)
    ring_mark_nonfinite_vals(p.sp.nonfin, p.sp.nonfin_any, p.sp.bnd, e0 + k, m[k], k + 1 < n ? m[k + 1] : 0.0,
                             k + 2 < n ? m[k + 2] : 0.0, k + 3 < n ? m[k + 3] : 0.0, n - k);
}

template <class D>
__device__ __forceinline__ double final_value(const RingParams& p, int64_t e, double mean, const double* fb_pre = nullptr,
                                              int64_t s = -1, bool ws_done = false) {
  if (s < 0) s = p.sp.bnd.shard_of(e);
  const uint8_t c = p.sp.cls[s];
  if (c == kFast) {
    if (p.merged) p.merged[e] = mean;
    return mean;
  }
  if (c == kSpecial && !ws_done) p.sp.ws[e] = mean;
  const uint8_t pr = p.sp.pred[s] & kPredMask;
  if (pr == kPredFallback) {
    const double v = fb_pre ? *fb_pre : fallback_one<D>(p, e);
    if (p.merged && (c == kLost || p.sp.merged_apart)) p.merged[e] = v;
    return v;
  }
  if (pr == kPredMean && p.sp.merged_apart) p.merged[e] = mean;
  return mean;
}

// ---------------------------------------------------------------------------
// the roles
// ---------------------------------------------------------------------------

struct Lane {
  int c;
  uint64_t base_c, base_r;  // steps of earlier rounds on this lane (chain side, relay side)
};

// barriers and small rings (in shared memory, after the stages)
struct Bars {
  uint64_t *rep_full, *rep_empty, *acc_full, *acc_empty, *out_full, *out_empty, *rel_full, *rel_empty, *tile_full,
      *tile_empty;
  volatile int64_t *tile_of, *rtile_of;  // tile of chain step i (ring kNT), of relay step i (ring kNR)
  uint64_t* mail;                        // [0] chain landed, [1] relay landed, [2] chain done, [3] relay done
  template <class D>
  __device__ static Bars at(unsigned char* sm) {
    uint64_t* b = reinterpret_cast<uint64_t*>(sm + RingGeom<D>::OFF_BAR);
    Bars r;
    r.rep_full = b;
    r.rep_empty = b + kNS;
    r.acc_full = b + 2 * kNS;
    r.acc_empty = r.acc_full + kNA;
    r.out_full = r.acc_empty + kNA;
    r.out_empty = r.out_full + kNO;
    r.rel_full = r.out_empty + kNO;
    r.rel_empty = r.rel_full + kNR;
    r.tile_full = r.rel_empty + kNR;
    r.tile_empty = r.tile_full + kNT;
    r.tile_of = reinterpret_cast<volatile int64_t*>(r.tile_empty + kNT);
    r.rtile_of = r.tile_of + kNT;
    r.mail = reinterpret_cast<uint64_t*>(const_cast<int64_t*>(r.rtile_of + kNR));
    return r;
  }
};

// the tile id a slot carries in its 16-byte header (-1: the lane's last step)
__device__ __forceinline__ int64_t slot_tile(const void* slot) {
  int64_t v;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
  return v;
}

// The tile of chain step j of lane c, from the schedule rank 0 writes ahead of its data.
__device__ __forceinline__ int64_t sched_read(const RingParams& p, int c, uint64_t j) {
  const uint64_t* w = reinterpret_cast<const uint64_t*>(p.my + p.off_sched) + (int64_t)c * kSR + j % kSR;
  const uint32_t want = (uint32_t)(j + 1);
  uint64_t v = ld_acquire_sys(w);
  if ((uint32_t)(v >> 32) != want) {
    const uint64_t t0 = global_ns();
    const volatile uint64_t* abort_word = flag_at(p.my, p, kFAbort, 0);
    while ((uint32_t)((v = ld_acquire_sys(w)) >> 32) != want) {
      __nanosleep(20);
      if (*abort_word || global_ns() - t0 > kRingTimeoutNs) ring_abort(p);
    }
  }
  return (int64_t)(uint32_t)v - 1;
}

// LOADER (lane 0 of warp kWLoad).  Rank 0 deals the tiles: each step takes the next
// tile of the round from a counter shared by its lanes (a lane on a slower SM simply
// takes fewer), and the tile id travels in every slot header, so lane c of every later
// rank processes exactly the tiles lane c of rank 0 took.  Then: replica tiles into
// the stages, the incoming running sums into an acc stage.
template <class D>
__device__ void ring_loader(const RingParams& p, const Lane& ln, unsigned char* sm, const void** s_src) {
  using G = RingGeom<D>;
  const Bars B = Bars::at<D>(sm);
  const bool has_in = p.g > 0;
  uint64_t* ready_in = flag_at(p.my, p, kFAccReady, ln.c);
  const uint64_t pol = policy_evict_first();
  uint64_t known = 0;
  int64_t rs = 0;  // replica stage uses so far
  const bool fb_pref = fb_prefetch_on(p);
  ShardCursor cursor;
  int64_t fu = 0;  // fallback tiles prefetched so far (last rank)
  Prof pf(p, 0);
  for (int64_t i = 0;; ++i) {
    const uint64_t j = ln.base_c + (uint64_t)i;
    const int k = (int)(i % kNT);
    if (i >= kNT) mbar_wait(p, B.tile_empty + k, (unsigned)((i / kNT - 1) & 1));
    int64_t tile;
    const unsigned char* in = reinterpret_cast<const unsigned char*>(acc_slot<D>(p.my, p, ln.c, (int)(j % (uint64_t)p.NB)));
    if (has_in) {  // the tile rank 0 dealt for this step, known before its running sums arrive
      pf.start();
      tile = sched_read(p, ln.c, j);
      pf.stop(1);
    } else {
      tile = (int64_t)atomicAdd(p.tile_ctr, 1ull);
      if (tile >= p.T) tile = -1;
      const uint64_t word = ((j + 1) << 32) | (uint64_t)(uint32_t)(tile + 1);
      for (int r = 1; r < p.G; ++r)
        st_relaxed_sys(reinterpret_cast<uint64_t*>(p.region[r] + p.off_sched) + (int64_t)ln.c * kSR + j % kSR, word);
    }
    B.tile_of[k] = tile;
    mbar_arrive(B.tile_full + k);
    if (tile < 0) break;
    const int64_t t0 = tile * G::TE;
    const int64_t n = min((int64_t)G::TE, p.P - t0);
    if (fb_pref && n == G::TE) {
      const TileShards ts = tile_shards(p, cursor, t0, G::TE);
      if (!ts.fast && tile_wants_fb(p, ts)) {
        const int f = (int)(fu % kNR);
        if (fu >= kNR) mbar_wait(p, B.rel_empty + f, (unsigned)((fu / kNR - 1) & 1));
        mbar_expect_tx(B.rel_full + f, (unsigned)G::FIN_BYTES);
        bulk_load(sm + G::OFF_REL + f * G::FIN_SLOT + 16, (const unsigned char*)p.sp.fb_src + t0 * G::ESIZE,
                  (unsigned)G::FIN_BYTES, B.rel_full + f);
        ++fu;
      }
    }
    for (int q0 = 0; n == G::TE && q0 < p.n_src; q0 += kRB, ++rs) {
      const int s = (int)(rs % kNS);
      const int64_t u = rs / kNS;
      const int nb = min(kRB, p.n_src - q0);
      pf.start();
      if (u >= 1) mbar_wait(p, B.rep_empty + s, (unsigned)((u - 1) & 1));
      pf.stop(0);
      mbar_expect_tx(B.rep_full + s, (unsigned)(nb * kTileBytes));
      unsigned char* dst = sm + G::OFF_REP + s * kRB * kTileBytes;
      for (int q = 0; q < nb; ++q)
        bulk_load_stream(dst + q * kTileBytes, (const unsigned char*)s_src[q0 + q] + t0 * G::ESIZE, kTileBytes,
                         B.rep_full + s, pol);
    }
    // (the partial last tile: compute warps read its replicas directly)
    if (has_in) {
      const int a = (int)(i % kNA);
      const int64_t ua = i / kNA;
      pf.start();
      flag_wait(p, ready_in, j + 1, known);
      if (ua >= 1) mbar_wait(p, B.acc_empty + a, (unsigned)((ua - 1) & 1));
      pf.stop(2);
      const unsigned bytes = round16(n * (int64_t)sizeof(typename G::Acc));
      mbar_expect_tx(B.acc_full + a, bytes);
      bulk_load(sm + G::OFF_ACC + a * G::ACC_BYTES, in + 16, bytes, B.acc_full + a);
    }
  }
  pf.flush();
}

// FUSE stats queue in shared memory: kNQ full barriers (the compute warps arrive after
// their workspace stores: release.cta), kNQ (tile, shard) entries, the stats warps'
// progress (entries finished) and the compute warps' enqueue decision.
struct StatQ {
  uint64_t* full;
  volatile int64_t* ent;
  volatile int64_t* progress;
  volatile int* admit;
  PairStat* part;  // [2][kStatWarps]
  __device__ explicit StatQ(unsigned char* q)
      : full(reinterpret_cast<uint64_t*>(q)),
        ent(reinterpret_cast<volatile int64_t*>(q + 8 * kNQ)),
        progress(reinterpret_cast<volatile int64_t*>(q + 24 * kNQ)),
        admit(reinterpret_cast<volatile int*>(q + 24 * kNQ + 8)),
        part(reinterpret_cast<PairStat*>(q + 24 * kNQ + 16)) {}
};

// Compute warps: offer special tile `tile` (one shard `shard`, means in the workspace) to
// the stats warps as entry q.  Never waits: a full queue (the stats warps behind) leaves
// the tile to FINISH's k_stats, so the stats can only take work off the ring's tail,
// never slow its HBM stream.  Returns whether the tile was queued (uniform across the
// compute warps: thread 0 decides, one named barrier).  tile -1 (the end marker) waits
// for a free entry.
__device__ __forceinline__ bool stats_offer(const RingParams& p, unsigned char* qmem, int64_t q, int64_t tile,
                                            int64_t shard) {
  const StatQ Q(qmem);
  if (tile < 0) {
    while (q - *Q.progress >= kNQ) __nanosleep(64);
  } else {
    if (threadIdx.x == 0) *Q.admit = q - *Q.progress < kNQ;
    asm volatile("bar.sync 1, %0;" ::"n"(kRingCompute) : "memory");  // the compute warps only
    const bool ok = *Q.admit;
    asm volatile("bar.sync 1, %0;" ::"n"(kRingCompute) : "memory");  // admit read before the next write
    if (!ok) return false;
  }
  const int k = (int)(q % kNQ);
  if (threadIdx.x == 0) {
    Q.ent[2 * k] = tile;
    Q.ent[2 * k + 1] = shard;
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(Q.full + k);
  return true;
}

// STATS warps (the last rank's two relay warps, FUSE): pair statistics of the queued
// special tiles from the means in the workspace — the work FINISH's k_stats would do
// after the kernel (Philox-bound: ~1.4 ms at config 5 on 4 GPUs), overlapped with the
// HBM-bound ring.  One slot per (tile, shard), done[tile] = 1, as k_stats writes them.
template <class D>
__device__ void ring_stats(const RingParams& p, unsigned char* sm) {
  using G = RingGeom<D>;
  const StatQ Q(sm + G::OFF_STAT);
  const int t = (int)threadIdx.x - kWRLoad * 32;  // 0 .. 63
  const int w = t >> 5;
  for (int64_t j = 0;; ++j) {
    const int k = (int)(j % kNQ);
    mbar_wait(p, Q.full + k, (unsigned)((j / kNQ) & 1));
    const int64_t tile = Q.ent[2 * k], s = Q.ent[2 * k + 1];
    if (tile < 0) break;
    // (the entry is copied: thread 0 frees it only after the whole tile, below)
    const int32_t* mem = p.sp.assign + s * 2;
    const bfly_corruption_t ca = p.sp.corr[mem[0]], cb = p.sp.corr[mem[1]];
    PairAcc acc;
    const int64_t t0 = tile * G::TE;
#pragma unroll 1
    for (int64_t e0 = t0 + 4 * t; e0 < t0 + G::TE; e0 += 4 * 32 * kStatWarps) {
      double m[4], x[4], y[4];
      // written by this CTA's compute warps before their release-arrive: a plain
      // (coherent) load, not the non-coherent path
      asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(m[0]), "=d"(m[1]) : "l"(p.sp.ws + e0) : "memory");
      asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(m[2]), "=d"(m[3]) : "l"(p.sp.ws + e0 + 2) : "memory");
      corrupt4(ca, m, e0, x);
      corrupt4(cb, m, e0, y);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc.add(x[i], y[i]);
    }
    const PairStat st = warp_combine(acc.finish());
    PairStat* part = Q.part + (j & 1) * kStatWarps;
    if ((t & 31) == 0) part[w] = st;
    asm volatile("bar.sync 2, %0;" ::"n"(32 * kStatWarps) : "memory");  // the stats warps only
    if (t == 0) {
      PairStat u = part[0];
#pragma unroll
      for (int v = 1; v < kStatWarps; ++v) {
        u.mx = max_nan(u.mx, part[v].mx);
        u.ab = __dadd_rn(u.ab, part[v].ab);
        u.aa = __dadd_rn(u.aa, part[v].aa);
        u.bb = __dadd_rn(u.bb, part[v].bb);
      }
      double* o = p.sp.stats + (tile + s) * 4;  // slot (tile, shard), r = 2: one pair
      o[0] = u.mx;
      o[1] = u.ab;
      o[2] = u.aa;
      o[3] = u.bb;
      p.sp.done[tile] = 1;
      __threadfence_block();
      *Q.progress = j + 1;  // entry k is free again
    }
  }
}

// COMPUTE warps: running sums (chain) or sum and mean (REDUCE) of the lane's tiles.
// FUSE (last rank, fuse_stats): also the special shards' pair statistics — a separate
// instantiation, so the plain kernel keeps its lean register allocation.
template <class D, bool REDUCE, bool FUSE = false>
__device__ void ring_compute(const RingParams& p, const Lane& ln, unsigned char* sm, const void** s_src,
                             void** s_dst) {
  using G = RingGeom<D>;
  using Acc = typename G::Acc;
  constexpr int KE = G::KE;
  const Bars B = Bars::at<D>(sm);
  const int tid = threadIdx.x;
  const bool lead = (tid & 31) == 0;
  const bool has_in = p.g > 0;
  int64_t rs = 0;
  ShardCursor cursor;  // the shards of this lane's (ascending) tiles
  const bool fb_pref = REDUCE && fb_prefetch_on(p);
  int64_t fu = 0;  // prefetched fallback tiles consumed so far
  int64_t nq = 0;  // FUSE: special tiles handed to the stats warps
  Prof pf(p, threadIdx.x == 0 ? 4 : -1);
  if (threadIdx.x) pf.out = nullptr;
  for (int64_t i = 0;; ++i) {
    mbar_wait(p, B.tile_full + (int)(i % kNT), (unsigned)((i / kNT) & 1));
    const int64_t tile = B.tile_of[i % kNT];
    if (tile < 0) {
      if constexpr (FUSE) stats_offer(p, sm + G::OFF_STAT, nq, -1, 0);  // the stats warps' end marker
      break;
    }
    const int64_t t0 = tile * G::TE;
    const int64_t n = min((int64_t)G::TE, p.P - t0);
    const int a = (int)(i % kNA);
    const int64_t ua = i / kNA;
    const Acc* in = reinterpret_cast<const Acc*>(sm + G::OFF_ACC + a * G::ACC_BYTES);
    const int o = (int)(i % kNO);
    const int64_t uo = i / kNO;
    unsigned char* out = sm + G::OFF_OUT + o * G::OUT_SLOT + 16;  // after the header
    pf.start();
    if (has_in) {
      mbar_wait(p, B.acc_full + a, (unsigned)(ua & 1));
      // the slot's sums are in shared memory: hand the slot back to the producer now,
      // not after this step's compute and store (a shorter credit round trip)
      if (tid == 0) st_relaxed_sys(flag_at(p.prv, p, kFAccFree, ln.c), ln.base_c + (uint64_t)i + 1);
    }
    pf.stop(0);
    pf.start();
    if (uo >= 1) mbar_wait(p, B.out_empty + o, (unsigned)((uo - 1) & 1));
    pf.stop(1);
    if (n == G::TE) {
      Acc acc[KE];
#pragma unroll
      for (int k = 0; k < KE; ++k) acc[k] = has_in ? in[tid * KE + k] : D::zero();
      for (int q0 = 0; q0 < p.n_src; q0 += kRB, ++rs) {
        const int s = (int)(rs % kNS);
        const int nb = min(kRB, p.n_src - q0);
        pf.start();
        mbar_wait(p, B.rep_full + s, (unsigned)((rs / kNS) & 1));
        pf.stop(2);
        const unsigned char* st = sm + G::OFF_REP + s * kRB * kTileBytes + tid * 16;
        for (int q = 0; q < nb; ++q) {  // ascending miner order (numpy's)
          Acc x[KE];
          unpack16<D>(*reinterpret_cast<const uint4*>(st + q * kTileBytes), x);
#pragma unroll
          for (int k = 0; k < KE; ++k) acc[k] = D::add(acc[k], x[k]);
        }
        __syncwarp();
        if (lead) mbar_arrive(B.rep_empty + s);
      }
      if constexpr (REDUCE) {
        // one branch-free test per thread: is any of its means NaN / Inf?
        bool nonfin = false;
#pragma unroll
        for (int k = 0; k < KE; ++k) {
          acc[k] = D::mean(acc[k], p.n_div);
          nonfin |= !finite64(D::widen(acc[k]));
        }
        if (nonfin) {
          double m[KE];
#pragma unroll
          for (int k = 0; k < KE; ++k) m[k] = D::widen(acc[k]);
          ring_mark_nonfinite(p, t0 + tid * KE, m, KE);
        }
        const TileShards ts = p.special ? tile_shards(p, cursor, t0, G::TE) : TileShards{0, 0, true};
        if (!ts.fast) {  // predicted outcomes (k_classify) of special / lost shards
          double v[KE], fb[KE];
          const int64_t e0 = t0 + tid * KE;
          // the shard of each element: forward from the tile's first shard
          int64_t sk[KE];
          int64_t sh = ts.lo, nxt = p.sp.bnd.start(sh + 1);
          while (e0 >= nxt) nxt = p.sp.bnd.start(++sh + 1);
          bool need_fb = false;
#pragma unroll
          for (int k = 0; k < KE; ++k) {
            while (e0 + k >= nxt) nxt = p.sp.bnd.start(++sh + 1);
            sk[k] = sh;
            need_fb |= p.sp.cls[sh] != kFast && (p.sp.pred[sh] & kPredMask) == kPredFallback;
          }
          if (fb_pref && tile_wants_fb(p, ts)) {  // the loader brought the fallback tile in
            const int f = (int)(fu % kNR);
            mbar_wait(p, B.rel_full + f, (unsigned)((fu / kNR) & 1));
            const uint4 w = *reinterpret_cast<const uint4*>(sm + G::OFF_REL + f * G::FIN_SLOT + 16 + tid * 16);
            __syncwarp();
            if (lead) mbar_arrive(B.rel_empty + f);
            ++fu;
            fallback_unpack16<D>(w, fb);
          } else if (need_fb) {
            fallback_vec16<D>(p, e0, fb);
          }
          // the means of a special shard to the workspace in one vector store
          const bool ws_vec = sk[0] == sk[KE - 1] && p.sp.cls[sk[0]] == kSpecial && KE % 2 == 0;
          if (ws_vec) {
            double* w = p.sp.ws + e0;
#pragma unroll
            for (int k = 0; k + 1 < KE; k += 2)
              asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(w + k), "d"(D::widen(acc[k])),
                           "d"(D::widen(acc[k + 1]))
                           : "memory");
          }
          // a whole tile of one special shard with two device-computable copies: its means
          // are in the workspace now; the stats warps take its pair statistics from there
          // (FINISH's k_stats skips the tile), off the compute warps' critical path
          if (FUSE && ts.hi == ts.lo && (p.sp.pred[ts.lo] & kPredFuse) && ws_vec) {
            if (stats_offer(p, sm + G::OFF_STAT, nq, tile, ts.lo)) ++nq;
          }
          if (ts.lo == ts.hi) {  // the whole tile in one special / lost shard: no per-element lookups
            const uint8_t c = p.sp.cls[ts.lo], pr = p.sp.pred[ts.lo] & kPredMask;
            const bool fb_out = pr == kPredFallback;
            // merged gets the final value where final_value would write it
            const bool to_merged = p.merged && (fb_out ? (c == kLost || p.sp.merged_apart)
                                                       : (pr == kPredMean && p.sp.merged_apart));
#pragma unroll
            for (int k = 0; k < KE; ++k) v[k] = fb_out ? fb[k] : D::widen(acc[k]);
            if (to_merged) {
#pragma unroll
              for (int k = 0; k < KE; ++k) p.merged[e0 + k] = v[k];
            }
          } else {
#pragma unroll
            for (int k = 0; k < KE; ++k)
              v[k] = final_value<D>(p, e0 + k, D::widen(acc[k]), need_fb ? fb + k : nullptr, sk[k], ws_vec);
          }
          *reinterpret_cast<uint4*>(out + tid * 16) = pack16d<D>(v);
        } else {
          if (p.merged) {
            double* m = p.merged + t0 + tid * KE;
#pragma unroll
            for (int k = 0; k < KE; ++k) m[k] = D::widen(acc[k]);
          }
          *reinterpret_cast<uint4*>(out + tid * 16) = pack16<D>(acc);

        }
      } else {
#pragma unroll
        for (int k = 0; k < KE; ++k) reinterpret_cast<Acc*>(out)[tid * KE + k] = acc[k];
      }
    } else {  // partial last tile: element by element from global memory
      for (int64_t e = tid; e < n; e += kRingCompute) {
        Acc v = has_in ? in[e] : D::zero();
        for (int q = 0; q < p.n_src; ++q) v = D::add(v, D::load(s_src[q], t0 + e));
        if constexpr (REDUCE) {
          v = D::mean(v, p.n_div);
          double f;
          if (!finite64(D::widen(v))) {
            const double m = D::widen(v);
            ring_mark_nonfinite(p, t0 + e, &m, 1);
          }
          if (p.special) {
            f = final_value<D>(p, t0 + e, D::widen(v));
          } else {
            f = D::widen(v);
            if (p.merged) p.merged[t0 + e] = f;
          }
          for (int d = 0; d < p.n_dst; ++d) D::store(s_dst[d], t0 + e, f);
          D::store(out, e, f);
        } else {
          reinterpret_cast<Acc*>(out)[e] = v;
        }
      }
    }
    if (has_in) {  // the incoming sums have been read
      __syncwarp();
      if (lead) mbar_arrive(B.acc_empty + a);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // out stage -> TMA reads
    __syncwarp();
    if (lead) mbar_arrive(B.out_full + o);
  }
  pf.flush();
}

// Persisted step count of a lane side (the next round's base), in the own region.
__device__ __forceinline__ uint64_t* steps_at(const RingParams& p, int side, int lane) {
  return reinterpret_cast<uint64_t*>(p.my + p.off_steps) + (int64_t)side * p.L + lane;
}

// STORER (lane 0 of warp kWStore): returns the inbox slot, bulk-stores the outgoing
// tile with its header (next rank's inbox; on the last rank also every local replica)
// and posts the steps that have landed to the publisher (p.lag steps later, so it
// never stalls the pipe).  The lane's last step sends the end marker (tile -1).
template <class D, bool REDUCE>
__device__ void ring_storer(const RingParams& p, const Lane& ln, unsigned char* sm, void** s_dst) {
  using G = RingGeom<D>;
  using Acc = typename G::Acc;
  const Bars B = Bars::at<D>(sm);
  uint64_t* credit = p.g > 0 ? flag_at(p.prv, p, kFAccFree, ln.c) : nullptr;
  uint64_t* free_out = REDUCE ? flag_at(p.my, p, kFFinFree, ln.c) : flag_at(p.my, p, kFAccFree, ln.c);
  const uint64_t pol = policy_evict_first();
  uint64_t known = 0;
  Prof pf(p, 8);
  int64_t i = 0;
  for (;; ++i) {
    const uint64_t j = ln.base_c + (uint64_t)i;
    const int slot = (int)(j % (uint64_t)p.NB);
    const int k = (int)(i % kNT);
    mbar_wait(p, B.tile_full + k, (unsigned)((i / kNT) & 1));
    const int64_t tile = B.tile_of[k];
    const int o = (int)(i % kNO);
    pf.start();
    if (tile >= 0) mbar_wait(p, B.out_full + o, (unsigned)((i / kNO) & 1));
    pf.stop(0);
    if (credit && tile < 0) st_relaxed_sys(credit, j + 1);  // the end marker's slot (data slots: compute)
    pf.start();
    if (j >= (uint64_t)p.NB) flag_wait(p, free_out, j + 1 - p.NB, known);
    pf.stop(1);
    unsigned char* out = sm + G::OFF_OUT + o * G::OUT_SLOT;
    *reinterpret_cast<volatile int64_t*>(out) = tile;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    unsigned bytes = 16;
    int64_t t0 = 0, n = 0;
    if (tile >= 0) {
      t0 = tile * G::TE;
      n = min((int64_t)G::TE, p.P - t0);
      bytes += REDUCE ? round16(n * G::ESIZE) : round16(n * (int64_t)sizeof(Acc));
    }
    if constexpr (REDUCE) {
      if (n == G::TE)
        for (int d = 0; d < p.n_dst; ++d)
          bulk_store_stream((unsigned char*)s_dst[d] + t0 * G::ESIZE, out + 16, kTileBytes, pol);
      bulk_store(fin_slot<D>(p.nxt, p, ln.c, slot), out, bytes);
    } else {
      bulk_store(acc_slot<D>(p.nxt, p, ln.c, slot), out, bytes);
    }
    bulk_commit();
    pf.start();
    bulk_wait_read<1>();  // step i - 1's stage has been read out: hand it back
    pf.stop(2);
    if (i >= 1) mbar_arrive(B.out_empty + (int)((i - 1) % kNO));
    mbar_arrive(B.tile_empty + k);
    if (tile < 0) break;
    if (i >= p.lag && (i % p.pub_every) == 0) {  // step i - lag has landed: post it
      pf.start();
      bulk_wait_landed_n(p.lag);
      pf.stop(3);
      mail_post(B.mail, j + 1 - p.lag);
    }
  }
  bulk_wait_landed<0>();
  const uint64_t total = ln.base_c + (uint64_t)i + 1;
  *steps_at(p, 0, ln.c) = total;
  mail_post(B.mail, total);
  mail_post(B.mail + 2, 1);
  pf.flush();
}

// RELAY (ranks < last): lane 0 of warp kWRLoad loads the final tile from the inbox,
// the warp after it bulk-stores the tile into every local replica and the successor
template <class D>
__device__ void ring_relay_loader(const RingParams& p, const Lane& ln, unsigned char* sm) {
  using G = RingGeom<D>;
  const Bars B = Bars::at<D>(sm);
  uint64_t* ready_in = flag_at(p.my, p, kFFinReady, ln.c);
  uint64_t known = 0;
  Prof pf(p, 12);
  for (int64_t i = 0;; ++i) {
    const uint64_t j = ln.base_r + (uint64_t)i;
    const int s = (int)(i % kNR);
    const int64_t u = i / kNR;
    pf.start();
    flag_wait(p, ready_in, j + 1, known);
    pf.stop(0);
    pf.start();
    if (u >= 1) mbar_wait(p, B.rel_empty + s, (unsigned)((u - 1) & 1));
    pf.stop(1);
    const unsigned char* in = fin_slot<D>(p.my, p, ln.c, (int)(j % (uint64_t)p.NB));
    const int64_t tile = slot_tile(in);
    B.rtile_of[s] = tile;
    if (tile < 0) {
      mbar_arrive(B.rel_full + s);
      break;
    }
    const int64_t n = min((int64_t)G::TE, p.P - tile * G::TE);
    const unsigned bytes = round16(n * G::ESIZE);
    mbar_expect_tx(B.rel_full + s, bytes);
    bulk_load(sm + G::OFF_REL + s * G::FIN_SLOT + 16, in + 16, bytes, B.rel_full + s);
  }
  pf.flush();
}

template <class D>
__device__ void ring_relay_storer(const RingParams& p, const Lane& ln, unsigned char* sm, void** s_dst) {
  using G = RingGeom<D>;
  const Bars B = Bars::at<D>(sm);
  const bool lead = (threadIdx.x & 31) == 0;
  uint64_t* credit = flag_at(p.fpred, p, kFFinFree, ln.c);
  uint64_t* free_out = p.fsucc ? flag_at(p.my, p, kFFinFree, ln.c) : nullptr;
  const uint64_t pol = policy_evict_first();
  uint64_t known = 0;
  Prof pf(p, 16);
  if (!lead) pf.out = nullptr;
  int64_t i = 0;
  for (;; ++i) {
    const uint64_t j = ln.base_r + (uint64_t)i;
    const int s = (int)(i % kNR);
    unsigned char* st = sm + G::OFF_REL + s * G::FIN_SLOT;
    pf.start();
    mbar_wait(p, B.rel_full + s, (unsigned)((i / kNR) & 1));
    pf.stop(0);
    const int64_t tile = B.rtile_of[s];
    const int64_t t0 = tile >= 0 ? tile * G::TE : 0;
    const int64_t n = tile >= 0 ? min((int64_t)G::TE, p.P - t0) : 0;
    if (tile >= 0 && n < G::TE) {  // partial last tile: the whole warp copies the bytes
      const int64_t nb = n * G::ESIZE;
      for (int d = 0; d < p.n_dst; ++d)
        for (int64_t b = threadIdx.x & 31; b < nb; b += 32) ((unsigned char*)s_dst[d])[t0 * G::ESIZE + b] = st[16 + b];
      __syncwarp();
    }
    if (lead) {
      st_relaxed_sys(credit, j + 1);  // the inbox slot has been read
      if (n == G::TE)
        for (int d = 0; d < p.n_dst; ++d)
          bulk_store_stream((unsigned char*)s_dst[d] + t0 * G::ESIZE, st + 16, kTileBytes, pol);
      if (p.fsucc) {
        pf.start();
        if (j >= (uint64_t)p.NB) flag_wait(p, free_out, j + 1 - p.NB, known);
        pf.stop(1);
        *reinterpret_cast<volatile int64_t*>(st) = tile;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_store(fin_slot<D>(p.fsucc, p, ln.c, (int)(j % (uint64_t)p.NB)), st, 16 + round16(n * G::ESIZE));
      }
      bulk_commit();
      pf.start();
      bulk_wait_read<1>();
      pf.stop(2);
      if (i >= 1) mbar_arrive(B.rel_empty + (int)((i - 1) % kNR));
      if (p.fsucc && tile >= 0 && i >= p.lag && (i % p.pub_every) == 0) {
        pf.start();
        bulk_wait_landed_n(p.lag);
        pf.stop(3);
        mail_post(B.mail + 1, j + 1 - p.lag);
      }
    }
    __syncwarp();
    if (tile < 0) break;
  }
  if (lead) {
    bulk_wait_landed<0>();  // the last replica stores have landed before the kernel ends
    const uint64_t total = ln.base_r + (uint64_t)i + 1;
    *steps_at(p, 1, ln.c) = total;
    if (p.fsucc) mail_post(B.mail + 1, total);
    mail_post(B.mail + 3, 1);
  }
  pf.flush();
}

// PUBLISHER (lane 0 of warp kWPub): forwards the storers' landed-step counts to the
// consumers' ready flags with a system-scope release.  The release (a MEMBAR.SYS)
// takes microseconds; in its own warp it overlaps the storers' work, and a slow
// publication simply covers several steps at once.  Runs until both storers are done.
template <class D>
__device__ void ring_publisher(const RingParams& p, const Lane& ln, unsigned char* sm) {
  const Bars B = Bars::at<D>(sm);
  const bool last = p.g == p.G - 1;
  uint64_t* out_c = last ? flag_at(p.nxt, p, kFFinReady, ln.c) : flag_at(p.nxt, p, kFAccReady, ln.c);
  uint64_t* out_r = (!last && p.fsucc) ? flag_at(p.fsucc, p, kFFinReady, ln.c) : nullptr;
  uint64_t done_c = ln.base_c, done_r = ln.base_r;
  bool fin_c = false, fin_r = last;  // the last rank has no relay
  uint64_t t0 = global_ns();
  const volatile uint64_t* abort_word = flag_at(p.my, p, kFAbort, 0);
  while (!(fin_c && fin_r)) {
    const bool end_c = mail_read(B.mail + 2) != 0, end_r = last || mail_read(B.mail + 3) != 0;
    bool moved = false;
    const uint64_t vc = mail_read(B.mail);
    if (vc > done_c) {
      publish(out_c, vc);
      done_c = vc;
      moved = true;
    }
    if (out_r) {
      const uint64_t vr = mail_read(B.mail + 1);
      if (vr > done_r) {
        publish(out_r, vr);
        done_r = vr;
        moved = true;
      }
    }
    fin_c = end_c && mail_read(B.mail) == done_c;
    fin_r = end_r && (!out_r || mail_read(B.mail + 1) == done_r);
    if (moved) {
      t0 = global_ns();
    } else {
      __nanosleep(64);
      if (*abort_word || global_ns() - t0 > kRingTimeoutNs) ring_abort(p);
    }
  }
}

// One CTA = one lane of one rank: the roles above, dispatched by warp.
template <class D, bool FUSE>
__device__ __forceinline__ void ring_body(const RingParams& p, int lane) {
  extern __shared__ __align__(1024) unsigned char sm[];
  using G = RingGeom<D>;
  const void** s_src = reinterpret_cast<const void**>(sm + G::OFF_PTR);
  void** s_dst = const_cast<void**>(s_src + p.n_src);
  for (int q = threadIdx.x; q < p.n_src; q += blockDim.x) s_src[q] = p.src[q];
  for (int q = threadIdx.x; q < p.n_dst; q += blockDim.x) s_dst[q] = p.dst[q];
  Lane ln;
  ln.c = lane;
  ln.base_c = *steps_at(p, 0, ln.c);
  ln.base_r = *steps_at(p, 1, ln.c);
  const Bars B = Bars::at<D>(sm);
  if (threadIdx.x == 0) {
    const unsigned warps = kRingCompute / 32;
    for (int s = 0; s < kNS; ++s) {
      mbar_init(B.rep_full + s, 1);       // the loader's expect_tx + the bytes
      mbar_init(B.rep_empty + s, warps);  // every compute warp
    }
    for (int a = 0; a < kNA; ++a) {
      mbar_init(B.acc_full + a, 1);
      mbar_init(B.acc_empty + a, warps);
    }
    for (int o = 0; o < kNO; ++o) {
      mbar_init(B.out_full + o, warps);
      mbar_init(B.out_empty + o, 1);  // the storer
    }
    for (int s = 0; s < kNR; ++s) {  // relay stages; on the last rank: fallback tiles
      mbar_init(B.rel_full + s, 1);
      mbar_init(B.rel_empty + s, p.g == p.G - 1 ? warps : 1);
    }
    for (int k = 0; k < kNT; ++k) {
      mbar_init(B.tile_full + k, 1);   // the loader
      mbar_init(B.tile_empty + k, 1);  // the storer
    }
    if (FUSE) {
      const StatQ Q(sm + RingGeom<D>::OFF_STAT);
      for (int k = 0; k < kNQ; ++k) mbar_init(Q.full + k, warps);  // every compute warp
      *Q.progress = 0;
    }
    B.mail[0] = ln.base_c;
    B.mail[1] = ln.base_r;
    B.mail[2] = B.mail[3] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const bool last = p.g == p.G - 1;
  const int w = (int)(threadIdx.x / 32);
  const bool lead = (threadIdx.x & 31) == 0;
  if (p.prof && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.prof[blockIdx.x * kProfSlots + 20] = global_ns();
    p.prof[blockIdx.x * kProfSlots + 22] = smid;
  }
  if (w < kWLoad) {
    const long long t_start = clock64();
    if (last)
      ring_compute<D, true, FUSE>(p, ln, sm, s_src, s_dst);
    else
      ring_compute<D, false>(p, ln, sm, s_src, s_dst);
    if (p.prof && threadIdx.x == 0) {
      p.prof[blockIdx.x * kProfSlots + 7] = (unsigned long long)(clock64() - t_start);
      p.prof[blockIdx.x * kProfSlots + 21] = global_ns();
    }
  } else if (w == kWLoad) {
    if (lead) ring_loader<D>(p, ln, sm, s_src);
  } else if (w == kWStore) {
    if (lead) {
      if (last)
        ring_storer<D, true>(p, ln, sm, s_dst);
      else
        ring_storer<D, false>(p, ln, sm, s_dst);
    }
  } else if (w == kWPub) {
    if (lead) ring_publisher<D>(p, ln, sm);
  } else if (last) {
    if (FUSE && (w == kWRLoad || w == kWRStore)) ring_stats<D>(p, sm);
  } else {
    if (w == kWRLoad) {
      if (lead) ring_relay_loader<D>(p, ln, sm);
    } else {
      ring_relay_storer<D>(p, ln, sm, s_dst);
    }
  }
}

// One rank per GPU: CTA c is lane c.  The parameters are taken by value (a per-thread
// copy the compiler keeps in registers / local memory): reading them from the parameter
// bank instead (__grid_constant__) measured 1.4% slower per round (4 GPUs, C3:
// 20.98 vs 20.69 ms, tools/_ab4.sh).
template <class D, bool FUSE = false>
__global__ void __launch_bounds__(kRingThreads, 1) k_ring(RingParams p) {
  ring_body<D, FUSE>(p, (int)blockIdx.x);
}

// Single-device loopback: every rank of the ring on this GPU, CTA c is lane c % L of
// rank c / L (all co-resident: one cooperative launch).
constexpr int kMaxLoop = 8;
struct RingLoopParams {
  RingParams r[kMaxLoop];
};
template <class D, bool FUSE = false>
__global__ void __launch_bounds__(kRingThreads, 1) k_ring_loop(const __grid_constant__ RingLoopParams lp) {
  const int L = lp.r[0].L;
  const RingParams p = lp.r[blockIdx.x / L];  // this rank's parameters, copied as k_ring has them
  ring_body<D, FUSE>(p, (int)(blockIdx.x % L));
}

template <class D>
static size_t ring_smem_bytes(int n_src, int n_dst) {
  return (size_t)RingGeom<D>::OFF_PTR + sizeof(void*) * (size_t)(n_src + n_dst);
}

template <class D>
static void ring_slot_bytes(int64_t* acc_b, int64_t* fin_b) {
  *acc_b = RingGeom<D>::ACC_SLOT;
  *fin_b = RingGeom<D>::FIN_SLOT;
}

constexpr int kRingMaxPtrs = 128;  // replica pointers a CTA stages (n_src + n_dst)

template <class D>
static int ring_lanes_for() {
  int per_sm = 0;
  const size_t smem = ring_smem_bytes<D>(kRingMaxPtrs, 0);
  cudaFuncSetAttribute(k_ring<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ring<D, false>, kRingThreads, smem) != cudaSuccess)
    return 0;
  return per_sm * sm_count();
}

// the last rank fuses the pair statistics when its FINISH uses this kernel's tiles
static bool ring_fuses(const RingParams& p, int te) { return p.special && p.sp.stile == te; }

template <class D>
static int ring_launch(RingParams p, cudaStream_t st) {
  if (p.n_src + p.n_dst > kRingMaxPtrs) return fail(BFLY_E_UNSUPPORTED, "fused ring: too many local replicas");
  p.T = (p.P + RingGeom<D>::TE - 1) / RingGeom<D>::TE;
  const size_t smem = ring_smem_bytes<D>(p.n_src, p.n_dst);
  const void* kern = ring_fuses(p, RingGeom<D>::TE) ? (const void*)k_ring<D, true> : (const void*)k_ring<D, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRingThreads, smem);
  if ((int64_t)per_sm * sm_count() < p.L)
    return fail(BFLY_E_UNSUPPORTED, "fused ring: " + std::to_string(p.L) + " CTAs cannot be co-resident");
  void* args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)p.L), dim3(kRingThreads), args, smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_ring cooperative launch");
  return BFLY_OK;
}

template <class D>
static int ring_launch_loop(RingLoopParams& lp, int G, cudaStream_t st) {
  int max_ptrs = 0;
  for (int g = 0; g < G; ++g) {
    RingParams& p = lp.r[g];
    if (p.n_src + p.n_dst > kRingMaxPtrs) return fail(BFLY_E_UNSUPPORTED, "fused ring: too many local replicas");
    p.T = (p.P + RingGeom<D>::TE - 1) / RingGeom<D>::TE;
    max_ptrs = max_ptrs > p.n_src + p.n_dst ? max_ptrs : p.n_src + p.n_dst;
  }
  const size_t smem = ring_smem_bytes<D>(max_ptrs, 0);
  const void* kern = ring_fuses(lp.r[G - 1], RingGeom<D>::TE) ? (const void*)k_ring_loop<D, true>
                                                               : (const void*)k_ring_loop<D, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRingThreads, smem);
  const int64_t ctas = (int64_t)G * lp.r[0].L;
  if ((int64_t)per_sm * sm_count() < ctas)
    return fail(BFLY_E_UNSUPPORTED, "fused ring loopback: " + std::to_string(ctas) + " CTAs cannot be co-resident");
  void* args[] = {&lp};
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)ctas), dim3(kRingThreads), args, smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_ring_loop cooperative launch");
  return BFLY_OK;
}

}  // namespace bfly

using namespace bfly;

extern "C" {

int32_t bfly_ring_fused_lanes(int32_t dtype) {
  switch (dtype) {
    case BFLY_F32: return ring_lanes_for<DF32>();
    case BFLY_BF16: return ring_lanes_for<DBF16>();
    case BFLY_F64WIRE: return ring_lanes_for<DF64W>();
    default: return 0;
  }
}

int32_t bfly_ring_fused_stat_tile(int32_t dtype) {
  auto fusable = [](int te) { return te >= kMinStatTile && te % kMinStatTile == 0 ? te : 0; };
  switch (dtype) {
    case BFLY_F32: return fusable(RingGeom<DF32>::TE);
    case BFLY_BF16: return fusable(RingGeom<DBF16>::TE);
    default: return 0;  // fp64 payloads: 512-element tiles, below the smallest statistics tile
  }
}

int bfly_ring_fused_layout(int32_t lanes, int32_t nb, int32_t dtype, int64_t* off_fin, int64_t* off_flags,
                           int64_t* total) {
  if (lanes < 1 || nb < 2 || !off_fin || !off_flags || !total) return fail(BFLY_E_INVALID_ARG, "bad ring layout");
  int64_t acc_b = 0, fin_b = 0;
  switch (dtype) {
    case BFLY_F32: ring_slot_bytes<DF32>(&acc_b, &fin_b); break;
    case BFLY_BF16: ring_slot_bytes<DBF16>(&acc_b, &fin_b); break;
    case BFLY_F64WIRE: ring_slot_bytes<DF64W>(&acc_b, &fin_b); break;
    default: return fail(BFLY_E_INVALID_ARG, "bad dtype");
  }
  auto align = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
  *off_fin = align((int64_t)lanes * nb * acc_b);
  *off_flags = align(*off_fin + (int64_t)lanes * nb * fin_b);
  // then the persisted step counts (2 x lanes), rank 0's tile counter and the schedule
  *total = align(align(align(align(*off_flags + (int64_t)(kFAbort + 1) * lanes * 8) + 2 * (int64_t)lanes * 8) + 8) +
                 (int64_t)kSR * lanes * 8);
  return BFLY_OK;
}

}  // extern "C"

namespace bfly {
// Descriptor -> kernel parameters of one rank (every check before the first CUDA
// call); the last rank's per-round setup (NaN entries, flags, classify) is issued on
// `stream` here.
static int ring_params(const bfly_ring_fused_desc_t* d, void* stream, RingParams* out) {
  if (!d || d->world < 2 || d->rank < 0 || d->rank >= d->world || d->lanes < 1 || d->nb < 2 || !d->peer_base ||
      d->payload_len < 1 || d->n_src < 0 || d->n_dst < 0 || (d->n_src > 0 && !d->d_src) ||
      (d->n_dst > 0 && !d->d_dst))
    return fail(BFLY_E_INVALID_ARG, "bad fused ring descriptor");
  const int g = d->rank, G = d->world, Z = G - 1;
  if (g == Z && d->n_div < 1) return fail(BFLY_E_INVALID_ARG, "fused ring: no alive miner");
  int64_t off_fin = 0, off_flags = 0, total = 0;
  int rc = bfly_ring_fused_layout(d->lanes, d->nb, d->dtype, &off_fin, &off_flags, &total);
  if (rc) return rc;
  if (g == Z && d->special && !d->merge_args) return fail(BFLY_E_INVALID_ARG, "fused ring: special shards need merge_args");
  if (G > kMaxG) return fail(BFLY_E_UNSUPPORTED, "fused ring: too many ranks");
  if ((int64_t)kSR < (int64_t)(G - 1) * (kNT + d->nb) + 1)
    return fail(BFLY_E_UNSUPPORTED, "fused ring: schedule ring too short for this many ranks and slots");
  const int pub_every = d->pub_every > 0 ? d->pub_every : 1;
  const int lag = d->lag < 1 ? 1 : (d->lag > kMaxLag ? kMaxLag : d->lag);
  // a step is visible at most lag + pub_every - 1 steps after it is stored; its producer
  // must not need the credit of that step before then
  if (pub_every > d->nb - lag) return fail(BFLY_E_INVALID_ARG, "fused ring: nb too small for the publication lag");
  cudaStream_t st = (cudaStream_t)stream;
  RingParams p{};
  p.pub_every = pub_every;
  p.lag = lag;
  if (g == Z && d->merge_args) {
    rc = ring_round_setup(d->merge_args, stream, &p.sp);
    if (rc) return rc;
    p.special = d->special != 0;
  }
  p.g = g;
  p.G = G;
  p.L = d->lanes;
  p.NB = d->nb;
  p.P = d->payload_len;
  auto region = [&](int r) { return reinterpret_cast<unsigned char*>((uintptr_t)d->peer_base[r]); };
  p.my = region(g);
  p.nxt = g == Z ? region(0) : region(g + 1);
  p.prv = g > 0 ? region(g - 1) : nullptr;
  p.fsucc = (g < Z && g + 1 < Z) ? region(g + 1) : nullptr;
  p.fpred = g == 0 ? region(Z) : region(g - 1);
  p.off_fin = off_fin;
  p.off_flags = off_flags;
  auto align = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
  p.off_steps = align(off_flags + (int64_t)(kFAbort + 1) * p.L * 8);
  p.tile_ctr = reinterpret_cast<unsigned long long*>(p.my + align(p.off_steps + 2 * (int64_t)p.L * 8));
  p.off_sched = align(align(p.off_steps + 2 * (int64_t)p.L * 8) + 8);
  for (int r = 0; r < G; ++r) p.region[r] = region(r);
  if (g == 0) {  // the tiles of this round are dealt from 0 again
    cudaError_t e = cudaMemsetAsync(p.tile_ctr, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "fused ring: tile counter");
  }
  p.src = d->d_src;
  p.n_src = d->n_src;
  p.dst = d->d_dst;
  p.n_dst = d->n_dst;
  p.n_div = d->n_div;
  p.merged = g == Z ? d->d_merged : nullptr;
  p.prof = d->d_profile;
  if (p.prof) {
    cudaError_t e = cudaMemsetAsync(p.prof, 0, sizeof(unsigned long long) * (size_t)p.L * kProfSlots, st);
    if (e != cudaSuccess) return cuda_fail(e, "fused ring: profile buffer");
  }
  *out = p;
  return BFLY_OK;
}
}  // namespace bfly

extern "C" {

int bfly_ring_fused(const bfly_ring_fused_desc_t* d, void* stream) {
  RingParams p;
  int rc = ring_params(d, stream, &p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  switch (d->dtype) {
    case BFLY_F32: return ring_launch<DF32>(p, st);
    case BFLY_BF16: return ring_launch<DBF16>(p, st);
    case BFLY_F64WIRE: return ring_launch<DF64W>(p, st);
    default: return fail(BFLY_E_INVALID_ARG, "bad dtype");
  }
}

int bfly_ring_fused_loopback(const bfly_ring_fused_desc_t* descs, int32_t world, void* stream) {
  if (!descs || world < 2 || world > kMaxLoop) return fail(BFLY_E_INVALID_ARG, "fused ring loopback: bad world");
  for (int g = 0; g < world; ++g) {
    const bfly_ring_fused_desc_t& d = descs[g];
    if (d.rank != g || d.world != world || d.lanes != descs[0].lanes || d.nb != descs[0].nb ||
        d.dtype != descs[0].dtype || d.payload_len != descs[0].payload_len)
      return fail(BFLY_E_INVALID_ARG, "fused ring loopback: descriptors disagree");
    if (d.d_profile) return fail(BFLY_E_UNSUPPORTED, "fused ring loopback: no profile buffer");
  }
  RingLoopParams local{};
  for (int g = 0; g < world; ++g) {
    int rc = ring_params(&descs[g], stream, &local.r[g]);
    if (rc) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (descs[0].dtype) {
    case BFLY_F32: return ring_launch_loop<DF32>(local, world, st);
    case BFLY_BF16: return ring_launch_loop<DBF16>(local, world, st);
    case BFLY_F64WIRE: return ring_launch_loop<DF64W>(local, world, st);
    default: return fail(BFLY_E_INVALID_ARG, "bad dtype");
  }
}

}  // extern "C"
