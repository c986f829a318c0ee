/*
 * bfly.h — C ABI of the B200-native butterfly merge (IOTA data-parallel merge step).
 *
 * The reference has no FFI: its boundary is the Python module API of
 * `iota_sim.butterfly` (pkg/src/iota_sim/butterfly.py:22-35).  Each entry point
 * below replaces one stage of that module; the Python mirror in
 * paper_2507_17766_b200/butterfly.py binds them with ctypes exactly as a
 * maintainer of the reference would.
 *
 * Conventions
 *   - plain pointers and sizes only; "d_" = device pointer, "h_" = host pointer;
 *   - every call returns an int status (BFLY_OK or one of the BFLY_E* codes,
 *     mapped 1:1 to the reference exception classes in errors.py:4-45) and
 *     leaves a message in bfly_last_error() (thread-local);
 *   - device work is stream-ordered on the `stream` argument (a cudaStream_t,
 *     passed as void* so this header needs no CUDA include); no call
 *     synchronises the device unless its comment says so.
 */
#ifndef BFLY_H_
#define BFLY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py) ------------------------------------------ */
#define BFLY_OK 0
#define BFLY_E_TOO_FEW_MINERS 1   /* TooFewMinersError       errors.py:28 */
#define BFLY_E_DEGENERATE 2       /* DegenerateShardsError   errors.py:32 */
#define BFLY_E_SHAPE 3            /* ShapeError              errors.py:12 */
#define BFLY_E_INVALID_ARG 4      /* InvalidArgumentError    errors.py:36 */
#define BFLY_E_CUDA 5             /* CUDA runtime failure (no reference analogue) */
#define BFLY_E_UNSUPPORTED 6      /* NotImplementedError (e.g. custom reducer) */

/* ---- element types of the miner replicas ------------------------------- */
#define BFLY_F32 0      /* fp32 wire values ("<f4", butterfly.py:213) */
#define BFLY_BF16 1     /* bf16 replicas, fp32 accumulation (C4 extension) */
#define BFLY_F64WIRE 2  /* fp64 payloads rounded to the fp32 wire on load (butterfly.py:213,230) */

/* ---- per-shard status (butterfly.py:151) ------------------------------- */
#define BFLY_MERGED 0
#define BFLY_LOST 1
#define BFLY_DISAGREEMENT 2

/* ---- corruption descriptors (GPU-native form of butterfly.py:168,232-233) */
#define BFLY_CORR_NONE 0
#define BFLY_CORR_ADD 1           /* copy = mean + a                              */
#define BFLY_CORR_SCALE 2         /* copy = mean * a                              */
#define BFLY_CORR_NOISE 3         /* copy = a * (2u - 1), u = Philox(key, elem)   */
#define BFLY_CORR_NOISE_ADD 4     /* copy = mean + a * (2u - 1)                   */
#define BFLY_CORR_HOST 5          /* copy supplied by the caller (Python callable) */

typedef struct bfly_corruption {
  int32_t kind;   /* BFLY_CORR_* */
  int32_t pad;
  double a;       /* constant, scale or noise amplitude */
  uint64_t key0;  /* Philox4x64-10 key of the noise stream (colluders share it) */
  uint64_t key1;
} bfly_corruption_t;

/* ---- merge phases ------------------------------------------------------ */
#define BFLY_PHASE_ALL 0       /* reduce + compare + decide + adopt/scatter-back */
#define BFLY_PHASE_REDUCE 1    /* reduce only: means of every element -> d_merged/d_ws */
#define BFLY_PHASE_FINISH 2    /* compare + decide + adopt, after PHASE_REDUCE and host copies */
#define BFLY_PHASE_CHECK 3     /* only decide fast shards whose mean came out non-finite (after a
                                  reduction that did not itself end at payload_len, e.g. the
                                  multi-GPU persistent ring); PHASE_ALL / FINISH and a REDUCE of
                                  the range ending at payload_len include it */

typedef struct bfly_merge_args {
  int32_t n_miners;      /* N = plan.pair_set.n_miners                    (butterfly.py:188) */
  int32_t redundancy;    /* r: 2 = reference pairs; 3 = triple extension              */
  int64_t payload_len;   /* P elements                                    (butterfly.py:195) */
  int64_t n_shards;      /* S = C(N, r)                                   (butterfly.py:57)  */
  int32_t dtype;         /* BFLY_F32 / BFLY_BF16 / BFLY_F64WIRE                       */
  int32_t n_alive;       /* number of miners not in `failures`           (butterfly.py:203) */
  const int32_t* d_assign;        /* [S*r] ascending miner indices of shard s        */
  const void* const* d_src;       /* [n_alive] replicas of the alive miners, ascending index */
  const uint8_t* d_failed;        /* [N] 1 = dropped before upload                  */
  const bfly_corruption_t* d_corr;/* [N] per-miner corruption (kind NONE if honest) */
  void* const* d_dst;             /* [n_dst] scatter-back targets (in place), or NULL */
  int32_t n_dst;
  int32_t stat_tile;              /* elements per statistics tile of the special shards' pair
                                     statistics (0 = the reduce kernel's tile); the persistent
                                     ring sets its own tile (bfly_ring_fused_stat_tile) */
  const double* d_fallback;       /* [P] fallback weights, or NULL (butterfly.py:169,268-273) */
  double* d_merged;               /* [P] fp64 merged vector, or NULL                */
  double* d_ws;                   /* [P] fp64 means of special (corrupted) shards; may be
                                     NULL when d_merged is given (then reused in place) */
  const double* d_host_copies;    /* [r*P] copies for BFLY_CORR_HOST survivors: slot k of
                                     shard s at d_host_copies[k*P + e]                */
  uint8_t* d_status;              /* [S] out: BFLY_MERGED / LOST / DISAGREEMENT     */
  double* d_entries;              /* [N*N] out: agreement matrix, NaN where undefined */
  uint8_t* d_flagged;             /* [N] out: 1 = flagged miner                     */
  int32_t* d_source;              /* [S] out: adopted assignee, -1 if fallback; may be NULL */
  void* d_scratch;                /* scratch, >= bfly_merge_scratch_bytes()         */
  size_t scratch_bytes;
  double tolerance;               /* agreement_tolerance (butterfly.py:171)         */
  int32_t phase;                  /* BFLY_PHASE_*                                   */
  int32_t pad1;
  /* multi-GPU (one process per GPU, miners in contiguous blocks per GPU): the
   * last GPU of the chain finishes the reduction from the running sums */
  const double* d_acc_in;         /* [elem_end-elem_begin] fp64 running sums from the previous GPUs, or NULL */
  int32_t n_div;                  /* divisor of the mean = alive miners on all GPUs; 0 = n_alive */
  int32_t pad2;
  int64_t elem_begin;             /* REDUCE this element range only; 0,0 = all.  The per-round */
  int64_t elem_end;               /* setup (NaN fill, classify) runs with the range starting at 0 */
  const void* d_fallback_src;     /* replica supplying fallback values (lowest alive miner);
                                     NULL = d_src[0]                                   */
  int64_t shard_begin;            /* FINISH these shards only; 0,0 = all (the multi-GPU */
  int64_t shard_end;              /* last rank finishes each chunk's shards early)      */
  const int32_t* d_shard_list;    /* FINISH these [n_shard_list] shards instead of the range
                                     (device array; e.g. shards straddling chunk edges) */
  int32_t n_shard_list;
  int32_t fallback_gone;          /* 1 = the fallback replica has been overwritten in place before
                                     the shards decided after the reduction read it (multi-GPU
                                     rounds: the relay); fast shards with non-finite means then
                                     take d_fallback or NaN */
} bfly_merge_args_t;

/* ---- validator replay checks ---------------------- */
/* For each of n_pairs (recomputed, reported) activation pairs, packed back to back in
 * d_rec / d_rep with pair i at [d_offsets[i], d_offsets[i+1]): the reference's
 * replay check `_check` (validator.py:148-167) — cosine similarity (validator.py:33-46),
 * then 0 if below h_policy[0] (cosine_threshold), if the norm ratio |rep|/|rec| is
 * outside [h_policy[1], h_policy[2]] (magnitude band, only when |rec| > 0), or if
 * max|rec - rep| / max(|rec|, 1) > h_policy[3] (max_rel_deviation).  d_sim[i] gets
 * the similarity, d_cos[i] (optional) the plain cosine.  Shapes are the caller's
 * business (ShapeError is raised on the host). */
int bfly_replay_check(const double* d_rec, const double* d_rep, const int64_t* d_offsets, int32_t n_pairs,
                      const double* h_policy, double* d_sim, double* d_cos, void* stream);

/* ---- library ----------------------------------------------------------- */
const char* bfly_version(void);
const char* bfly_last_error(void);

/* C(n, r) shard count; -1 on overflow.  enumerate_pairs  butterfly.py:76-81 */
int64_t bfly_n_shards(int32_t n_miners, int32_t redundancy);

/* Philox key of RngStream(seed, stream_id): first 16 bytes of
 * SHA-256(f"{seed}\x1f{stream_id}") as two little-endian u64.
 * `seed_decimal` is str(int(seed)).   simkernel.py:203-205,216-219 */
int bfly_philox_key(const char* seed_decimal, const char* stream_id, uint64_t out_key[2]);

/* Shard plan on the host: h_assign[S*r] (ascending members of the combination
 * assigned to shard s) and h_bounds[S+1] element offsets.
 * plan_shards  butterfly.py:84-114 (permutation simkernel.py:237-238). */
int bfly_plan_host(int32_t n_miners, int32_t redundancy, int64_t payload_len, uint64_t key0,
                   uint64_t key1, int32_t* h_assign, int64_t* h_bounds);

/* RngStream(seed, stream_id).permutation(n) on the host (simkernel.py:237-238):
 * h_out[n] = Fisher-Yates from i = n-1 down to 1 with numpy's random_interval.
 * plan_shards uses it for a caller-built PairSet: assignment[s] = pairs[h_out[s]]
 * (butterfly.py:98-100). */
int bfly_permutation_host(int64_t n, uint64_t key0, uint64_t key1, int64_t* h_out);

/* Same plan computed on the device (GPU index map).  d_perm[S] receives the
 * shard -> combination-rank permutation; d_assign[S*r] the members. */
int bfly_plan_device(int32_t n_miners, int32_t redundancy, int64_t payload_len, uint64_t key0,
                     uint64_t key1, int64_t* d_perm, int32_t* d_assign, void* stream);

/* Scratch bytes bfly_merge needs for these sizes. */
size_t bfly_merge_scratch_bytes(int32_t n_miners, int32_t redundancy, int64_t payload_len);

/* One merge round: run_all_reduce  butterfly.py:161-295, device-resident. */
int bfly_merge(const bfly_merge_args_t* args, void* stream);

/* One link of the cross-GPU reduction chain (multi-GPU merge): for elements
 * e in [begin, end), d_acc_out[e-begin] = (d_acc_in ? d_acc_in[e-begin] : +0.0)
 * + x_0[e] + x_1[e] + ... over this GPU's alive replicas in ascending miner
 * order — the reference's summation order continued across GPUs. */
int bfly_chain_step(const void* const* d_src, int32_t n_src, int32_t dtype, const double* d_acc_in,
                    double* d_acc_out, int64_t begin, int64_t end, void* stream);

/* Upload n fp64 host payloads of P elements (pageable or pinned) as fp32 wire
 * values ("<f4", butterfly.py:213) into the device buffers d_wire[i]: `threads`
 * host threads (0 = all cores) convert blocks of `block` elements (0 = 384 Ki, 1.5 MB
 * copies) into a ring of pinned staging slots while earlier slots are copied, so
 * conversion and PCIe overlap.  Returns when the last copy has been issued on
 * `stream` (the host payloads may be reused after the stream reaches that point). */
int bfly_upload_wire(const double* const* h_payloads, int32_t n, int64_t P, float* const* d_wire,
                     int32_t threads, int64_t block, void* stream);

/* The drop-in merge of host payloads as one pipeline (run_all_reduce's upload +
 * reduce stages, butterfly.py:205-240, and the copy of the merged vector back):
 * the upload of bfly_upload_wire runs element-major in n_chunks chunks and, as
 * each chunk lands, bfly_merge(args) reduces it (phase REDUCE over the chunk's
 * elements; the first chunk runs the per-round setup) and args->d_merged[chunk] is
 * copied to h_merged (NULL: no copy) while later chunks are still converting and
 * uploading.  The caller runs phase FINISH afterwards when shards need it (and then
 * copies those shards' merged values again). */
int bfly_merge_host(const double* const* h_payloads, int32_t n, int64_t P, float* const* d_wire,
                    const bfly_merge_args_t* args, double* h_merged, int32_t n_chunks, int32_t threads,
                    int64_t block, void* stream);

/* ---- peer memory for the multi-GPU merge (one process per GPU, one node) ---- */
/* cudaMalloc a zero-filled region and export its CUDA IPC handle (64 bytes). */
int bfly_ipc_alloc(size_t bytes, void** d_ptr, uint8_t handle[64]);
/* Map a neighbour's region (peer access over NVLink enabled lazily). */
int bfly_ipc_open(const uint8_t handle[64], void** d_ptr);
/* Export an existing device buffer (e.g. a framework tensor inside a larger cudaMalloc
 * block): the IPC handle of its allocation and the byte offset of d_ptr in it.  The
 * importer maps the handle with bfly_ipc_open and adds the offset. */
int bfly_ipc_export(const void* d_ptr, uint8_t handle[64], uint64_t* offset);
int bfly_ipc_close(void* d_ptr);
int bfly_ipc_free(void* d_ptr);
/* Stream-ordered cross-GPU signalling (CUDA stream memory operations, no SM spin):
 * the stream waits until (int32)(*d_flag - value) >= 0, flushing remote writes
 * when the device supports it; or writes value to *d_flag (with a memory
 * barrier) once all earlier work in the stream is done. */
/* Load every kernel of the merge and of the chunked multi-GPU ring now (CUDA lazy loading
 * would load each at its first launch, which can wait for the device: fatal when several
 * ranks share one device and their streams already wait on each other — the loopback). */
int bfly_preload(void);

/* A CUDA stream of this process's own (non-blocking, priority as cudaStreamCreateWithPriority):
 * the multi-GPU executors' streams wait on flags other ranks write, so they must never be
 * shared with anything else (torch hands out pooled streams, which wrap around). */
int bfly_stream_create(int32_t priority, void** stream);
int bfly_stream_destroy(void* stream);
int bfly_stream_wait_value(const uint32_t* d_flag, uint32_t value, void* stream);
int bfly_stream_write_value(uint32_t* d_flag, uint32_t value, void* stream);

/* One round of the multi-GPU ring (chain -> last rank -> relay), issued natively.
 * Every rank calls it with its own descriptor; ops follow ringsched.chunk_ops. */
typedef struct bfly_ring_desc {
  int32_t rank, world;           /* this process's rank and the ring size           */
  int32_t k_chunks, nb;          /* chunks per round, inbox slots                   */
  int64_t payload_len, chunk;    /* P and elements per chunk                        */
  int32_t dtype, esize;          /* BFLY_* element type of the replicas, its bytes  */
  const uint64_t* peer_base;     /* [world] region base of every rank as mapped here */
  int64_t off_acc, off_fin, off_flags;  /* region layout                             */
  const void* const* d_src_table;/* chain: this rank's alive replicas (device table) */
  int32_t n_src;
  int32_t fan_n;                 /* relay: pointers per fan-out table               */
  const uint64_t* fan_tables;    /* [k_chunks*nb] device tables (host array)         */
  bfly_merge_args_t* merge_args; /* last rank: the round's prepared merge arguments  */
  const uint64_t* reduce_tables; /* [k_chunks*nb] scatter-back tables of the last rank */
  int32_t reduce_n, window;      /* pointers per reduce table; chunks of run-ahead   */
  void* stream_c;                /* chain / reduce stream                           */
  void* stream_r;                /* relay stream                                    */
  const int64_t* finish_ranges;  /* last rank, optional: [k_chunks*2] shard range to FINISH
                                    after reducing chunk k (shards inside the chunk), on
                                    stream_f, before the chunk enters the relay          */
  void* stream_f;                /* last rank: late-shard stream (with finish_ranges)  */
  void* const* reduce_events;    /* last rank, optional: [k_chunks] cudaEvent_t (or NULL)
                                    the C stream waits for before reducing chunk k (the
                                    chunk's fallback values have arrived)               */
  const int64_t* chunk_edges;    /* optional [k_chunks+1] element boundaries of the chunks
                                    (each <= chunk); NULL = uniform chunks of `chunk`   */
} bfly_ring_desc_t;
int bfly_ring_round(const bfly_ring_desc_t* desc, uint32_t round_index);
/* The op list of one rank for one round as rows of 7 int32
 * {kind, stream, peer, flag, slot, chunk, value}; returns the row count or -1. */
int bfly_ring_ops(int32_t rank, int32_t world, int32_t k_chunks, int32_t nb, uint32_t round_index,
                  int32_t late, int32_t* out, int32_t cap);

/* The whole multi-GPU round in ONE persistent kernel per GPU (k_ring,
 * csrc/bfly_ring.cu): the payload is cut into tiles (4 KB of each replica) dealt
 * round-robin to `lanes` lanes, one CTA per SM; lane c of every rank hands tile after
 * tile to lane c of the neighbouring rank through a slot ring in the neighbour's IPC
 * region.  Warp-specialised: a loader warp bulk-loads replica tiles and incoming sums
 * (TMA, mbarrier stage ring), compute warps add in ascending miner order, a storer
 * warp bulk-stores into the next rank's inbox, relay warps move the final tiles into
 * every replica, a publisher warp releases 64-bit monotonic flags (st.release.sys;
 * consumers poll with ld.acquire.sys) — the NVLink transfer of tile i overlaps the
 * HBM stream of tile i+1.  Same values as bfly_ring_round (running fp64 sums in
 * ascending miner order).  Needs shards of >= 2 elements and 16-byte aligned
 * replicas.  Rounds with corrupted / lost shards (desc.special on the last rank):
 * the relayed tiles carry k_classify's predicted outcome, FINISH on the last rank
 * decides those shards after the kernel, and the caller re-broadcasts the few whose
 * decision differs from the prediction.
 * Replaces, for these rounds, the chunked exchange of bfly_ring_round; the reference
 * has no multi-GPU path (run_all_reduce, butterfly.py:161-295, is one process).     */
typedef struct bfly_ring_fused_desc {
  int32_t rank, world;           /* this process's rank and the ring size            */
  int32_t lanes, nb;             /* lanes (equal on every rank), slots per lane      */
  int32_t dtype;                 /* BFLY_* element type of the replicas              */
  int32_t n_src, n_dst, n_div;   /* alive local replicas, all local replicas, divisor */
  int64_t payload_len;           /* P                                                */
  uint64_t round_index;          /* informational: the flags are monotonic step counts the
                                    kernel persists per lane in the region itself      */
  const uint64_t* peer_base;     /* [world] region base of every rank as mapped here  */
  const void* const* d_src;      /* device table of the alive local replicas          */
  void* const* d_dst;            /* device table of every local replica (scatter-back) */
  double* d_merged;              /* last rank, optional: fp64 merged vector            */
  const bfly_merge_args_t* merge_args; /* last rank, optional: the round's per-shard
                                    setup (status / entries / flags) runs first       */
  int32_t special;               /* last rank: some shard may be corrupted or lost — its
                                    tiles get k_classify's predicted outcome (and the means
                                    go to the workspace); FINISH runs after the kernel  */
  int32_t pub_every;             /* publish a lane's ready flag every pub_every-th step (0 = 1) */
  int32_t lag;                   /* ... once the step is lag steps old (1..3; 0 = 1); needs
                                    nb >= lag + pub_every                              */
  int32_t pad;
  unsigned long long* d_profile; /* diagnostics, or NULL: [lanes * 24] per-CTA wait cycles
                                    per role, CTA start / end times (globaltimer), SM id */
} bfly_ring_fused_desc_t;
/* Lanes this device runs (all CTAs co-resident: cooperative launch). */
int32_t bfly_ring_fused_lanes(int32_t dtype);
/* Byte layout of one rank's region for (lanes, nb, dtype): offsets of the final-vector
 * slots and of the flags, and the total size to allocate (bfly_ipc_alloc zeroes it). */
int bfly_ring_fused_layout(int32_t lanes, int32_t nb, int32_t dtype, int64_t* off_fin, int64_t* off_flags,
                           int64_t* total);
int bfly_ring_fused(const bfly_ring_fused_desc_t* desc, void* stream);
/* Elements per k_ring tile when the last rank accumulates the special shards' pair
 * statistics inside the kernel (set bfly_merge_args_t.stat_tile to it for the round's
 * FINISH), or 0 when this dtype's tiles are too small to (fp64 payloads). */
int32_t bfly_ring_fused_stat_tile(int32_t dtype);
/* Single-device loopback: `world` ranks of one ring on THIS device, in one cooperative
 * launch of world x lanes CTAs (CTA c serves lane c % lanes of rank c / lanes).  descs[g]
 * is rank g's descriptor exactly as bfly_ring_fused takes it, with the regions being
 * plain allocations of this device (peer_base[r] = rank r's region).  The same kernel
 * code, protocol and results as the multi-GPU ring — driver-testable and profileable
 * (ncu) on one GPU.  world <= 8. */
int bfly_ring_fused_loopback(const bfly_ring_fused_desc_t* descs, int32_t world, void* stream);

/* Copy nbytes from d_src into each of n_dst device buffers (scatter-back fan-out). */
int bfly_fanout(const void* d_src, void* const* d_dst, int32_t n_dst, int64_t nbytes, void* stream);

/* For every shard s with d_mask[s] != 0 and d_status[s] == BFLY_DISAGREEMENT: element e of
 * the shard := d_fallback[e] (NULL: NaN) in each of the n_dst replicas.  Multi-GPU ranks
 * other than the last apply the last rank's decision on fast shards whose mean was not
 * finite (butterfly.py:127-133,264-273) to their own replicas — no host round trip. */
int bfly_fill_shards(const uint8_t* d_status, const uint8_t* d_mask, const double* d_fallback, void* const* d_dst,
                     int32_t n_dst, int32_t dtype, int64_t payload_len, int64_t n_shards, void* stream);

/* Element ranges between a full-length vector and a packed buffer:
 * scatter == 0: d_packed[off_r + i] = d_full[lo_r + i];
 * scatter == 1: d_dst[k][lo_r + i] = d_packed[off_r + i] for every k.
 * d_ranges = n_ranges x {lo, hi, off} (int64, device).  Multi-GPU redistribution
 * of the shards decided after the chain (corrupted / lost shards). */
int bfly_copy_ranges(const void* d_full, void* d_packed, void* const* d_dst, int32_t n_dst,
                     const int64_t* d_ranges, int32_t n_ranges, int32_t elem_size, int32_t scatter,
                     void* stream);

/* Pairwise agreement of two device vectors into *d_out (fp64).
 * agreement  butterfly.py:117-133. */
int bfly_agreement(const double* d_a, const double* d_b, int64_t len, double tolerance,
                   double* d_out, void* d_scratch, size_t scratch_bytes, void* stream);

/* Copy of one assignee under a corruption descriptor: d_out[i] = corrupt(d_in[i])
 * for global elements start_elem + i (the GPU form of butterfly.py:232-233). */
int bfly_apply_corruption(const bfly_corruption_t* h_desc, const double* d_in, int64_t start_elem,
                          int64_t len, double* d_out, void* stream);

/* Element-wise mean over the rows of a (n_rows, width) fp64 stack, in the
 * reference's order.  mean_reducer  butterfly.py:156-158. */
int bfly_mean_rows(const double* d_stack, int32_t n_rows, int64_t width, double* d_out,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BFLY_H_ */
