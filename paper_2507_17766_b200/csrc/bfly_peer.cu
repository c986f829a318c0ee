// bfly_peer.cu — peer-memory plumbing of the multi-GPU merge (one process per
// GPU on one NVLink/NVSwitch node).
//
// Each rank exports one device region (its inboxes + flags) with CUDA IPC; the
// neighbours map it and the chain / relay kernels store straight into it over
// NVLink (fused compute + transfer).  Ordering between GPUs uses CUDA stream
// memory operations: the producer's stream writes a 32-bit flag in the
// consumer's region after the kernel that filled a slot, and the consumer's
// stream waits in the front end (no SM spins) until the flag reaches the
// slot's sequence number.  Driver entry points are resolved at run time
// (cudaGetDriverEntryPoint), so the library does not link libcuda directly.
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "bfly_internal.cuh"

namespace bfly {

typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_addr_range)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_wait32 g_wait32 = nullptr;
static PFN_write32 g_write32 = nullptr;
static PFN_addr_range g_addr_range = nullptr;
static std::once_flag g_once;
static int g_flush_supported = 0;

static int load_driver_ops() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait32 = (PFN_wait32)fn;
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write32 = (PFN_write32)fn;
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_addr_range = (PFN_addr_range)fn;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&g_flush_supported, (cudaDeviceAttr)98 /* CAN_FLUSH_REMOTE_WRITES */, dev);
  });
  if (!g_wait32 || !g_write32) return fail(BFLY_E_CUDA, "stream memory operations unavailable in this driver");
  return BFLY_OK;
}

}  // namespace bfly

using namespace bfly;

extern "C" {

int bfly_ipc_alloc(size_t bytes, void** d_ptr, uint8_t handle[64]) {
  if (!d_ptr || !handle || bytes == 0) return fail(BFLY_E_INVALID_ARG, "bad ipc alloc arguments");
  cudaError_t e = cudaMalloc(d_ptr, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "bfly_ipc_alloc cudaMalloc");
  e = cudaMemset(*d_ptr, 0, bytes);  // flags start at 0 = "nothing yet"
  if (e != cudaSuccess) return cuda_fail(e, "bfly_ipc_alloc memset");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *d_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  return BFLY_OK;
}

int bfly_ipc_open(const uint8_t handle[64], void** d_ptr) {
  if (!d_ptr || !handle) return fail(BFLY_E_INVALID_ARG, "bad ipc open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return BFLY_OK;
}

int bfly_ipc_export(const void* d_ptr, uint8_t handle[64], uint64_t* offset) {
  if (!d_ptr || !handle || !offset) return fail(BFLY_E_INVALID_ARG, "bad ipc export arguments");
  load_driver_ops();
  if (!g_addr_range) return fail(BFLY_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (g_addr_range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) return fail(BFLY_E_CUDA, "cuMemGetAddressRange");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle (export)");
  memcpy(handle, &h, 64);
  *offset = (uint64_t)((CUdeviceptr)d_ptr - base);
  return BFLY_OK;
}

int bfly_ipc_close(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return BFLY_OK;
}

int bfly_ipc_free(void* d_ptr) {
  cudaError_t e = cudaFree(d_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "bfly_ipc_free");
  return BFLY_OK;
}

int bfly_stream_create(int32_t priority, void** out) {
  if (!out) return fail(BFLY_E_INVALID_ARG, "null stream out");
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreateWithPriority");
  *out = (void*)s;
  return BFLY_OK;
}

int bfly_stream_destroy(void* stream) {
  if (!stream) return BFLY_OK;
  cudaError_t e = cudaStreamDestroy((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamDestroy");
  return BFLY_OK;
}

int bfly_stream_wait_value(const uint32_t* d_flag, uint32_t value, void* stream) {
  int rc = load_driver_ops();
  if (rc) return rc;
  const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (g_flush_supported ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
  CUresult r = g_wait32((CUstream)stream, (CUdeviceptr)d_flag, value, flags);
  if (r != CUDA_SUCCESS) return fail(BFLY_E_CUDA, "cuStreamWaitValue32 failed: " + std::to_string((int)r));
  return BFLY_OK;
}

int bfly_stream_write_value(uint32_t* d_flag, uint32_t value, void* stream) {
  int rc = load_driver_ops();
  if (rc) return rc;
  CUresult r = g_write32((CUstream)stream, (CUdeviceptr)d_flag, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(BFLY_E_CUDA, "cuStreamWriteValue32 failed: " + std::to_string((int)r));
  return BFLY_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Native executor of one multi-GPU ring round.  The op lists are the ones of
// paper_2507_17766_b200/ringsched.py (chunk_ops); bfly_ring_ops exports them
// so tests/test_ringsched.py checks both generators agree op for op.
// ---------------------------------------------------------------------------

namespace bfly {

enum RingOp : int32_t { kOpWait = 0, kOpWrite = 1, kOpChain = 2, kOpReduce = 3, kOpFanout = 4, kOpFinish = 5 };
enum RingFlag : int32_t { kAccReady = 0, kAccFree = 1, kFinReady = 2, kFinFree = 3, kReduced = 4 };

struct Op {
  int32_t kind, stream;  // stream 0 = C (chain/reduce), 1 = R (relay), 2 = F (late shards, last rank)
  int32_t peer, flag, slot, k;
  uint32_t value;
};

// The ops of rank g for chunk k (ringsched.chunk_ops, same order).
static int chunk_ops(int g, int G, int K, int NB, uint32_t round_index, int k, bool late, Op* out) {
  const int Z = G - 1;
  const uint64_t idx = (uint64_t)round_index * (uint64_t)K + (uint64_t)k;
  const int s = (int)(idx % (uint64_t)NB);
  const uint32_t v = (uint32_t)(idx + 1);
  const bool first_use = idx < (uint64_t)NB;
  const uint32_t prev = v - (uint32_t)NB;
  int n = 0;
  auto add = [&](int kind, int st, int peer, int flag, uint32_t val) {
    out[n++] = Op{kind, st, peer, flag, s, k, val};
  };
  if (g < Z) {
    if (g > 0) add(kOpWait, 0, g, kAccReady, v);
    if (!first_use) add(kOpWait, 0, g, kAccFree, prev);
    add(kOpChain, 0, g + 1, -1, 0);
    add(kOpWrite, 0, g + 1, kAccReady, v);
    if (g > 0) add(kOpWrite, 0, g - 1, kAccFree, v);
    const int succ = g + 1 < Z ? g + 1 : -1;
    const int pred = g == 0 ? Z : g - 1;
    add(kOpWait, 1, g, kFinReady, v);
    if (succ >= 0 && !first_use) add(kOpWait, 1, g, kFinFree, prev);
    add(kOpFanout, 1, succ, -1, 0);
    if (succ >= 0) add(kOpWrite, 1, succ, kFinReady, v);
    add(kOpWrite, 1, pred, kFinFree, v);
  } else {
    add(kOpWait, 0, g, kAccReady, v);
    if (!first_use) add(kOpWait, 0, g, kFinFree, prev);
    add(kOpReduce, 0, 0, -1, 0);
    if (late) {
      add(kOpWrite, 0, g, kReduced, v);
      add(kOpWrite, 0, Z - 1, kAccFree, v);
      add(kOpWait, 2, g, kReduced, v);
      add(kOpFinish, 2, 0, -1, 0);
      add(kOpWrite, 2, 0, kFinReady, v);
    } else {
      add(kOpWrite, 0, 0, kFinReady, v);
      add(kOpWrite, 0, Z - 1, kAccFree, v);
    }
  }
  return n;
}

}  // namespace bfly

extern "C" {

int bfly_ring_ops(int32_t g, int32_t G, int32_t K, int32_t NB, uint32_t round_index, int32_t late, int32_t* out,
                  int32_t cap) {
  if (G < 2 || NB < 2 || g < 0 || g >= G || K < 0) return -1;
  int n = 0;
  Op ops[16];
  for (int k = 0; k < K; ++k) {
    const int m = chunk_ops(g, G, K, NB, round_index, k, late != 0, ops);
    for (int i = 0; i < m; ++i) {
      if (n + 1 > cap) return -1;
      int32_t* r = out + 7 * n;
      r[0] = ops[i].kind;
      r[1] = ops[i].stream;
      r[2] = ops[i].peer;
      r[3] = ops[i].flag;
      r[4] = ops[i].slot;
      r[5] = ops[i].k;
      r[6] = (int32_t)ops[i].value;
      ++n;
    }
  }
  return n;
}

int bfly_ring_round(const bfly_ring_desc_t* d, uint32_t round_index) {
  if (!d || d->world < 2 || d->nb < 2 || d->k_chunks < 1) return fail(BFLY_E_INVALID_ARG, "bad ring descriptor");
  int rc = load_driver_ops();
  if (rc) return rc;
  const int g = d->rank, G = d->world, K = d->k_chunks, NB = d->nb;
  const bool last = g == G - 1;
  cudaStream_t sc = (cudaStream_t)d->stream_c, sr = (cudaStream_t)d->stream_r, sf = (cudaStream_t)d->stream_f;
  const bool late = last && d->finish_ranges != nullptr;
  // run-ahead throttle: the host never has more than `window` chunks queued per
  // stream; a launch blocked on a full queue behind a wait must not keep the host
  // from issuing the other stream's ops that wait depends on
  const int W = d->window > 0 ? d->window : 4;
  std::vector<cudaEvent_t> ev(3 * (W + 1));
  for (auto& e : ev) {
    cudaError_t ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (ce != cudaSuccess) return cuda_fail(ce, "ring event");
  }
  auto flag_addr = [&](int owner, int flag, int s) -> CUdeviceptr {
    return (CUdeviceptr)(d->peer_base[owner] + (uint64_t)d->off_flags + (uint64_t)(flag * NB + s) * 4);
  };
  bfly_merge_args_t args;
  if (last) args = *d->merge_args;
  Op ops[16];
  int result = BFLY_OK;
  for (int k = 0; k < K && result == BFLY_OK; ++k) {
    int64_t b = (int64_t)k * d->chunk;
    int64_t e = b + d->chunk < d->payload_len ? b + d->chunk : d->payload_len;
    if (d->chunk_edges) {
      b = d->chunk_edges[k];
      e = d->chunk_edges[k + 1];
      if (e - b > d->chunk || e < b) {
        result = fail(BFLY_E_INVALID_ARG, "chunk larger than an inbox slot");
        break;
      }
    }
    const int m = chunk_ops(g, G, K, NB, round_index, k, late, ops);
    for (int i = 0; i < m && result == BFLY_OK; ++i) {
      const Op& o = ops[i];
      cudaStream_t st = o.stream == 0 ? sc : (o.stream == 1 ? sr : sf);
      const int s = o.slot;
      if (o.kind == kOpWait) {
        const unsigned fl = CU_STREAM_WAIT_VALUE_GEQ | (g_flush_supported ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
        if (g_wait32((CUstream)st, flag_addr(g, o.flag, s), o.value, fl) != CUDA_SUCCESS)
          result = fail(BFLY_E_CUDA, "ring wait");
      } else if (o.kind == kOpWrite) {
        if (g_write32((CUstream)st, flag_addr(o.peer, o.flag, s), o.value, CU_STREAM_WRITE_VALUE_DEFAULT) !=
            CUDA_SUCCESS)
          result = fail(BFLY_E_CUDA, "ring write");
      } else if (o.kind == kOpChain) {  // sums stored into the next GPU's inbox (TMA bulk stores)
        const double* acc_in =
            g > 0 ? (const double*)(d->peer_base[g] + d->off_acc + (uint64_t)s * d->chunk * 8) : nullptr;
        double* acc_out = (double*)(d->peer_base[o.peer] + d->off_acc + (uint64_t)s * d->chunk * 8);
        result = bfly_chain_step(d->d_src_table, d->n_src, d->dtype, acc_in, acc_out, b, e, st);
      } else if (o.kind == kOpReduce) {
        if (d->reduce_events && d->reduce_events[k]) {
          cudaError_t ce = cudaStreamWaitEvent(st, (cudaEvent_t)d->reduce_events[k], 0);
          if (ce != cudaSuccess) {
            result = cuda_fail(ce, "ring reduce event");
            break;
          }
        }
        args.phase = BFLY_PHASE_REDUCE;
        args.d_acc_in = (const double*)(d->peer_base[g] + d->off_acc + (uint64_t)s * d->chunk * 8);
        args.elem_begin = b;
        args.elem_end = e;
        args.d_dst = (void* const*)d->reduce_tables[(int64_t)k * NB + s];
        args.n_dst = d->reduce_n;
        result = bfly_merge(&args, st);
      } else if (o.kind == kOpFinish) {
        // late shards lying inside chunk k are decided before the final chunk enters
        // the relay, through the same scatter-back table (own replicas + rank 0's inbox)
        if (d->finish_ranges[2 * k + 1] > d->finish_ranges[2 * k]) {
          bfly_merge_args_t fa = args;
          fa.phase = BFLY_PHASE_FINISH;
          fa.shard_begin = d->finish_ranges[2 * k];
          fa.shard_end = d->finish_ranges[2 * k + 1];
          fa.d_dst = (void* const*)d->reduce_tables[(int64_t)k * NB + s];
          fa.n_dst = d->reduce_n;
          result = bfly_merge(&fa, st);
        }
      } else if (o.kind == kOpFanout) {
        const void* src = (const void*)(d->peer_base[g] + d->off_fin + (uint64_t)s * d->chunk * d->esize);
        result = bfly_fanout(src, (void* const*)d->fan_tables[(int64_t)k * NB + s], d->fan_n,
                             (e - b) * d->esize, st);
      }
    }
    const int slot_ev = k % (W + 1);
    cudaEventRecord(ev[3 * slot_ev], sc);
    cudaEventRecord(ev[3 * slot_ev + 1], sr);
    cudaEventRecord(ev[3 * slot_ev + 2], late ? sf : sc);
    if (k >= W) {  // wait for chunk k - W on every stream before queueing more
      const int old = (k - W) % (W + 1);
      for (int q = 0; q < 3; ++q) cudaEventSynchronize(ev[3 * old + q]);
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return result;
}

}  // extern "C"
