// bfly_host.cu — host side of the drop-in path: fp64 payloads -> fp32 wire
// values in HBM.
//
// The reference's upload stage serialises every surviving miner's payload as
// "<f4" bytes (butterfly.py:213, payload.astype("<f4").tobytes()).  Doing that
// conversion on the host halves the PCIe bytes (4 B instead of 8 B per weight).
// The conversion runs on a team of host threads, each with its own ring of small
// pinned staging slots and its own copy stream, so conversion and PCIe overlap
// and the staging stays cache-resident.  Rounding is IEEE round-to-nearest-even,
// the same as numpy's astype.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bfly_internal.cuh"

extern "C" void bfly_host_f64_to_f32(const double* src, float* dst, int64_t n);  // bfly_convert.cpp

namespace bfly {

namespace {

// Each worker thread owns a small ring of pinned slots and its own copy stream:
// it converts one block of one payload into a slot and queues that slot's H2D copy
// itself, so no thread ever waits for another.  Blocks are small enough that the
// ring's lines are still in the host's last-level cache when the copy engine reads
// them back: the host memory traffic stays near the 8 B/element of the fp64 read.
constexpr int64_t kDefaultBlock = 3 << 17;  // 1.5 MB copies: best of tools/e2e_probe.py (profiles/r02_e2e_probe.log)
constexpr int kRing = 3;                     // staging slots per worker

struct Worker {
  std::vector<float*> slot;
  std::vector<cudaEvent_t> done;
  cudaStream_t stream = nullptr;
  cudaEvent_t fin = nullptr;
  int64_t count = 0;
};

// One block of one payload onto the device, by this worker: converted on the host into
// its next pinned slot (once that slot's previous copy has left) and copied.  (Copying
// some blocks raw as fp64 and converting on the GPU — PCIe traded for host-memory
// traffic — was measured slower: profiles/r01_upload_probe_raw_blocks.log.)
cudaError_t upload_block(Worker& w, int ring, const double* src, float* dst, int64_t len) {
  const int k = (int)(w.count++ % ring);
  cudaError_t ce = cudaEventSynchronize(w.done[k]);  // the slot's previous copy has left
  if (ce != cudaSuccess) return ce;
  float* slot = w.slot[k];
  bfly_host_f64_to_f32(src, slot, len);  // RNE, as numpy's astype (bfly_convert.cpp)
  ce = cudaMemcpyAsync(dst, slot, sizeof(float) * len, cudaMemcpyHostToDevice, w.stream);
  if (ce != cudaSuccess) return ce;
  return cudaEventRecord(w.done[k], w.stream);
}

struct Pool {
  std::mutex busy;  // one upload at a time uses the workers' slots and streams
  int device = -1;
  int64_t block = 0;
  int ring = 0;
  std::vector<Worker> workers;
};

std::mutex g_pool_mu;
std::vector<Pool*> g_pools;  // one per (device, shape), kept for the process lifetime

int get_pool(int threads, int64_t block, Pool** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (block == 0) block = kDefaultBlock;
  const int ring = kRing;
  if (block < 1024) return fail(BFLY_E_INVALID_ARG, "upload block must be >= 1024 elements");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (Pool* p : g_pools)
    if (p->device == dev && p->block == block && p->ring == ring && (int)p->workers.size() >= threads) {
      *out = p;
      return BFLY_OK;
    }
  Pool* p = new Pool();
  p->device = dev;
  p->block = block;
  p->ring = ring;
  p->workers.resize(threads);
  for (Worker& w : p->workers) {
    w.slot.resize(ring);
    w.done.resize(ring);
    for (int i = 0; i < ring; ++i) {
      e = cudaHostAlloc((void**)&w.slot[i], sizeof(float) * block, cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc staging");
      e = cudaEventCreateWithFlags(&w.done[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    }
    e = cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    e = cudaEventCreateWithFlags(&w.fin, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    for (int i = 0; i < ring; ++i) cudaEventRecord(w.done[i], w.stream);
  }
  g_pools.push_back(p);
  *out = p;
  return BFLY_OK;
}

}  // namespace
}  // namespace bfly

using namespace bfly;

extern "C" int bfly_upload_wire(const double* const* h_payloads, int32_t n, int64_t P, float* const* d_wire,
                                int32_t threads, int64_t block, void* stream) {
  if (!h_payloads || !d_wire || n < 0 || P < 0) return fail(BFLY_E_INVALID_ARG, "bad upload arguments");
  if (n == 0 || P == 0) return BFLY_OK;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  Pool* pool = nullptr;
  int rc = get_pool(threads, block, &pool);
  if (rc) return rc;
  std::lock_guard<std::mutex> busy(pool->busy);
  cudaStream_t st = (cudaStream_t)stream;
  // the copies must not start before work already queued on the caller's stream
  // (e.g. a previous round still reading the destination buffers)
  cudaEvent_t start;
  cudaError_t e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  cudaEventRecord(start, st);
  const int64_t B = pool->block, per = (P + B - 1) / B, total = per * (int64_t)n;
  std::atomic<int64_t> next{0};
  std::atomic<int> err{BFLY_OK};
  std::string err_msg;
  std::mutex err_mu;
  auto body = [&](int t) {
    Worker& w = pool->workers[t];
    cudaSetDevice(pool->device);
    cudaStreamWaitEvent(w.stream, start, 0);
    for (int64_t id = next.fetch_add(1); id < total && err.load() == BFLY_OK; id = next.fetch_add(1)) {
      const int32_t m = (int32_t)(id / per);
      const int64_t b = (id % per) * B, len = std::min<int64_t>(B, P - b);
      cudaError_t ce = upload_block(w, pool->ring, h_payloads[m] + b, d_wire[m] + b, len);
      if (ce != cudaSuccess) {
        std::lock_guard<std::mutex> lk(err_mu);
        err_msg = cudaGetErrorString(ce);
        err.store(BFLY_E_CUDA);
      }
    }
    cudaEventRecord(w.fin, w.stream);
  };
  std::vector<std::thread> team;
  for (int t = 1; t < threads; ++t) team.emplace_back(body, t);
  body(0);
  for (auto& th : team) th.join();
  for (int t = 0; t < threads; ++t) cudaStreamWaitEvent(st, pool->workers[t].fin, 0);
  cudaEventDestroy(start);
  if (err.load() != BFLY_OK) return fail(BFLY_E_CUDA, "upload: " + err_msg);
  return BFLY_OK;
}

// The drop-in merge of host payloads as one pipeline: the upload runs element-major
// in chunks; as soon as every worker has queued its copies of chunk c, the calling
// thread reduces chunk c on the device and copies its merged values back, while the
// workers convert and upload the next chunks (PCIe is full duplex).
extern "C" int bfly_merge_host(const double* const* h_payloads, int32_t n, int64_t P, float* const* d_wire,
                               const bfly_merge_args_t* args, double* h_merged, int32_t n_chunks, int32_t threads,
                               int64_t block, void* stream) {
  if (!h_payloads || !d_wire || !args || n < 1 || P < 1 || n_chunks < 1)
    return fail(BFLY_E_INVALID_ARG, "bad merge-host arguments");
  if (h_merged && !args->d_merged) return fail(BFLY_E_INVALID_ARG, "h_merged needs d_merged");
  // the calling thread issues the reduce of each chunk: the workers take the other cores
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency() - 1);
  Pool* pool = nullptr;
  int rc = get_pool(threads, block, &pool);
  if (rc) return rc;
  std::lock_guard<std::mutex> busy(pool->busy);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t B = pool->block;
  int64_t CL = (P + n_chunks - 1) / n_chunks;
  CL = (CL + B - 1) / B * B;  // chunk = whole blocks
  const int NC = (int)((P + CL - 1) / CL);
  const int64_t bpc = CL / B;  // blocks per full chunk and miner
  auto chunk_len = [&](int c) { return std::min<int64_t>(CL, P - (int64_t)c * CL); };
  // block ids: chunk-major, then miner, then block within the chunk
  std::vector<int64_t> first_id(NC + 1, 0);
  for (int c = 0; c < NC; ++c) first_id[c + 1] = first_id[c] + (int64_t)n * ((chunk_len(c) + B - 1) / B);
  const int64_t total = first_id[NC];

  std::vector<cudaEvent_t> ev((size_t)threads * NC);
  for (auto& e : ev) {
    cudaError_t ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaEventCreate");
  }
  cudaEvent_t start;
  cudaError_t e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  cudaEventRecord(start, st);
  std::unique_ptr<std::atomic<int>[]> queued(new std::atomic<int>[NC]);
  for (int c = 0; c < NC; ++c) queued[c].store(0);
  std::mutex q_mu;
  std::condition_variable q_cv;  // a worker finished queueing a chunk (the caller sleeps, not spins)
  std::atomic<int64_t> next{0};
  std::atomic<int> err{BFLY_OK};
  std::string err_msg;
  std::mutex err_mu;
  auto set_err = [&](cudaError_t ce) {
    std::lock_guard<std::mutex> lk(err_mu);
    err_msg = cudaGetErrorString(ce);
    err.store(BFLY_E_CUDA);
  };
  auto worker = [&](int t) {
    Worker& w = pool->workers[t];
    cudaSetDevice(pool->device);
    cudaStreamWaitEvent(w.stream, start, 0);
    int cur = 0;  // chunks below `cur` are fully queued by this worker
    auto pass = [&](int upto) {  // mark chunks [cur, upto) queued on this worker's stream
      for (; cur < upto; ++cur) {
        cudaEventRecord(ev[(size_t)t * NC + cur], w.stream);
        if (queued[cur].fetch_add(1) + 1 == threads) {
          std::lock_guard<std::mutex> lk(q_mu);
          q_cv.notify_one();
        }
      }
    };
    for (int64_t id = next.fetch_add(1); id < total; id = next.fetch_add(1)) {
      int c = cur;
      while (id >= first_id[c + 1]) ++c;
      pass(c);
      if (err.load() != BFLY_OK) continue;
      const int64_t local = id - first_id[c], nb = (chunk_len(c) + B - 1) / B;
      const int32_t m = (int32_t)(local / nb);
      const int64_t b = (int64_t)c * CL + (local % nb) * B;
      const int64_t len = std::min<int64_t>(B, (int64_t)c * CL + chunk_len(c) - b);
      cudaError_t ce = upload_block(w, pool->ring, h_payloads[m] + b, d_wire[m] + b, len);
      if (ce != cudaSuccess) set_err(ce);
    }
    pass(NC);
  };
  (void)bpc;
  std::vector<std::thread> team;
  for (int t = 0; t < threads; ++t) team.emplace_back(worker, t);
  bfly_merge_args_t a = *args;
  a.phase = BFLY_PHASE_REDUCE;
  a.shard_begin = a.shard_end = 0;
  a.d_shard_list = nullptr;
  a.n_shard_list = 0;
  int result = BFLY_OK;
  for (int c = 0; c < NC; ++c) {
    {
      std::unique_lock<std::mutex> lk(q_mu);
      q_cv.wait(lk, [&] { return queued[c].load() >= threads; });
    }
    if (result != BFLY_OK || err.load() != BFLY_OK) continue;
    for (int t = 0; t < threads; ++t) cudaStreamWaitEvent(st, ev[(size_t)t * NC + c], 0);
    a.elem_begin = (int64_t)c * CL;
    a.elem_end = a.elem_begin + chunk_len(c);
    result = bfly_merge(&a, st);
    if (result == BFLY_OK && h_merged) {
      cudaError_t ce = cudaMemcpyAsync(h_merged + a.elem_begin, args->d_merged + a.elem_begin,
                                       sizeof(double) * chunk_len(c), cudaMemcpyDeviceToHost, st);
      if (ce != cudaSuccess) result = cuda_fail(ce, "merged D2H");
    }
  }
  for (auto& th : team) th.join();
  for (auto& x : ev) cudaEventDestroy(x);
  cudaEventDestroy(start);
  if (err.load() != BFLY_OK) return fail(BFLY_E_CUDA, "upload: " + err_msg);
  return result;
}
