// bfly_host.cu — host side of the drop-in path: fp64 payloads -> fp32 wire
// values in HBM.
//
// The reference's upload stage serialises every surviving miner's payload as
// "<f4" bytes (butterfly.py:213, payload.astype("<f4").tobytes()).  Doing that
// conversion on the host halves the PCIe bytes (4 B instead of 8 B per weight).
// The conversion runs on a team of host threads into a ring of pinned staging
// slots, and each slot is copied to the device asynchronously while the next one
// is being converted, so conversion and PCIe overlap.  Rounding is IEEE
// round-to-nearest-even, the same as numpy's astype.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "bfly_internal.cuh"

namespace bfly {

namespace {

constexpr int kSlots = 4;
constexpr int64_t kSlotElems = 1 << 22;  // 16 MB of fp32 per slot

struct Staging {
  float* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  int device = -1;
};

std::mutex g_staging_mu;
std::vector<Staging*> g_staging;  // one ring per device, kept for the process lifetime

int get_staging(Staging** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_staging_mu);
  for (Staging* s : g_staging)
    if (s->device == dev) {
      *out = s;
      return BFLY_OK;
    }
  Staging* s = new Staging();
  s->device = dev;
  for (int i = 0; i < kSlots; ++i) {
    e = cudaHostAlloc((void**)&s->slot[i], sizeof(float) * kSlotElems, cudaHostAllocPortable);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc staging");
    e = cudaEventCreateWithFlags(&s->done[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    e = cudaEventRecord(s->done[i], 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  }
  g_staging.push_back(s);
  *out = s;
  return BFLY_OK;
}

// Fork-join team: the calling thread hands out one unit at a time and works on
// its own share; the team converts [begin, end) of src into dst.
class Team {
 public:
  explicit Team(int n) : n_(n) {
    for (int t = 1; t < n_; ++t) threads_.emplace_back([this, t] { loop(t); });
  }
  ~Team() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& th : threads_) th.join();
  }
  void convert(const double* src, float* dst, int64_t len) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      src_ = src;
      dst_ = dst;
      len_ = len;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    work(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void work(int t) {
    const int64_t per = (len_ + n_ - 1) / n_;
    const int64_t b = std::min<int64_t>(len_, per * t), e = std::min<int64_t>(len_, b + per);
    const double* s = src_;
    float* d = dst_;
    for (int64_t i = b; i < e; ++i) d[i] = (float)s[i];
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      work(t);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  const double* src_ = nullptr;
  float* dst_ = nullptr;
  int64_t len_ = 0;
};

}  // namespace
}  // namespace bfly

using namespace bfly;

extern "C" int bfly_upload_wire(const double* const* h_payloads, int32_t n, int64_t P, float* const* d_wire,
                                int32_t threads, void* stream) {
  if (!h_payloads || !d_wire || n < 0 || P < 0) return fail(BFLY_E_INVALID_ARG, "bad upload arguments");
  if (n == 0 || P == 0) return BFLY_OK;
  Staging* stg = nullptr;
  int rc = get_staging(&stg);
  if (rc) return rc;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  Team team(threads);
  cudaStream_t st = (cudaStream_t)stream;
  int slot = 0;
  for (int32_t m = 0; m < n; ++m) {
    for (int64_t b = 0; b < P; b += kSlotElems) {
      const int64_t len = std::min<int64_t>(kSlotElems, P - b);
      cudaError_t e = cudaEventSynchronize(stg->done[slot]);  // the slot's previous copy has left
      if (e != cudaSuccess) return cuda_fail(e, "staging event");
      team.convert(h_payloads[m] + b, stg->slot[slot], len);
      e = cudaMemcpyAsync(d_wire[m] + b, stg->slot[slot], sizeof(float) * len, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "staging H2D");
      e = cudaEventRecord(stg->done[slot], st);
      if (e != cudaSuccess) return cuda_fail(e, "staging record");
      slot = (slot + 1) % kSlots;
    }
  }
  return BFLY_OK;
}
