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

#include "bfly_internal.cuh"

namespace bfly {

typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static PFN_wait32 g_wait32 = nullptr;
static PFN_write32 g_write32 = nullptr;
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
