// sz_peer.cu — device-side flags for the fused encode -> NVLink handoff
// (SURVEY §8f row 2).
//
// The sender's encoder writes its sections straight into the receiver's
// HBM (peer / IPC-mapped pointers: every code, sign-mantissa and escape
// store crosses NVLink once, no staging copy, no NCCL kernel taking SMs),
// then raises a flag in the receiver's memory; the receiver's stream waits
// on that flag, decodes, and raises a "slot free" flag in the sender's
// memory.  The host only enqueues: the whole pipeline is ordered on the two
// GPUs by these two tiny kernels.
//
// Ordering: a kernel boundary on a stream orders all prior device work
// before the signal kernel; the signal adds a system-scope fence and a
// release store.  The waiter polls with system-scope acquire loads, and the
// consumer kernels that follow it on its stream see the producer's data.
// Waits give up after a timeout (default 30 s) and record it, so a lost
// peer never wedges the GPU.
#include "sz_common.cuh"

namespace sz {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_signal_kernel(uint64_t* flag, uint64_t value) {
  // (runs after every prior kernel of its stream has completed)
  __threadfence_system();
  st_release_sys(flag, value);
}

__global__ void peer_wait_kernel(const uint64_t* flag, uint64_t value, uint64_t timeout_ns,
                                 uint32_t* timed_out) {
  // after one timeout the link is broken: later waits return at once, so a
  // lost peer costs one timeout, not one per piece
  if (timed_out && *reinterpret_cast<volatile uint32_t*>(timed_out)) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys(flag) < value) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      if (timed_out) atomicOr(timed_out, 1u);
      return;
    }
    __nanosleep(1000);
  }
}

}  // namespace sz

extern "C" {

int sz_record_cuda(cudaError_t e);  // sz_misc.cu

int sz_peer_signal(uint64_t* d_flag, uint64_t value, void* stream) {
  if (!d_flag) return SZ_ECONFIG;
  sz::peer_signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_flag, value);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

int sz_peer_wait(const uint64_t* d_flag, uint64_t value, uint64_t timeout_ns,
                 uint32_t* d_timed_out, void* stream) {
  if (!d_flag) return SZ_ECONFIG;
  // The one-thread poller must not shrink its SM's shared-memory carveout:
  // a codec kernel on another stream of this GPU (the persistent encoder
  // wants ~200 KB per SM) has to fit beside it, or that CTA would wait for
  // the poller — which may be waiting for that very kernel.
  // (a function attribute of the current device's context: set once per device)
  static bool carved[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !carved[dev]) {
    const cudaError_t carve = cudaFuncSetAttribute(
        sz::peer_wait_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
        static_cast<int>(cudaSharedmemCarveoutMaxShared));
    if (carve != cudaSuccess) return sz_record_cuda(carve);
    if (dev >= 0 && dev < 64) carved[dev] = true;
  }
  sz::peer_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      d_flag, value, timeout_ns ? timeout_ns : 30000000000ull, d_timed_out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

// ---- device memory shared across processes (CUDA IPC) --------------------
// The receive slots live in one dedicated cudaMalloc region (IPC handles name
// whole allocations, never caching-allocator sub-blocks); both sides carve
// it with the same layout, so one 64-byte handle describes every buffer.
int sz_device_alloc(uint64_t bytes, void** d_out) {
  if (!d_out || !bytes) return SZ_ECONFIG;
  cudaError_t e = cudaMalloc(d_out, bytes);
  if (e == cudaSuccess) e = cudaMemset(*d_out, 0, bytes);
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

int sz_device_free(void* d) {
  const cudaError_t e = cudaFree(d);
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

int sz_ipc_export(const void* d_base, uint8_t* handle_out) {
  if (!d_base || !handle_out) return SZ_ECONFIG;
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_base));
  if (e != cudaSuccess) return sz_record_cuda(e);
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  for (int i = 0; i < 64; ++i) handle_out[i] = static_cast<uint8_t>(h.reserved[i]);
  return SZ_OK;
}

int sz_ipc_import(const uint8_t* handle, void** d_base_out) {
  if (!handle || !d_base_out) return SZ_ECONFIG;
  cudaIpcMemHandle_t h;
  for (int i = 0; i < 64; ++i) h.reserved[i] = static_cast<char>(handle[i]);
  const cudaError_t e = cudaIpcOpenMemHandle(d_base_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

int sz_ipc_close(void* d_base) {
  const cudaError_t e = cudaIpcCloseMemHandle(d_base);
  return e == cudaSuccess ? SZ_OK : sz_record_cuda(e);
}

}  // extern "C"
