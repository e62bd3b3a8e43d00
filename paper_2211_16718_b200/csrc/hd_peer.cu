// hd_peer.cu -- z-slab halo over NVLink peer memory (one process per GPU).
//
// Replaces the NCCL face exchange of the reference's RankHalo (decomp.py:183-241)
// for z-slab decompositions.  The workspaces of the two z neighbours are mapped
// into this process with CUDA IPC; the kernels that produce a stage state (the
// z sweep's RK update) or a z-differentiated viscous flux (the flux kernel)
// store the values of their g boundary planes straight into the neighbours'
// ghost planes (Geo::zpeer: the periodic image deltas shifted into the peer's
// mapping, hd_device.cuh), so the exchange overlaps the compute tile by tile
// and no copy kernel or NCCL call runs.  Ordering uses monotonic counters in
// HD_BUF_SYNC: a one-thread kernel publishes "stage v done" into both
// neighbours' flags after the producing kernel (fence.sc.sys first), and a
// one-thread kernel on the consumer's stream spins (bounded) until both
// neighbours reached v.
#include <cuda.h>
#include <cstring>

#include "hd_internal.cuh"

namespace hd {
namespace {

constexpr int SYNC_TIMEOUT = 7;  // slot of the timeout word

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_signal_kernel(unsigned long long* lo_slot, unsigned long long* hi_slot,
                                   unsigned long long v) {
  __threadfence_system();  // the producing kernel's peer stores are performed first
  atomicMax_system(lo_slot, v);
  atomicMax_system(hi_slot, v);
}

__global__ void peer_wait_kernel(unsigned long long* sync, int which, unsigned long long v) {
  const unsigned long long t0 = global_ns();
  for (;;) {
    const unsigned long long a = ld_acquire_sys(sync + 2 * which);
    const unsigned long long b = ld_acquire_sys(sync + 2 * which + 1);
    if (a >= v && b >= v) break;
    if (global_ns() - t0 > 30ull * 1000000000ull) {  // a peer died or desynchronised
      atomicExch(sync + SYNC_TIMEOUT, 1ull);
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRangeFn get_range_fn() {
  static GetRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult st;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &st) != cudaSuccess ||
        st != cudaDriverEntryPointSuccess)
      return (GetRangeFn) nullptr;
    return (GetRangeFn)f;
  }();
  return fn;
}

unsigned long long* sync_of(hd_plan* p) { return (unsigned long long*)(p->ws + p->off[HD_BUF_SYNC]); }

}  // namespace
}  // namespace hd

using namespace hd;

extern "C" {

int hd_ipc_handle(const void* ptr, void* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return HD_E_ARG;
  GetRangeFn range = get_range_fn();
  if (!range) return HD_E_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return HD_E_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return HD_E_CUDA;
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((const char*)ptr - (const char*)base);
  return HD_OK;
}

int hd_ipc_open(const void* handle64, int64_t offset, void** ptr) {
  if (!handle64 || !ptr || offset < 0) return HD_E_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HD_E_CUDA;
  *ptr = (char*)base + offset;
  return HD_OK;
}

int hd_ipc_close(void* ptr, int64_t offset) {
  if (!ptr) return HD_E_ARG;
  return cudaIpcCloseMemHandle((char*)ptr - offset) == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_attach(hd_plan* p, void* lo_ws, void* hi_ws, void* stream) {
  if (!p) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (!lo_ws && !hi_ws) {
    p->geo.zpeer = 0;
    p->geo.zpeer_lo = p->geo.zpeer_hi = 0;
    p->peer_lo = p->peer_hi = nullptr;
    return HD_OK;
  }
  if (!lo_ws || !hi_ws || p->geo.periodic[2]) return HD_E_ARG;
  const int64_t dlo = (char*)lo_ws - p->ws, dhi = (char*)hi_ws - p->ws;
  if (dlo % 8 || dhi % 8) return HD_E_ARG;
  p->geo.zpeer = 1;
  p->geo.zpeer_lo = dlo / 8;
  p->geo.zpeer_hi = dhi / 8;
  p->peer_lo = (char*)lo_ws;
  p->peer_hi = (char*)hi_ws;
  return cudaMemsetAsync(sync_of(p), 0, 64, (cudaStream_t)stream) == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_signal(hd_plan* p, int which, int64_t value, void* stream) {
  if (!p || (which != HD_PEER_STATE && which != HD_PEER_VFLUX) || value < 0) return HD_E_ARG;
  if (!p->geo.zpeer) return HD_E_UNSUPPORTED;
  const int64_t off = p->off[HD_BUF_SYNC];
  // I am the lower neighbour's "hi" and the upper neighbour's "lo"
  unsigned long long* lo_slot = (unsigned long long*)(p->peer_lo + off) + 2 * which + 1;
  unsigned long long* hi_slot = (unsigned long long*)(p->peer_hi + off) + 2 * which;
  peer_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(lo_slot, hi_slot, (unsigned long long)value);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_wait(hd_plan* p, int which, int64_t value, void* stream) {
  if (!p || (which != HD_PEER_STATE && which != HD_PEER_VFLUX)) return HD_E_ARG;
  if (!p->geo.zpeer) return HD_E_UNSUPPORTED;
  if (value <= 0) return HD_OK;
  peer_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sync_of(p), which, (unsigned long long)value);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_timed_out(hd_plan* p, int* out, void* stream) {
  if (!p || !out) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  unsigned long long v = 0;
  if (cudaMemcpyAsync(&v, sync_of(p) + SYNC_TIMEOUT, 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream) !=
          cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
    return HD_E_CUDA;
  *out = v ? 1 : 0;
  return HD_OK;
}

}  // extern "C"
