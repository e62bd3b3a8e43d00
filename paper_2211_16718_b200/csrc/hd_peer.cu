// hd_peer.cu -- block-decomposition halo over NVLink peer memory (one process per GPU).
//
// Replaces the NCCL face exchange of the reference's RankHalo (decomp.py:183-241)
// for any block decomposition.  The workspaces of the neighbours along every
// split axis are mapped into this process with CUDA IPC; the kernels that
// produce a stage state (the z sweep's RK update) or a viscous flux field (the
// flux kernel) store the values of their g boundary layers straight into the
// neighbours' ghost layers (Geo::peer: the periodic image deltas shifted into
// the peer's mapping, hd_device.cuh), so the exchange overlaps the compute tile
// by tile and no copy/pack kernel or NCCL call runs.  Ordering uses monotonic counters in
// HD_BUF_SYNC: a one-thread kernel publishes "stage v done" into every
// neighbour's flag after the producing kernel (fence.sc.sys first), and a
// one-thread kernel on the consumer's stream spins (bounded) until every
// neighbour reached v.
#include <cuda.h>
#include <cstring>

#include "hd_internal.cuh"

namespace hd {
namespace {

// HD_BUF_SYNC slots: [axis][which][side] counters (side 0: from the lower
// neighbour, 1: from the upper), then the timeout word
__host__ __device__ constexpr int sync_slot(int d, int which, int side) { return d * 4 + which * 2 + side; }
constexpr int SYNC_TIMEOUT = 15;

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

struct PeerSlots {
  unsigned long long* slot[6];  // remote counters to raise (up to two per split axis)
  int n;
};

__global__ void peer_signal_kernel(PeerSlots t, unsigned long long v) {
  __threadfence_system();  // the producing kernel's peer stores are performed first
  for (int s = 0; s < t.n; ++s) atomicMax_system(t.slot[s], v);
}

// spin until every listed local counter reached v (bounded; then the timeout word)
__global__ void peer_wait_kernel(unsigned long long* sync, int mask, int which, unsigned long long v) {
  // after one timeout the march is lost: later waits return at once instead of
  // spinning another 30 s each (the host raises HaloProtocolError at its next check)
  if (ld_acquire_sys(sync + SYNC_TIMEOUT)) return;
  const unsigned long long t0 = global_ns();
  for (;;) {
    bool ok = true;
    for (int d = 0; d < 3; ++d)
      if (mask & (1 << d))
        ok = ok && ld_acquire_sys(sync + sync_slot(d, which, 0)) >= v &&
             ld_acquire_sys(sync + sync_slot(d, which, 1)) >= v;
    if (ok) break;
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

int hd_peer_attach3(hd_plan* p, void* const* lo_ws, void* const* hi_ws, void* stream) {
  if (!p || !lo_ws || !hi_ws) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  int any = 0;
  for (int d = 0; d < 3; ++d) {
    if ((lo_ws[d] == nullptr) != (hi_ws[d] == nullptr)) return HD_E_ARG;
    if (lo_ws[d] && p->geo.periodic[d]) return HD_E_ARG;  // a periodic axis wraps locally
    const int64_t dlo = lo_ws[d] ? (char*)lo_ws[d] - p->ws : 0;
    const int64_t dhi = hi_ws[d] ? (char*)hi_ws[d] - p->ws : 0;
    if (dlo % 8 || dhi % 8) return HD_E_ARG;
  }
  for (int d = 0; d < 3; ++d) {
    p->geo.peer[d] = lo_ws[d] ? 1 : 0;
    p->geo.peer_lo[d] = lo_ws[d] ? ((char*)lo_ws[d] - p->ws) / 8 : 0;
    p->geo.peer_hi[d] = hi_ws[d] ? ((char*)hi_ws[d] - p->ws) / 8 : 0;
    p->peer_lo[d] = (char*)lo_ws[d];
    p->peer_hi[d] = (char*)hi_ws[d];
    any |= p->geo.peer[d];
  }
  p->geo.peer_any = any;
  if (!any) return HD_OK;
  return cudaMemsetAsync(sync_of(p), 0, 128, (cudaStream_t)stream) == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_attach(hd_plan* p, void* lo_ws, void* hi_ws, void* stream) {
  void* lo[3] = {nullptr, nullptr, lo_ws};
  void* hi[3] = {nullptr, nullptr, hi_ws};
  return hd_peer_attach3(p, lo, hi, stream);
}

int hd_peer_signal(hd_plan* p, int which, int64_t value, void* stream) {
  if (!p || (which != HD_PEER_STATE && which != HD_PEER_VFLUX) || value < 0) return HD_E_ARG;
  if (!p->geo.peer_any) return HD_E_UNSUPPORTED;
  const int64_t off = p->off[HD_BUF_SYNC];
  PeerSlots t;
  t.n = 0;
  for (int d = 0; d < 3; ++d) {
    if (!p->geo.peer[d]) continue;
    // I am the lower neighbour's upper side and the upper neighbour's lower side
    t.slot[t.n++] = (unsigned long long*)(p->peer_lo[d] + off) + sync_slot(d, which, 1);
    t.slot[t.n++] = (unsigned long long*)(p->peer_hi[d] + off) + sync_slot(d, which, 0);
  }
  peer_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(t, (unsigned long long)value);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_peer_wait(hd_plan* p, int which, int64_t value, void* stream) {
  if (!p || (which != HD_PEER_STATE && which != HD_PEER_VFLUX)) return HD_E_ARG;
  if (!p->geo.peer_any) return HD_E_UNSUPPORTED;
  if (value <= 0) return HD_OK;
  const int mask = (p->geo.peer[0] ? 1 : 0) | (p->geo.peer[1] ? 2 : 0) | (p->geo.peer[2] ? 4 : 0);
  peer_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sync_of(p), mask, which, (unsigned long long)value);
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
