// hd_compat.cu -- the C entry points under the names SURVEY.md 8(b) proposes
// (hd_rk4_step, hd_max_signal, hd_totals, hd_error_flags, hd_halo_exchange),
// each a thin composition of the plan API for callers that bind one function
// per reference operation.
#include "hd_device.cuh"
#include "hd_internal.cuh"

namespace hd {
namespace {

constexpr int64_t RED_RESULT = 2048 * 9;  // result slot of HD_BUF_RED (after the partials)

__global__ void pick_kernel(const double* red, double* out, int first, int n, double scale) {
  const int t = threadIdx.x;
  if (t < n) out[t] = red[first + t] * scale;
}

// boundary layers of the peer axes into the neighbours' ghost layers
__global__ void push_faces_kernel(double* f, int nfields, Geo G, int mask) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= G.n[0] || j >= G.n[1]) return;
  const int g = G.g;
  const bool edge = ((mask & 1) && (i < g || i >= G.n[0] - g)) ||
                    ((mask & 2) && (j < g || j >= G.n[1] - g)) ||
                    ((mask & 4) && (k < g || k >= G.n[2] - g));
  if (!edge) return;
  for (int v = 0; v < nfields; ++v) {
    double* fv = f + (int64_t)v * G.npts;
    store_face_images(fv, G, i, j, k, mask, fv[G.idx(i, j, k)]);
  }
  __threadfence_system();
}

}  // namespace
}  // namespace hd

using namespace hd;

extern "C" {

int hd_rk4_step(hd_plan* p, double* u, const double* dt_dev, void* stream) {
  return hd_step(p, HD_SCHEME_RK4, u, dt_dev, 0, stream);
}

int hd_max_signal(hd_plan* p, const double* u, double* out_dev, int mode, void* stream) {
  if (!p || !u || !out_dev || (mode != 0 && mode != 1)) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  double* red = (double*)(p->ws + p->off[HD_BUF_RED]) + RED_RESULT;
  int rc = launch_reduce(p, u, red, 0, (cudaStream_t)stream);
  if (rc) return rc;
  pick_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(red, out_dev, mode ? HD_RED_SIGNAL_SUM : HD_RED_SIGNAL_MAX,
                                                  1, 1.0);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_totals(hd_plan* p, const double* u, double* out5_dev, void* stream) {
  if (!p || !u || !out5_dev) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  double* red = (double*)(p->ws + p->off[HD_BUF_RED]) + RED_RESULT;
  int rc = launch_reduce(p, u, red, 0, (cudaStream_t)stream);
  if (rc) return rc;
  const double vol = p->geo.h[0] * p->geo.h[1] * p->geo.h[2];  // timeint.py:100-107
  pick_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(red, out5_dev, HD_RED_MASS, 5, vol);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int hd_error_flags(hd_plan* p, int* flags, int64_t* where, void* stream) {
  if (!p || !flags) return HD_E_ARG;
  uint64_t key = 0;
  const int rc = hd_error_read(p, &key, stream);
  if (rc) return rc;
  *flags = 0;
  if (where) *where = -1;
  if (!key) return HD_OK;
  const int code = (int)((key >> 34) & 3);
  *flags = code == 1 ? 1 : (code == 2 ? 2 : 4);  // density, pressure, CFL signal
  if (where && code != 3) *where = (int64_t)(key & ((1ull << 34) - 1));
  return HD_OK;
}

int hd_halo_exchange(hd_plan* p, double* fields, int nfields, void* stream) {
  if (!p || !fields || nfields < 1) return HD_E_ARG;
  const Geo& G = p->geo;
  // peer images are stored at workspace offsets in the neighbours' mappings:
  // `fields` must lie inside this plan's workspace
  if (G.peer_any && ((const char*)fields < p->ws ||
                     (const char*)(fields + (int64_t)nfields * G.npts) > p->ws + p->ws_bytes))
    return HD_E_ARG;
  int rc = launch_fill_ghosts(p, fields, nfields, 7, (cudaStream_t)stream);  // periodic axes
  if (rc || !G.peer_any) return rc;
  const int mask = (G.peer[0] ? 1 : 0) | (G.peer[1] ? 2 : 0) | (G.peer[2] ? 4 : 0);
  dim3 block(32, 4, 1), grid((G.n[0] + 31) / 32, (G.n[1] + 3) / 4, G.n[2]);
  Geo only = G;  // images along the peer axes only (the periodic ones are filled)
  for (int d = 0; d < 3; ++d) only.periodic[d] = 0;
  push_faces_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(fields, nfields, only, mask);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

}  // extern "C"
