// hd_bench.cu -- the layout / traversal study of the reference, on the GPU.
//
// The reference times its nonlinear-weight kernel over two memory layouts and
// two traversal orders (kernels.py:236-329 bench_weights_lex / _tiled, driven
// by bench.py:102-140 run_case).  Here the same study maps onto the GPU:
//
//   layout    INTERLEAVED (AoS, the 5 variables of a point adjacent) or
//             COMPONENT_CONTIGUOUS (SoA, var * npts + point)
//   traversal "lex":   one thread per active point, in lexicographic order
//                      (x fastest): consecutive lanes take consecutive x
//             "tiled": (tx, ty) thread blocks over x-y tiles of each z plane;
//                      lanes past the active extent idle, like the
//                      reference's wasted iterations (kernels.py:300-329)
//
// Weights use the reference operation order with explicit round-to-nearest
// intrinsics (never contracted to DFMA), so every layout x traversal writes
// bitwise the same point-major output as the numba kernel.
#include "hd_internal.cuh"

namespace hd {
namespace {

// kernels.py:243-266 _weights3
__device__ __forceinline__ void weights3(double f0, double f1, double f2, double f3, double f4,
                                         double eps, int power, double& w1, double& w2,
                                         double& w3) {
  const double t1 = xa(xs(f0, xm(2.0, f1)), f2);
  const double s1 = xa(xs(f0, xm(4.0, f1)), xm(3.0, f2));
  const double b1 = xa(xm(C13_12, xm(t1, t1)), xm(0.25, xm(s1, s1)));
  const double t2 = xa(xs(f1, xm(2.0, f2)), f3);
  const double s2 = xs(f1, f3);
  const double b2 = xa(xm(C13_12, xm(t2, t2)), xm(0.25, xm(s2, s2)));
  const double t3 = xa(xs(f2, xm(2.0, f3)), f4);
  const double s3 = xa(xs(xm(3.0, f2), xm(4.0, f3)), f4);
  const double b3 = xa(xm(C13_12, xm(t3, t3)), xm(0.25, xm(s3, s3)));
  const double d1 = xa(eps, b1), d2 = xa(eps, b2), d3 = xa(eps, b3);
  double e1 = d1, e2 = d2, e3 = d3;
  for (int r = 1; r < power; ++r) {
    e1 = xm(e1, d1);
    e2 = xm(e2, d2);
    e3 = xm(e3, d3);
  }
  const double a1 = xd(0.1, e1), a2 = xd(0.6, e2), a3 = xd(0.3, e3);
  const double asum = xa(xa(a1, a2), a3);
  w1 = xd(a1, asum);
  w2 = xd(a2, asum);
  w3 = xd(a3, asum);
}

// kernels.py:269-291 _bench_point (x stencil, stride 1 point)
template <bool AOS>
__device__ __forceinline__ void bench_point(const double* __restrict__ data, int64_t npts, int64_t p,
                                            double eps, int power, double* __restrict__ out) {
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double f[5];
#pragma unroll
    for (int s = 0; s < 5; ++s)
      f[s] = AOS ? __ldg(data + NV * (p + s - 2) + v) : __ldg(data + v * npts + p + s - 2);
    double w1, w2, w3;
    weights3(f[0], f[1], f[2], f[3], f[4], eps, power, w1, w2, w3);
    double* o = out + 3 * (NV * p + v);
    o[0] = w1;
    o[1] = w2;
    o[2] = w3;
  }
}

template <bool AOS>
__global__ void __launch_bounds__(256) bench_lex_kernel(const double* __restrict__ data, int nx, int ny,
                                                        int nz, int pad, double eps, int power,
                                                        double* __restrict__ out) {
  const int64_t px = nx + 2 * pad;
  const int64_t npts = px * ny * nz;
  const int64_t active = (int64_t)nx * ny * nz;
  if (active < (1ll << 31)) {  // 32-bit index arithmetic (64-bit division is ~20x dearer)
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < (unsigned)active;
         t += gridDim.x * blockDim.x) {
      const unsigned row = t / (unsigned)nx, i = t - row * (unsigned)nx;  // row = k * ny + j
      bench_point<AOS>(data, npts, (int64_t)row * px + pad + i, eps, power, out);
    }
    return;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < active;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % nx, row = t / nx;
    bench_point<AOS>(data, npts, row * px + pad + i, eps, power, out);
  }
}

template <bool AOS>
__global__ void bench_tiled_kernel(const double* __restrict__ data, int nx, int ny, int nz, int pad,
                                   double eps, int power, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= nx || j >= ny) return;  // wasted lane
  const int64_t px = nx + 2 * pad;
  const int64_t npts = px * ny * nz;
  bench_point<AOS>(data, npts, ((int64_t)k * ny + j) * px + pad + i, eps, power, out);
}

}  // namespace
}  // namespace hd

extern "C" int hd_bench_weights(const double* data, int layout, int traversal, int nx, int ny, int nz,
                                int pad, int tx, int ty, double eps, int power, double* out,
                                int64_t* wasted, void* stream) {
  using namespace hd;
  if (!data || !out || nx < 1 || ny < 1 || nz < 1 || pad < 2 || power < 1 || !(eps > 0.0))
    return HD_E_ARG;
  if (layout != 0 && layout != 1) return HD_E_ARG;
  if (traversal != 0 && traversal != 1) return HD_E_ARG;
  const bool aos = layout == 0;  // grid.py Layout.INTERLEAVED
  cudaStream_t s = (cudaStream_t)stream;
  int64_t idle = 0;
  if (traversal == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t active = (int64_t)nx * ny * nz;
    const int64_t want = (active + 255) / 256;
    const int blocks = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
    if (aos) bench_lex_kernel<true><<<blocks, 256, 0, s>>>(data, nx, ny, nz, pad, eps, power, out);
    else bench_lex_kernel<false><<<blocks, 256, 0, s>>>(data, nx, ny, nz, pad, eps, power, out);
  } else {
    if (tx < 1 || ty < 1 || tx * ty > 1024 || nz > 65535) return HD_E_ARG;
    const dim3 grid((nx + tx - 1) / tx, (ny + ty - 1) / ty, nz);
    const dim3 block(tx, ty);
    if (aos) bench_tiled_kernel<true><<<grid, block, 0, s>>>(data, nx, ny, nz, pad, eps, power, out);
    else bench_tiled_kernel<false><<<grid, block, 0, s>>>(data, nx, ny, nz, pad, eps, power, out);
    idle = (int64_t)grid.x * tx * grid.y * ty * nz - (int64_t)nx * ny * nz;
  }
  count_launches(1);
  if (wasted) *wasted = idle;
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}
