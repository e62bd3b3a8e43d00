// Accuracy of the fp64 MUFU seeds (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64) and of
// one / two Newton steps, against the IEEE results, over log-uniform inputs.
#include <cstdio>
#include <cmath>
__global__ void k(int n, double* out) {
  double m[6] = {0, 0, 0, 0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double x = exp(-9.0 + 18.0 * (i + 0.5) / n);
    double r, s;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(s) : "d"(x));
    double rx = 1.0 / x, sx = 1.0 / sqrt(x);
    double r1 = fma(r, fma(-x, r, 1.0), r);
    double r2 = fma(r1, fma(-x, r1, 1.0), r1);
    // rsqrt Newton: s' = s (1.5 - 0.5 x s^2) = s + s * 0.5 * (1 - x s^2)
    double s1 = fma(s, 0.5 * fma(-x * s, s, 1.0), s);
    double s2 = fma(s1, 0.5 * fma(-x * s1, s1, 1.0), s1);
    double e[6] = {fabs(r / rx - 1), fabs(r1 / rx - 1), fabs(r2 / rx - 1),
                   fabs(s / sx - 1), fabs(s1 / sx - 1), fabs(s2 / sx - 1)};
    for (int j = 0; j < 6; ++j) m[j] = fmax(m[j], e[j]);
  }
  for (int j = 0; j < 6; ++j) {
    unsigned long long* p = (unsigned long long*)&out[j];
    atomicMax(p, __double_as_longlong(m[j]));
  }
}
int main() {
  double* d;
  cudaMalloc(&d, 6 * sizeof(double));
  cudaMemset(d, 0, 6 * sizeof(double));
  k<<<1024, 256>>>(1 << 26, d);
  double h[6];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("rcp seed %.3e  1 Newton %.3e  2 Newton %.3e\n", h[0], h[1], h[2]);
  printf("rsqrt seed %.3e  1 Newton %.3e  2 Newton %.3e\n", h[3], h[4], h[5]);
  return 0;
}
