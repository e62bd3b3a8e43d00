// FP64 pipe microbenchmark on sm_100a: throughput of DFMA / DMUL / DADD streams
// (8 independent chains per thread) and of a DFMA chain with a MUFU.RCP64H every
// 16 operations, at 8 and 24 warps per SM.  Answers whether DMUL/DADD issue at the
// DFMA rate (the sweeps are 42 % DFMA, 38 % DMUL, 20 % DADD).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mix tools/fp64_mix.cu && /tmp/fp64_mix
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP, int NCH = 8>
__global__ void kern(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS * 8 / NCH; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (OP == 0) x[i] = fma(x[i], a, b);
      else if (OP == 1) x[i] = x[i] * a;
      else if (OP == 2) x[i] = x[i] + b;
      else {  // DFMA with an approximate reciprocal every 16 ops
        if ((it & 1) == 0 && i == 0) {
          double r;
          asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
          x[i] = r;
        } else {
          x[i] = fma(x[i], a, b);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const char* names[] = {"DFMA", "DMUL", "DADD", "DFMA+MUFU/16"};
  for (int warps : {8, 24}) {
    for (int op = 0; op < 4; ++op) {
      dim3 grid(sms * warps / 4), block(128);
      auto launch = [&] {
        if (op == 0) kern<0><<<grid, block>>>(out, 0.999999, 1e-7);
        else if (op == 1) kern<1><<<grid, block>>>(out, 0.999999, 1e-7);
        else if (op == 2) kern<2><<<grid, block>>>(out, 0.999999, 1e-7);
        else kern<3><<<grid, block>>>(out, 0.999999, 1e-7);
      };
      launch();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 5.0 * grid.x * block.x * (double)ITERS * 8;
      printf("%-14s warps/SM %2d : %.2f Gop/s (%.1f%% of 64/clk/SM at 1.965 GHz)\n", names[op], warps,
             ops / (ms * 1e6), 100.0 * ops / (ms * 1e-3) / (sms * 64.0 * 1.965e9));
    }
  }
  // latency: DFMA with 1, 2, 4 independent chains per thread
  for (int warps : {8, 16}) {
    for (int nch : {1, 2, 4}) {
      dim3 grid(sms * warps / 4), block(128);
      auto launch = [&] {
        if (nch == 1) kern<0, 1><<<grid, block>>>(out, 0.999999, 1e-7);
        else if (nch == 2) kern<0, 2><<<grid, block>>>(out, 0.999999, 1e-7);
        else kern<0, 4><<<grid, block>>>(out, 0.999999, 1e-7);
      };
      launch();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 5.0 * grid.x * block.x * (double)ITERS * 8;
      printf("DFMA chains/thread %d warps/SM %2d : %.1f%% of peak\n", nch, warps,
             100.0 * ops / (ms * 1e-3) / (sms * 64.0 * 1.965e9));
    }
  }
  return 0;
}
