// FP64 pipe microbenchmark (B200): DFMA throughput, DMMA (mma.sync f64) throughput,
// and both issued from the same warps, to tell whether DMMA has its own pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: DFMA only, 1: DMMA only, 2: both
__global__ void k(double* out, int iters) {
  double a[8], b[8];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i), b[i] = 0.5 + 1e-9 * i;
  double c0 = 0, c1 = 0, d[4] = {0, 0, 0, 0}, e[4] = {0, 0, 0, 0};
  double ma = 1.0 + 1e-12 * threadIdx.x, mb = 1.0;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] = fma(a[i], b[i], 1e-3);
        b[i] = fma(b[i], a[i], -1e-3);
      }
    }
    if (MODE != 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        // m8n8k4 f64: A 1 reg, B 1 reg, C/D 2 regs per thread
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[r]), "+d"(e[r]) : "d"(ma), "d"(mb));
      }
    }
  }
  double s = c0 + c1;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i];
  for (int r = 0; r < 4; ++r) s += d[r] + e[r];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, threads = 512, blocks = sms * 2;
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double thr = (double)blocks * threads;
    const double dfma_flop = mode != 1 ? thr * iters * 16 * 2 : 0;           // 16 DFMA per iter
    const double dmma_flop = mode != 0 ? (double)blocks * (threads / 32) * iters * 4 * (8 * 8 * 4 * 2) : 0;
    printf("mode %d (%s): %.3f ms  DFMA %.2f TFLOP/s  DMMA %.2f TFLOP/s  total %.2f\n", mode,
           mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "both", best, dfma_flop / best / 1e9, dmma_flop / best / 1e9,
           (dfma_flop + dmma_flop) / best / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
