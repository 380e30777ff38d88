// FP64 roofline denominators on B200 (sm_100a): DFMA pipe and DMMA (mma.sync f64 -> DMMA.8x8x4).
// MEASURED_PEAKS.json has no FP64 entry, so this microbenchmark supplies it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  double c4[2] = {0, 0}, c5[2] = {0, 0}, c6[2] = {0, 0}, c7[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    dmma(c0, a, b); dmma(c1, a, b); dmma(c2, a, b); dmma(c3, a, b);
    dmma(c4, a, b); dmma(c5, a, b); dmma(c6, a, b); dmma(c7, a, b);
  }
  double s = c0[0] + c1[0] + c2[0] + c3[0] + c4[1] + c5[1] + c6[1] + c7[1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 1024 * sizeof(double)));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_fma = 0, best_mma = 0;
  for (int threads : {256, 512}) {
    for (int bps : {2, 4, 8}) {
      int blocks = sms * bps, iters = 2000;
      dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 64.0 * iters * (double)blocks * threads;
      float tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_fma) best_fma = tf;
      printf("dfma threads=%d blocks/sm=%d: %.2f TFLOP/s\n", threads, bps, tf);
      dmma_kernel<<<blocks, threads>>>(out, 10);
      CK(cudaEventRecord(e0));
      dmma_kernel<<<blocks, threads>>>(out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 256.0 * 8.0 * iters * (double)blocks * (threads / 32);
      tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_mma) best_mma = tf;
      printf("dmma threads=%d blocks/sm=%d: %.2f TFLOP/s\n", threads, bps, tf);
    }
  }
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d}\n", best_fma, best_mma, sms);
  return 0;
}
