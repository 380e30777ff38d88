// How many warps per SM does the pass's DMMA inner loop (32 x 32 warp tile, fragments from
// shared memory, K = 32 per stage as in gj_update2_kernel) need to keep the DMMA pipe busy?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_warps_probe tools/dmma_warps_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
constexpr int LDA = 36, LDB = 68;
template <bool PF>
__global__ void probe(double* out, int iters) {
  __shared__ double As[64 * LDA];
  __shared__ double Bs[32 * LDB];
  for (int i = threadIdx.x; i < 64 * LDA; i += blockDim.x) As[i] = 1.0 + i * 1e-9;
  for (int i = threadIdx.x; i < 32 * LDB; i += blockDim.x) Bs[i] = 1.0 - i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = ((warp >> 1) & 1) * 32, c0 = (warp & 1) * 32;
  double acc[4][4][2] = {};
  for (int it = 0; it < iters; ++it) {
    if (PF) {  // fragments of k + 4 loaded while k's DMMAs issue
      double a[4], b[4], an[4], bn[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[(r0 + mi * 8 + g) * LDA + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[t * LDB + c0 + ni * 8 + g];
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        if (k + 4 < 32) {
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) an[mi] = As[(r0 + mi * 8 + g) * LDA + k + 4 + t];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) bn[ni] = Bs[(k + 4 + t) * LDB + c0 + ni * 8 + g];
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
#pragma unroll
        for (int q = 0; q < 4; ++q) { a[q] = an[q]; b[q] = bn[q]; }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = As[(r0 + mi * 8 + g) * LDA + k + t];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k + t) * LDB + c0 + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int pf = 0; pf < 2; ++pf)
    for (int warps : {1, 2, 4, 8, 12, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (pf) probe<true><<<sms, warps * 32>>>(out, iters);
        else probe<false><<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 32 * 32 * 32 * (double)iters * warps * sms;
        if (rep) printf("prefetch %d warps/SM %2d: %.2f TFLOP/s (%.1f%% of 36.945)\n", pf, warps, fl / ms / 1e9,
                        100.0 * fl / ms / 1e9 / 36.945);
      }
    }
  return 0;
}
