// Shared-memory broadcast-load throughput probe (B200): how many SM cycles does a warp-uniform
// LDS.128 / LDS.64 cost, against the DFMA rate it feeds in the Gauss-Jordan pivot steps
// (each thread reads the whole 256-byte pivot row per step)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_bcast_probe tools/lds_bcast_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void probe(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double row[2][64];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 128) (&row[0][0])[tid] = 1.0 + 1e-9 * tid;
  __syncthreads();
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = tid + j;
  double g = 1e-12 * (lane + 1);
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const double* pr = row[it & 1];
    if (MODE == 0) {  // 16 uniform LDS.128 + 32 DFMA (the pivot step's inner loop)
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
        r[c] = fma(-g, p2.x, r[c]);
        r[c + 1] = fma(-g, p2.y, r[c + 1]);
      }
    } else if (MODE == 1) {  // 32 DFMA only (operands in registers)
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = fma(-g, r[(c + 1) & 31], r[c]);
    } else if (MODE == 2) {  // 16 uniform LDS.128, 2 adds (loads dominate)
      double a = 0, b = 0;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
        a += p2.x;
        b += p2.y;
      }
      r[0] += a;
      r[1] += b;
    } else if (MODE == 3) {  // 16 per-lane (conflict-free) LDS.128
      double a = 0, b = 0;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const double2 p2 = *reinterpret_cast<const double2*>(&row[0][0] + ((2 * lane + 64 * (c & 1)) & 127));
        a += p2.x;
        b += p2.y;
      }
      r[0] += a;
      r[1] += b;
    } else if (MODE == 4) {  // 32 uniform LDS.64
      double a = 0, b = 0;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        a += pr[c];
        b += pr[c + 1];
      }
      r[0] += a;
      r[1] += b;
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[5] = {"16 uniform LDS.128 + 32 DFMA", "32 DFMA (registers)", "16 uniform LDS.128",
                          "16 per-lane LDS.128", "32 uniform LDS.64"};
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {1, 4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: probe<0><<<148, warps * 32>>>(out, cyc, iters); break;
          case 1: probe<1><<<148, warps * 32>>>(out, cyc, iters); break;
          case 2: probe<2><<<148, warps * 32>>>(out, cyc, iters); break;
          case 3: probe<3><<<148, warps * 32>>>(out, cyc, iters); break;
          case 4: probe<4><<<148, warps * 32>>>(out, cyc, iters); break;
        }
        cudaDeviceSynchronize();
      }
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%-32s warps/SM %2d: %7.1f cycles per iteration (warp 0), %6.1f SM-cycles per warp-iteration\n", names[mode],
             warps, (double)h[0] / iters, (double)h[0] / iters / warps);
    }
  return 0;
}
