// Rank-K combined-pass probe: the gj_update2_kernel tile scheme (64 x 64 output tile per CTA of
// 4 warps, C fragments loaded from global into registers, the K columns of A and K rows of W
// staged by cp.async in 32-wide halves, DMMA m8n8k4) for K = 64 and K = 128 over a batch of
// n x n matrices: how much of the DMMA peak does a rank-128 pass reach?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pass_probe tools/pass_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TK = 32, LDA_S = 36, LDB_S = 68;
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
// A: [job][n][K] row-major, W: [job][K][n], C: [job][n][n]
template <int NH>  // NH = K / 32
__global__ void __launch_bounds__(128) pass_k(const double* A, const double* W, double* C, int n) {
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                       // [NH][64][LDA_S]
  double* Bs = As + NH * 64 * LDA_S;     // [NH][32][LDB_S]
  const int K = NH * 32;
  const int job = blockIdx.z, row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  const double* Aj = A + (size_t)job * n * K;
  const double* Wj = W + (size_t)job * K * n;
  double* Cj = C + (size_t)job * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int h = 0; h < NH; ++h) {
    for (int idx = tid; idx < 64 * 16; idx += 128) {
      const int r = idx >> 4, c = (idx & 15) * 2;
      cp16(&As[(h * 64 + r) * LDA_S + c], &Aj[(size_t)(row0 + r) * K + h * 32 + c]);
    }
    for (int idx = tid; idx < 32 * 32; idx += 128) {
      const int r = idx >> 5, c = (idx & 31) * 2;
      cp16(&Bs[(h * 32 + r) * LDB_S + c], &Wj[(size_t)(h * 32 + r) * n + col0 + c]);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(&Cj[(size_t)(r0 + mi * 8 + g) * n + c0 + ni * 8 + 2 * t]);
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
    }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int lr0 = (warp >> 1) * 32, lc0 = (warp & 1) * 32;
#pragma unroll
  for (int h = 0; h < NH; ++h)
#pragma unroll
    for (int k = 0; k < TK; k += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[(h * 64 + lr0 + mi * 8 + g) * LDA_S + k + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(h * 32 + k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(&Cj[(size_t)(r0 + mi * 8 + g) * n + c0 + ni * 8 + 2 * t]) =
          make_double2(acc[mi][ni][0], acc[mi][ni][1]);
}
template <int NH>
void run(int n, int jobs, double* A, double* W, double* C) {
  const size_t smem = (size_t)(NH * 64 * LDA_S + NH * 32 * LDB_S) * 8;
  cudaFuncSetAttribute(pass_k<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(n / 64, n / 64, jobs);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  pass_k<NH><<<grid, 128, smem>>>(A, W, C, n);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) pass_k<NH><<<grid, 128, smem>>>(A, W, C, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_k<NH>, 128, smem);
  const double fl = 2.0 * jobs * (double)n * n * (NH * 32);
  printf("n %d jobs %d K %3d: %.3f ms  %.2f TFLOP/s (%.1f%% of 36.945)  %d CTAs/SM  smem %zu  %s\n", n, jobs, NH * 32, ms,
         fl / ms / 1e9, 100 * fl / ms / 1e9 / 36.945, occ, smem, cudaGetErrorString(cudaGetLastError()));
}
// K-pipelined: a 2-slot ring of 32-wide halves (the K = 64 kernel's shared memory, any K)
template <int NH, int SLOTS>
__global__ void __launch_bounds__(128) pass_ring(const double* A, const double* W, double* C, int n) {
  extern __shared__ __align__(16) double sm[];
  const int K = NH * 32;
  const int job = blockIdx.z, row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  const double* Aj = A + (size_t)job * n * K;
  const double* Wj = W + (size_t)job * K * n;
  double* Cj = C + (size_t)job * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  auto issue = [&](int h) {
    double* As = sm + (h % SLOTS) * (64 * LDA_S + 32 * LDB_S);
    double* Bs = As + 64 * LDA_S;
    for (int idx = tid; idx < 64 * 16; idx += 128) {
      const int r = idx >> 4, c = (idx & 15) * 2;
      cp16(&As[r * LDA_S + c], &Aj[(size_t)(row0 + r) * K + h * 32 + c]);
    }
    for (int idx = tid; idx < 32 * 32; idx += 128) {
      const int r = idx >> 5, c = (idx & 31) * 2;
      cp16(&Bs[r * LDB_S + c], &Wj[(size_t)(h * 32 + r) * n + col0 + c]);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  issue(0);
  if (NH > 1 && SLOTS > 1) issue(1);
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(&Cj[(size_t)(r0 + mi * 8 + g) * n + c0 + ni * 8 + 2 * t]);
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
    }
  const int lr0 = (warp >> 1) * 32, lc0 = (warp & 1) * 32;
#pragma unroll 1
  for (int h = 0; h < NH; ++h) {
    if (SLOTS > 1 && h + 1 < NH) asm volatile("cp.async.wait_group 1;\n" ::);
    else asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    const double* As = sm + (h % SLOTS) * (64 * LDA_S + 32 * LDB_S);
    const double* Bs = As + 64 * LDA_S;
#pragma unroll
    for (int k = 0; k < TK; k += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[(lr0 + mi * 8 + g) * LDA_S + k + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
    __syncthreads();
    if (h + SLOTS < NH) issue(h + SLOTS);
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(&Cj[(size_t)(r0 + mi * 8 + g) * n + c0 + ni * 8 + 2 * t]) =
          make_double2(acc[mi][ni][0], acc[mi][ni][1]);
}
template <int NH, int SLOTS = 2>
void run_ring(int n, int jobs, double* A, double* W, double* C) {
  const size_t smem = (size_t)SLOTS * (64 * LDA_S + 32 * LDB_S) * 8;
  cudaFuncSetAttribute(pass_ring<NH, SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(n / 64, n / 64, jobs);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  pass_ring<NH, SLOTS><<<grid, 128, smem>>>(A, W, C, n);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) pass_ring<NH, SLOTS><<<grid, 128, smem>>>(A, W, C, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_ring<NH, SLOTS>, 128, smem);
  const double fl = 2.0 * jobs * (double)n * n * (NH * 32);
  printf("ring%d n %d jobs %d K %3d: %.3f ms  %.2f TFLOP/s (%.1f%% of 36.945)  %d CTAs/SM  %s\n", SLOTS, n, jobs, NH * 32, ms,
         fl / ms / 1e9, 100 * fl / ms / 1e9 / 36.945, occ, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int n = cfg ? 512 : 4096, jobs = cfg ? 512 : 16;
    double *A, *W, *C;
    cudaMalloc(&A, (size_t)jobs * n * 256 * 8);
    cudaMalloc(&W, (size_t)jobs * 256 * n * 8);
    cudaMalloc(&C, (size_t)jobs * n * n * 8);
    cudaMemset(A, 0, (size_t)jobs * n * 256 * 8);
    cudaMemset(W, 0, (size_t)jobs * 256 * n * 8);
    cudaMemset(C, 0, (size_t)jobs * n * n * 8);
    run<2>(n, jobs, A, W, C);
    run<4>(n, jobs, A, W, C);
    run_ring<2>(n, jobs, A, W, C);
    run_ring<4>(n, jobs, A, W, C);
    run_ring<8>(n, jobs, A, W, C);
    run_ring<2, 1>(n, jobs, A, W, C);
    run_ring<4, 3>(n, jobs, A, W, C);
    cudaFree(A);
    cudaFree(W);
    cudaFree(C);
  }
  return 0;
}
