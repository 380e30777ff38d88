// Microbenchmark (design study, not product code): batched 32x32 pivoted Gauss-Jordan inversion,
// one warp per matrix, two formulations --
//   A: Engine F's register GJ (row per lane, shift-in-FMA, 32 FMAs + 16 broadcast loads per step);
//   B: blocked in shared memory: 8-column panels factored in registers (8-wide rows), trailing
//      rank-8 update of the other 24 columns on DMMA (mma.sync m8n8k4 f64).
// Both leave the inverse in permuted storage R[piv[k]][j] = Minv[k][piv[j]]; the harness checks
// ||A * Minv - I|| on the host and times throughput (8 warps per CTA) and isolated latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gj_micro tools/gj_micro.cu && tools/gj_micro
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int N = 32, LD = 33;

__device__ __forceinline__ double rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---- A: register GJ (Engine F's formulation) -------------------------------------------------
__global__ void __launch_bounds__(256) inv_reg(const double* A, double* R, int* P, int batch) {
  __shared__ __align__(16) double prow[8][2][34];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  if (b >= batch) return;
  double r[N];
  for (int j = 0; j < N; ++j) r[j] = A[(size_t)b * N * N + lane * N + j];
  bool used = false;
  double rowscale = 1.0;
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
    const double r0 = r[0];
    const bool cand = !used && r0 != 0.0;
    const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~63u) | (unsigned)(63 - lane)) : 0u;
    const unsigned km = __reduce_max_sync(0xffffffffu, key);
    const int p = 63 - (int)(km & 63u);
    const double pv = __shfl_sync(0xffffffffu, r0, p);
    const double rp = rcp(pv);
    double* pw = prow[warp][k & 1];
    const bool own = lane == p;
    if (own) {
      used = true;
      rowscale = rp;
#pragma unroll
      for (int j = 0; j < N; j += 2) *reinterpret_cast<double2*>(pw + j) = make_double2(r[j], r[j + 1]);
      P[(size_t)b * N + k] = lane;
    }
    __syncwarp();
    const double g = own ? 0.0 : r0 * rp, last = own ? 1.0 : -g;
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(pw + j);
      if (j > 0) r[j - 1] = fma(-g, p2.x, r[j]);
      r[j] = fma(-g, p2.y, r[j + 1 < N ? j + 1 : j]);
    }
    r[N - 1] = last;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) R[(size_t)b * N * N + lane * N + j] = r[j] * rowscale;
}

// ---- B: blocked GJ in shared memory, DMMA trailing updates -----------------------------------
constexpr int PB = 8;  // panel width
__global__ void __launch_bounds__(128) inv_blk(const double* A, double* R, int* P, int batch) {
  __shared__ __align__(16) double Ms[4][N * LD];
  __shared__ __align__(16) double Wsh[4][PB * LD];
  __shared__ __align__(16) double prow[4][2][PB + 2];
  __shared__ int rstep_s[4][N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + warp;
  if (b >= batch) return;
  double* M = Ms[warp];
  double* W = Wsh[warp];
  int* rstep = rstep_s[warp];
  for (int i = 0; i < N; ++i) M[i * LD + lane] = A[(size_t)b * N * N + i * N + lane];
  rstep[lane] = -1;
  __syncwarp();
  const int g = lane >> 2, t = lane & 3;
  bool used = false;
#pragma unroll 1
  for (int k0 = 0; k0 < N; k0 += PB) {
    double a[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) a[c] = M[lane * LD + k0 + c];
    double rowscale = 1.0;
    bool piv_here = false;
#pragma unroll
    for (int kk = 0; kk < PB; ++kk) {
      const double r0 = a[0];
      const bool cand = !used && r0 != 0.0;
      const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~63u) | (unsigned)(63 - lane)) : 0u;
      const unsigned km = __reduce_max_sync(0xffffffffu, key);
      const int p = 63 - (int)(km & 63u);
      const double pv = __shfl_sync(0xffffffffu, r0, p);
      const double rp = rcp(pv);
      double* pw = prow[warp][kk & 1];
      const bool own = lane == p;
      if (own) {
        used = true;
        piv_here = true;
        rowscale = rp;
#pragma unroll
        for (int c = 0; c < PB; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(a[c], a[c + 1]);
        rstep[lane] = k0 + kk;
        P[(size_t)b * N + k0 + kk] = lane;
      }
      __syncwarp();
      const double gg = own ? 0.0 : r0 * rp, last = own ? 1.0 : -gg;
#pragma unroll
      for (int c = 0; c < PB; c += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pw + c);
        if (c > 0) a[c - 1] = fma(-gg, p2.x, a[c]);
        a[c] = fma(-gg, p2.y, a[c + 1 < PB ? c + 1 : c]);
      }
      a[PB - 1] = last;
    }
    if (piv_here) {
#pragma unroll
      for (int c = 0; c < PB; ++c) a[c] *= rowscale;
    }
    // snapshot the panel's pivot rows outside the panel, then write the factored panel
    __syncwarp();
    for (int c = 0; c < PB; ++c) {
      const int pr = P[(size_t)b * N + k0 + c];  // (global read of the pivot index, same warp)
      W[c * LD + lane] = (lane >= k0 && lane < k0 + PB) ? 0.0 : M[pr * LD + lane];
    }
#pragma unroll
    for (int c = 0; c < PB; ++c) M[lane * LD + k0 + c] = a[c];
    __syncwarp();
    // trailing update of the 3 other 8-column groups: C(32 x 8 each) = live ? C : 0, += A W
#pragma unroll
    for (int grp = 0; grp < N / 8; ++grp) {
      const int c0 = grp * 8;
      if (c0 == k0) continue;
      double acc[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int i = mi * 8 + g;
        const int rs = rstep[i];
        const bool live = !(rs >= k0 && rs < k0 + PB);
        acc[mi][0] = live ? M[i * LD + c0 + 2 * t] : 0.0;
        acc[mi][1] = live ? M[i * LD + c0 + 2 * t + 1] : 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < PB; ks += 4) {
        const double bb = W[(ks + t) * LD + c0 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma(acc[mi], M[(mi * 8 + g) * LD + k0 + ks + t], bb);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        M[(mi * 8 + g) * LD + c0 + 2 * t] = acc[mi][0];
        M[(mi * 8 + g) * LD + c0 + 2 * t + 1] = acc[mi][1];
      }
    }
    __syncwarp();
  }
  for (int i = 0; i < N; ++i) R[(size_t)b * N * N + i * N + lane] = M[i * LD + lane];
}

static void check(const char* what, const std::vector<double>& A, const std::vector<double>& R,
                  const std::vector<int>& P, int batch) {
  double worst = 0.0;
  for (int b = 0; b < batch; b += 97) {
    const double* a = &A[(size_t)b * N * N];
    const double* r = &R[(size_t)b * N * N];
    const int* p = &P[(size_t)b * N];
    int rs[N];
    for (int k = 0; k < N; ++k) rs[p[k]] = k;
    // Minv[a][c] = R[piv[a]][rowstep[c]]  (R[piv[k]][j] = Minv[k][piv[j]])
    double err = 0.0;
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < N; ++c) {
        double s = 0.0;
        for (int m = 0; m < N; ++m) s += a[i * N + m] * r[p[m] * N + rs[c]];
        err = fmax(err, fabs(s - (i == c ? 1.0 : 0.0)));
      }
    worst = fmax(worst, err);
  }
  printf("%-4s max |A Minv - I| = %.3g\n", what, worst);
}

int main() {
  const int batch = 148 * 64;
  std::vector<double> A((size_t)batch * N * N);
  srand(1);
  for (auto& v : A) v = (rand() / (double)RAND_MAX - 0.5) * 0.2;
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < N; ++i) A[(size_t)b * N * N + i * N + i] += 1.0;
  double *dA, *dR;
  int* dP;
  cudaMalloc(&dA, A.size() * 8);
  cudaMalloc(&dR, A.size() * 8);
  cudaMalloc(&dP, (size_t)batch * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  std::vector<double> R(A.size());
  std::vector<int> P((size_t)batch * N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    auto run = [&](int bat) {
      if (variant == 0) inv_reg<<<(bat + 7) / 8, 256>>>(dA, dR, dP, bat);
      else inv_blk<<<(bat + 3) / 4, 128>>>(dA, dR, dP, bat);
    };
    run(batch);
    cudaDeviceSynchronize();
    cudaMemcpy(R.data(), dR, R.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(P.data(), dP, P.size() * 4, cudaMemcpyDeviceToHost);
    check(variant ? "blk" : "reg", A, R, P, batch);
    for (int bat : {148 * 8, batch}) {  // one CTA (8 warps) per SM, and 8 CTAs per SM
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        run(bat);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = fminf(best, ms);
      }
      printf("%s batch %6d: %.3f ms  %.2f M inversions/s\n", variant ? "blk" : "reg", bat, best, bat / best / 1e3);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
