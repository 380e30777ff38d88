// Shared device helpers for the logm kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/logmpoly_b200.h"
#include "lgm_constants.h"

// process-wide count of kernels launched by this library (lgm_launch_count in the ABI)
int lgm_count_launch();

#define LGM_UNIT_ROUNDOFF 1.1102230246251565e-16  // 2^-53 (matcore.py:19-20)
#define LGM_SCALING_SWITCH 1e-2                   // sqrtm.py:21
#define LGM_MU_MIN 1e-8                           // sqrtm.py:24
#define LGM_MU_MAX 1e8
#define LGM_FUSED_WS 8                            // Engine F workspace: n^2 slots per matrix

// Everything the driver needs besides the matrices; passed by value as a kernel parameter.
struct LgmParams {
  int max_k, maxiter_s, db_maxiter, est_itmax, balance;
  int cplx;       // input = real 2n x 2n embeddings of n x n complex matrices (decisions on Z)
  double db_tol;  // 0 -> 10 n u
  double theta[LGM_K_MAX];
  int order[LGM_K_MAX];
  int coef_off[LGM_K_MAX];
  double coef[LGM_NCOEF];
};

// Scheme k (1-based) coefficient rows, layout written by tools/gen_constants.py:
// lhs rows j = 0..k-1 (j+2 entries), rhs rows, out (k+2 entries).
__host__ __device__ __forceinline__ const double* lgm_lhs(const LgmParams& p, int k, int j) {
  return p.coef + p.coef_off[k - 1] + j * (j + 3) / 2;
}
__host__ __device__ __forceinline__ const double* lgm_rhs(const LgmParams& p, int k, int j) {
  return p.coef + p.coef_off[k - 1] + k * (k + 3) / 2 + j * (j + 3) / 2;
}
__host__ __device__ __forceinline__ const double* lgm_out(const LgmParams& p, int k) {
  return p.coef + p.coef_off[k - 1] + k * (k + 3);
}

// Order-preserving key of a non-negative double (+1 so that "no candidate" = 0 is below
// every real value, including +0.0).
__device__ __forceinline__ uint64_t lgm_key(double nonneg) {
  return (uint64_t)__double_as_longlong(nonneg) + 1ull;
}
__device__ __forceinline__ double lgm_unkey(uint64_t key) {
  return __longlong_as_double((long long)(key - 1ull));
}

// Warp argmax over 64-bit keys; ties -> lowest lane.  Returns max key (0 if none).
__device__ __forceinline__ uint64_t lgm_warp_argmax(uint64_t key, int& lane_win) {
  const unsigned FULL = 0xffffffffu;
  unsigned hi = __reduce_max_sync(FULL, (unsigned)(key >> 32));
  unsigned lo = __reduce_max_sync(FULL, ((unsigned)(key >> 32) == hi) ? (unsigned)key : 0u);
  uint64_t kmax = ((uint64_t)hi << 32) | lo;
  unsigned b = __ballot_sync(FULL, key == kmax);
  lane_win = __ffs(b) - 1;
  return kmax;
}

static __device__ __noinline__ double lgm_div_slow(double x) { return 1.0 / x; }

// 1/x from the MUFU approximation refined by two Newton steps (<= 1 ulp; the Gauss-Jordan
// pivot reciprocal -- not bit-identical to the IEEE quotient, which the parity bar does not
// require of the inverse).  Zero, subnormal and non-finite x take the IEEE division.
__device__ __forceinline__ double lgm_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  // |x| < 2^-1022 (zero / subnormal, flushed by .ftz) or |x| >= 2^1021 (reciprocal near the
  // subnormal range) or inf / nan: IEEE division
  const unsigned hx = (unsigned)__double2hiint(x) & 0x7fffffffu;
  if (hx - 0x00100000u >= 0x7fc00000u - 0x00100000u) y = lgm_div_slow(x);
  return y;
}

// Cheap reciprocal for margin bookkeeping (relative error ~1e-7 is irrelevant there).
__device__ __forceinline__ double lgm_rcp_rough(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// FP64 tensor-core MMA (SASS DMMA.8x8x4): d[0..1] += A(8x4, row) * B(4x8, col); lane (g, t) =
// (lane / 4, lane % 4) supplies A[g][t] and B[t][g] and holds D[g][2t], D[g][2t + 1].
__device__ __forceinline__ void lgm_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double lgm_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double lgm_warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// numpy's pairwise summation for a 1-D reduction (numpy loops_utils.h pairwise_sum):
// n < 8 sequential from 0.0; n <= 128: 8 interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail sequentially; else split at
// n2 = n/2 - (n/2)%8 and recurse.  Used so that balancing decisions are bit-identical
// to matcore.py:194-195.  `get(i)` returns the i-th (already |.|'d) term.
template <class F>
__host__ __device__ inline double lgm_pairwise_block(F get, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += get(off + i);
    return r;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = get(off + q);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] += get(off + i + q);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += get(off + i);
  return res;
}

template <class F>
__host__ __device__ double lgm_pairwise_rec(F get, int off, int n) {
  if (n <= 128) return lgm_pairwise_block(get, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  double left = lgm_pairwise_rec(get, off, n2);
  return left + lgm_pairwise_rec(get, off + n2, n - n2);
}

template <class F>
__host__ __device__ inline double lgm_pairwise_sum(F get, int n) {
  return lgm_pairwise_rec(get, 0, n);
}
