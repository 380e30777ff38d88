// On-device spectrum pre-check (validation helper; eig_small, matcore.py:343-355; SPEC.md:448,
// 490): flags[b] = 1 when matrix b has an eigenvalue on the closed negative real axis (a real
// eigenvalue <= 0, where the principal logarithm does not exist), 0 otherwise, 2 when the QR
// iteration did not converge (eig_small raises ConvergenceError there).
//
// One CTA per matrix, the working copy in the caller's workspace (L1 / L2 resident):
//   1. Householder reduction to upper Hessenberg form (the whole CTA: column / row updates in
//      parallel, one reflector per column);
//   2. Francis implicit double-shift QR on the Hessenberg matrix, eigenvalues only (one warp:
//      the scalar shift / deflation logic on every lane, the 3-row / 3-column bulge updates
//      spread over the lanes), deflating 1 x 1 blocks (real eigenvalues) and 2 x 2 blocks
//      (a real pair when the discriminant is >= 0, else a complex pair), with exceptional
//      shifts every 10 iterations.
// As with LAPACK's dhseqr, a real eigenvalue comes out with an exactly zero imaginary part.
#include <cstdint>
#include <cuda_runtime.h>

#include "lgm_common.cuh"

namespace {

constexpr int SP_NT = 256;
constexpr int SP_MAXIT = 60;  // QR iterations per eigenvalue before giving up

__device__ double sp_block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < SP_NT / 32; ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(SP_NT) spectrum_kernel(const double* __restrict__ A, long long ld, int n,
                                                        double* ws, int* flags) {
  __shared__ double red[SP_NT / 32];
  extern __shared__ double v[];  // Householder vector (n) + product workspace (n)
  double* w = v + n;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  double* H = ws + (size_t)b * n * n;
  const double* Ab = A + (size_t)b * n * ld;
  for (size_t idx = tid; idx < (size_t)n * n; idx += SP_NT) {
    const int i = idx / n, j = idx - (size_t)i * n;
    H[idx] = Ab[(size_t)i * ld + j];
  }
  __syncthreads();
  // ---- 1. Hessenberg reduction: H <- Q^T H Q, reflector k annihilates H[k+2.., k]
  for (int k = 0; k + 2 < n; ++k) {
    double ss = 0.0;
    for (int i = k + 2 + tid; i < n; i += SP_NT) ss += H[(size_t)i * n + k] * H[(size_t)i * n + k];
    const double xn2 = sp_block_sum(ss, red);
    if (xn2 == 0.0) continue;
    const double alpha = H[(size_t)(k + 1) * n + k];
    const double beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
    const double tau = (beta - alpha) / beta;
    const double sc = 1.0 / (alpha - beta);
    for (int i = tid; i < n; i += SP_NT) v[i] = (i < k + 1) ? 0.0 : (i == k + 1 ? 1.0 : H[(size_t)i * n + k] * sc);
    __syncthreads();
    // left: rows k+1.. of columns k.. : H -= tau v (v^T H)
    for (int j = k + tid; j < n; j += SP_NT) {
      double d = 0.0;
      for (int i = k + 1; i < n; ++i) d += v[i] * H[(size_t)i * n + j];
      w[j] = tau * d;
    }
    __syncthreads();
    for (size_t idx = tid; idx < (size_t)(n - k - 1) * (n - k); idx += SP_NT) {
      const int i = k + 1 + (int)(idx / (n - k)), j = k + (int)(idx % (n - k));
      H[(size_t)i * n + j] -= v[i] * w[j];
    }
    __syncthreads();
    // right: all rows, columns k+1.. : H -= (H v) tau v^T
    for (int i = tid; i < n; i += SP_NT) {
      double d = 0.0;
      for (int j = k + 1; j < n; ++j) d += H[(size_t)i * n + j] * v[j];
      w[i] = tau * d;
    }
    __syncthreads();
    for (size_t idx = tid; idx < (size_t)n * (n - k - 1); idx += SP_NT) {
      const int i = (int)(idx / (n - k - 1)), j = k + 1 + (int)(idx % (n - k - 1));
      H[(size_t)i * n + j] -= w[i] * v[j];
    }
    __syncthreads();
    for (int i = k + 2 + tid; i < n; i += SP_NT) H[(size_t)i * n + k] = 0.0;
    __syncthreads();
  }
  if (tid >= 32) return;
  // ---- 2. Francis double-shift QR (eigenvalues only), one warp
  auto h = [&](int i, int j) -> double& { return H[(size_t)i * n + j]; };
  double anorm = 0.0;
  for (int i = lane; i < n; i += 32)
    for (int j = (i > 0 ? i - 1 : 0); j < n; ++j) anorm += fabs(h(i, j));
  for (int o = 16; o > 0; o >>= 1) anorm += __shfl_xor_sync(0xffffffffu, anorm, o);
  __syncwarp();
  int bad = 0;
  double t = 0.0;
  int nn = n - 1;
  while (nn >= 0 && !bad) {
    int its = 0, l = 0;
    for (;;) {
      for (l = nn; l >= 1; --l) {  // a negligible subdiagonal splits the matrix
        double s = fabs(h(l - 1, l - 1)) + fabs(h(l, l));
        if (s == 0.0) s = anorm;
        if (fabs(h(l, l - 1)) + s == s) {
          __syncwarp();
          if (lane == 0) h(l, l - 1) = 0.0;
          __syncwarp();
          break;
        }
      }
      double x = h(nn, nn);
      if (l == nn) {  // one real root
        const double wr = x + t;
        if (wr <= 0.0) bad = 1;
        nn -= 1;
        break;
      }
      double y = h(nn - 1, nn - 1), wv = h(nn, nn - 1) * h(nn - 1, nn);
      if (l == nn - 1) {  // a 2 x 2 block
        const double p = 0.5 * (y - x), q = p * p + wv;
        double z = sqrt(fabs(q));
        x += t;
        if (q >= 0.0) {  // a real pair
          z = p + copysign(z, p);
          const double w1 = x + z, w2 = (z != 0.0) ? x - wv / z : x + z;
          if (w1 <= 0.0 || w2 <= 0.0) bad = 1;
        }
        nn -= 2;
        break;
      }
      if (its == SP_MAXIT) { bad = 2; break; }
      if (its == 10 || its == 20 || its == 40) {  // exceptional shift
        t += x;
        __syncwarp();
        for (int i = lane; i <= nn; i += 32) h(i, i) -= x;
        __syncwarp();
        const double s = fabs(h(nn, nn - 1)) + fabs(h(nn - 1, nn - 2));
        y = x = 0.75 * s;
        wv = -0.4375 * s * s;
      }
      ++its;
      int m;
      double p = 0.0, q = 0.0, r = 0.0, z;
      for (m = nn - 2; m >= l; --m) {  // two consecutive small subdiagonals?
        z = h(m, m);
        r = x - z;
        const double s0 = y - z;
        p = (r * s0 - wv) / h(m + 1, m) + h(m, m + 1);
        q = h(m + 1, m + 1) - z - r - s0;
        r = h(m + 2, m + 1);
        const double s = fabs(p) + fabs(q) + fabs(r);
        p /= s;
        q /= s;
        r /= s;
        if (m == l) break;
        const double u = fabs(h(m, m - 1)) * (fabs(q) + fabs(r));
        const double vv = fabs(p) * (fabs(h(m - 1, m - 1)) + fabs(z) + fabs(h(m + 1, m + 1)));
        if (u + vv == vv) break;
      }
      __syncwarp();
      for (int i = m + 2 + lane; i <= nn; i += 32) {
        h(i, i - 2) = 0.0;
        if (i != m + 2) h(i, i - 3) = 0.0;
      }
      __syncwarp();
      for (int k = m; k <= nn - 1; ++k) {  // chase the bulge
        if (k != m) {
          p = h(k, k - 1);
          q = h(k + 1, k - 1);
          r = (k != nn - 1) ? h(k + 2, k - 1) : 0.0;
          x = fabs(p) + fabs(q) + fabs(r);
          if (x != 0.0) {
            p /= x;
            q /= x;
            r /= x;
          }
        }
        const double s = copysign(sqrt(p * p + q * q + r * r), p);
        if (s == 0.0) continue;
        __syncwarp();
        if (lane == 0) {
          if (k == m) {
            if (l != m) h(k, k - 1) = -h(k, k - 1);
          } else {
            h(k, k - 1) = -s * x;
          }
        }
        p += s;
        x = p / s;
        y = q / s;
        z = r / s;
        q /= p;
        r /= p;
        __syncwarp();
        for (int j = k + lane; j <= nn; j += 32) {  // rows k, k+1, k+2
          double pp = h(k, j) + q * h(k + 1, j);
          if (k != nn - 1) {
            pp += r * h(k + 2, j);
            h(k + 2, j) -= pp * z;
          }
          h(k + 1, j) -= pp * y;
          h(k, j) -= pp * x;
        }
        __syncwarp();
        const int mmin = nn < k + 3 ? nn : k + 3;
        for (int i = l + lane; i <= mmin; i += 32) {  // columns k, k+1, k+2
          double pp = x * h(i, k) + y * h(i, k + 1);
          if (k != nn - 1) {
            pp += z * h(i, k + 2);
            h(i, k + 2) -= pp * r;
          }
          h(i, k + 1) -= pp * q;
          h(i, k) -= pp;
        }
        __syncwarp();
      }
    }
  }
  if (lane == 0) flags[b] = bad;
}

}  // namespace

extern "C" int lgm_spectrum_check_f64(const double* A, int32_t* flags, int64_t n, int64_t batch, int64_t ld,
                                      void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!A || !flags || n < 1 || batch < 0 || ld < n || batch > (int64_t)0x7fffffff) return LGM_ERR_ARG;
  if (batch == 0) return 0;
  if (!ws || ws_bytes < (size_t)batch * n * n * sizeof(double)) return LGM_ERR_WORKSPACE;
  const size_t smem = 2 * (size_t)n * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return LGM_ERR_CUDA;
  lgm_count_launch(), spectrum_kernel<<<(unsigned)batch, SP_NT, smem, (cudaStream_t)stream>>>(A, ld, (int)n,
                                                                                              (double*)ws, flags);
  return cudaGetLastError() == cudaSuccess ? 0 : LGM_ERR_CUDA;
}
