// C-ABI entry points (include/logmpoly_b200.h) and the kernels behind them.
//
// n <= 64: Engine F (lgm_fused.cuh), one CTA per matrix, the whole pipeline in one launch.
// n  > 64: Engine G (lgm_grid.cu), device-driven batched kernels in one CUDA graph per call
//          over a caller-owned workspace (lgm_workspace_bytes).
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "lgm_fused.cuh"
#include "lgm_grid.cuh"

using namespace lgm;

static std::atomic<long long> g_lgm_launches{0};
int lgm_count_launch() { g_lgm_launches.fetch_add(1, std::memory_order_relaxed); return 0; }

// ------------------------------------------------------------------------------ kernels

#ifndef LGM_F32_MINB
#define LGM_F32_MINB 8
#endif
template <int NMAX, bool FULL>
__global__ void __launch_bounds__(Cfg<NMAX>::NT, NMAX == 32 ? LGM_F32_MINB : 1) logm_fused_kernel(const double* __restrict__ A, double* __restrict__ L,
                                                                  lgm_report* rep, long long ld, int n, double* ws,
                                                                  long long wst, const __grid_constant__ LgmParams P) {
  extern __shared__ __align__(16) double smem[];
  Ctx<NMAX, FULL> c;
  c.init(smem, n, &P);
  const long long b = blockIdx.x;
  logm_one<NMAX, FULL>(c, A + b * n * ld, L + b * n * ld, ld, rep + b, ws + b * wst);
}

// Engine F workspace stride per matrix (doubles): LGM_FUSED_WS n^2 (+ the LGM_WS_GUARD band)
static long long fused_wst(int64_t n) { return (long long)LGM_FUSED_WS * n * n + (long long)(lgm_ws_guard_bytes() / 8); }

// guard bands after each matrix's Engine F workspace: check = 0 fills (0xA5 bytes), 1 counts
__global__ void fused_guard_kernel(unsigned long long* ws, long long n2, long long wst, long long batch, int check,
                                   unsigned long long* bad) {
  const long long gw = wst - n2;
  unsigned long long nbad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < batch * gw; i += (long long)gridDim.x * blockDim.x) {
    const long long at = (i / gw) * wst + n2 + i % gw;
    if (check) nbad += ws[at] != 0xA5A5A5A5A5A5A5A5ull;
    else ws[at] = 0xA5A5A5A5A5A5A5A5ull;
  }
  if (check && nbad) atomicAdd(bad, nbad);
}

template <int NMAX>
__global__ void __launch_bounds__(Cfg<NMAX>::NT) sqrt_db_kernel(const double* __restrict__ A, double* __restrict__ X,
                                                               long long ld, int n, double tol, int maxiter,
                                                               int* iters, int* status, const __grid_constant__ LgmParams P) {
  extern __shared__ __align__(16) double smem[];
  Ctx<NMAX> c;
  c.init(smem, n, &P);
  const long long b = blockIdx.x;
  c.zero_all();
  __syncthreads();
  int st = 0, its = 0;
  if (c.load(0, A + b * n * ld, ld)) st = LGM_NONFINITE;
  else st = c.sqrt_db(0, 1, tol > 0.0 ? tol : 10.0 * n * LGM_UNIT_ROUNDOFF, maxiter, its);
  __syncthreads();
  c.store(0, X + b * n * ld, ld);
  if (c.tid == 0) { iters[b] = its; status[b] = st; }
}

template <int NMAX>
__global__ void __launch_bounds__(Cfg<NMAX>::NT) est_kernel(const double* __restrict__ M1, int p1,
                                                           const double* __restrict__ M2, long long ld, int n,
                                                           int itmax, int zero_shortcut, double* est, int* passes,
                                                           const __grid_constant__ LgmParams P) {
  extern __shared__ __align__(16) double smem[];
  Ctx<NMAX> c;
  c.init(smem, n, &P);
  const long long b = blockIdx.x;
  c.zero_all();
  __syncthreads();
  typedef typename Ctx<NMAX>::MRef MR;
  const MR m1{const_cast<double*>(M1) + b * n * ld, (int)ld};
  const MR m2{M2 ? const_cast<double*>(M2) + b * n * ld : nullptr, (int)ld};
  int ps = 0;
  double e = 0.0;
  bool go = true;
  c.init_ramp();
  if (zero_shortcut) go = c.any_nonzero_ref(m1);  // matcore.py:309-310
  if (go) e = c.estimate(m1, p1, M2 != nullptr, m2, itmax, ps);
  if (c.tid == 0) { est[b] = e; passes[b] = ps; }
}

template <int NMAX>
__global__ void __launch_bounds__(Cfg<NMAX>::NT) balance_kernel(const double* __restrict__ A, double* __restrict__ B,
                                                               double* scale, long long ld, int n, int max_sweeps,
                                                               int* sweeps, const __grid_constant__ LgmParams P) {
  extern __shared__ __align__(16) double smem[];
  Ctx<NMAX> c;
  c.init(smem, n, &P);
  const long long b = blockIdx.x;
  c.zero_all();
  __syncthreads();
  c.load(0, A + b * n * ld, ld);
  int sw = c.balance(0, max_sweeps);
  c.store(0, B + b * n * ld, ld);
  for (int i = c.tid; i < n; i += Cfg<NMAX>::NT) scale[b * n + i] = c.scale()[i];
  if (c.tid == 0) sweeps[b] = sw;
}

template <int NMAX>
__global__ void __launch_bounds__(Cfg<NMAX>::NT) degopt_kernel(const double* __restrict__ X, const double* __restrict__ FP,
                                                              double* __restrict__ Z, long long ld, int n, int k,
                                                              int* products, const __grid_constant__ LgmParams P) {
  extern __shared__ __align__(16) double smem[];
  Ctx<NMAX> c;
  c.init(smem, n, &P);
  const long long b = blockIdx.x;
  c.zero_all();
  __syncthreads();
  c.load(BUF_B, X + b * n * ld, ld);
  // P3 (the first product) and P4..P6 in the extra shared buffers of this kernel
  typedef typename Ctx<NMAX>::MRef MR;
  const MR p3{c.sm() + Cfg<NMAX>::SMEM_DOUBLES, Cfg<NMAX>::LDM};
  if (FP) {
    for (int i = c.warp; i < n; i += Cfg<NMAX>::NT / 32)
      for (int j = c.lane; j < n; j += 32) p3.p[i * Cfg<NMAX>::LDM + j] = FP[b * n * ld + (long long)i * ld + j];
  }
  for (int i = c.tid; i < n; i += Cfg<NMAX>::NT) c.scale()[i] = 1.0;
  __syncthreads();
  int prods = 0;
  c.degopt(k, BUF_B, p3, FP != nullptr, BUF_Y, c.sm() + Cfg<NMAX>::SMEM_DOUBLES + Cfg<NMAX>::MAT, Cfg<NMAX>::LDM, Cfg<NMAX>::MAT, 1.0,
           false, Z + b * n * ld, ld, prods);
  if (c.tid == 0) products[b] = prods;
}

// ------------------------------------------------------------------------------ host side

static void fill_params(LgmParams& P, const lgm_opts* o) {
  lgm_opts d;
  lgm_default_opts(&d);
  if (!o) o = &d;
  P.max_k = o->max_k;
  P.maxiter_s = o->maxiter_s;
  P.db_maxiter = o->db_maxiter;
  P.est_itmax = o->est_itmax;
  P.balance = o->balance;
  P.cplx = o->embedded_complex ? 1 : 0;
  P.db_tol = o->db_tol;
  for (int k = 0; k < LGM_K_MAX; ++k) {
    P.theta[k] = (o->theta && k < o->max_k) ? o->theta[k] : LGM_THETA_DEFAULT[k];
    P.order[k] = LGM_ORDER_DEFAULT[k];
    P.coef_off[k] = LGM_COEF_OFFSET[k];
  }
  std::memcpy(P.coef, LGM_COEF_DEFAULT, sizeof(P.coef));
}

static int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::fprintf(stderr, "logmpoly_b200: CUDA error %s\n", cudaGetErrorString(e));
    return LGM_ERR_CUDA;
  }
  return 0;
}

template <int NMAX, class K>
static int prep(K kernel, size_t bytes = Cfg<NMAX>::SMEM_BYTES) {
  static_assert(Cfg<NMAX>::SMEM_BYTES_X <= 227 * 1024, "shared memory budget");
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return e == cudaSuccess ? 0 : LGM_ERR_CUDA;
}

static bool args_ok(const void* p, int64_t n, int64_t batch, int64_t ld) {
  return p && n >= 1 && batch >= 0 && ld >= n && batch <= (int64_t)0x7fffffff;
}

template <int NMAX, bool FULL>
static int launch_fused(const double* A, double* L, lgm_report* rep, int64_t ld, int64_t n, int64_t batch, void* ws,
                        const LgmParams& P, cudaStream_t s) {
  // LGM_F_SMEM=<bytes>: launch with at least that much dynamic shared memory (caps the
  // resident CTAs per SM; occupancy A/B experiments only)
  static const size_t sm_bytes = [] {
    const char* e = std::getenv("LGM_F_SMEM");
    const size_t want = e ? (size_t)std::atol(e) : 0;
    return want > Cfg<NMAX>::SMEM_BYTES ? want : Cfg<NMAX>::SMEM_BYTES;
  }();
  if (prep<NMAX>(logm_fused_kernel<NMAX, FULL>, sm_bytes)) return LGM_ERR_CUDA;
  const long long wst = fused_wst(n);
  if (lgm_ws_guard_bytes())
    fused_guard_kernel<<<256, 256, 0, s>>>((unsigned long long*)ws, (long long)LGM_FUSED_WS * n * n, wst, batch, 0, nullptr);
  lgm_count_launch(), logm_fused_kernel<NMAX, FULL><<<(unsigned)batch, Cfg<NMAX>::NT, sm_bytes, s>>>(
                          A, L, rep, ld, (int)n, (double*)ws, wst, P);
  return check_launch();
}

extern "C" {

void lgm_default_opts(lgm_opts* o) {
  if (!o) return;
  o->max_k = LGM_K_DEFAULT;
  o->maxiter_s = 40;
  o->db_maxiter = 50;
  o->est_itmax = 5;
  o->balance = 1;
  o->embedded_complex = 0;
  o->db_tol = 0.0;
  o->theta = nullptr;
}

#ifndef LGM_FUSED_MAX
#define LGM_FUSED_MAX 64
#endif
int lgm_max_fused_n(void) { return LGM_FUSED_MAX; }

// devices on which Engine G graphs have run (their device-side executed-kernel counters)
static std::atomic<unsigned long long> g_grid_devs{0};
static void note_grid_device() {
  int d = 0;
  if (cudaGetDevice(&d) == cudaSuccess && d < 64) g_grid_devs.fetch_or(1ull << d, std::memory_order_relaxed);
}

// Direct launches (Engine F, graph setup kernels) + kernels executed inside Engine G graphs
// (counted on the device by the graphs' decide kernels; read back synchronously -- call it
// after synchronising, as bench.py does).
long long lgm_launch_count(void) {
  long long v = g_lgm_launches.load(std::memory_order_relaxed);
  const unsigned long long m = g_grid_devs.load(std::memory_order_relaxed);
  if (m) {
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < 64; ++d)
      if ((m >> d) & 1ull) {
        if (cudaSetDevice(d) == cudaSuccess) v += (long long)lgm_grid_exec_nodes();
      }
    cudaSetDevice(cur);
  }
  return v;
}

// Engine G launches index matrices (and their X / Y inversion jobs) in grid.y / grid.z, so a
// larger batch runs as consecutive passes of at most this many matrices over one workspace.
// LGM_GRID_CHUNK overrides it (tests exercise the pass loop with tiny chunks).
static int64_t grid_chunk() {
  const char* e = std::getenv("LGM_GRID_CHUNK");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? (int64_t)v : (int64_t)16384;
}

int lgm_workspace_bytes(int64_t n, int64_t batch, size_t* bytes) {
  if (!bytes || n < 1 || batch < 0) return LGM_ERR_ARG;
  // n <= 64: LGM_FUSED_WS n^2 doubles per matrix: polynomial nodes P4..P10 and A_prev / A_I2
  // (only P4..P6 and A_I2 are touched with the shipped k <= 5 schemes: L2 resident)
  *bytes = n <= LGM_FUSED_MAX ? (size_t)batch * fused_wst(n) * sizeof(double)
                   : lgm_grid_workspace_bytes(n, batch < grid_chunk() ? batch : grid_chunk());
  return 0;
}

int lgm_block_workspace_bytes(int64_t n, int64_t batch, size_t* bytes) {
  if (!bytes || n < 1 || batch < 0) return LGM_ERR_ARG;
  // n <= 64 needs it only for eval_degopt with k > 5 (graph path); sized for every case
  *bytes = lgm_grid_workspace_bytes(n, batch < grid_chunk() ? batch : grid_chunk());
  return 0;
}

// n <= 64 building blocks run in one fused kernel without scratch (eval_degopt with k > 5
// excepted); everything else takes the caller's workspace
static bool block_ws_ok(int64_t n, int64_t batch, const void* ws, size_t ws_bytes, bool fused = true) {
  if (n <= LGM_FUSED_MAX && fused) return true;
  size_t need = 0;
  lgm_block_workspace_bytes(n, batch, &need);
  return ws && ws_bytes >= need;
}

int lgm_expm_ref_f64(const double* A, double* E, int64_t n, int64_t batch, int64_t ld, void* ws, size_t ws_bytes,
                     lgm_stream_t stream) {
  if (!args_ok(A, n, batch, ld) || !E || (const void*)E == (const void*)A) return LGM_ERR_ARG;
  if (batch == 0) return 0;
  if (!block_ws_ok(n, batch, ws, ws_bytes, false)) return LGM_ERR_WORKSPACE;
  note_grid_device();
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    const int rc = lgm_grid_expm(A + b0 * n * ld, E + b0 * n * ld, n, cnt, ld, ws, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

const char* lgm_status_string(int code) {
  switch (code) {
    case LGM_OK: return "ok";
    case LGM_SINGULAR: return "matrix is exactly singular (zero pivot) in a square-root step";
    case LGM_DB_NOCONV: return "square root did not converge (eigenvalues on the negative real axis?)";
    case LGM_SCALING_MAXITER: return "no convergence after maxiter square roots";
    case LGM_NONFINITE: return "non-finite entries (input, or overflow of the result)";
    case LGM_SPECTRUM: return "spectrum check failed";
    case LGM_ERR_ARG: return "invalid argument";
    case LGM_ERR_CUDA: return "CUDA error";
    case LGM_ERR_UNSUPPORTED: return "unsupported size";
    case LGM_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int lgm_logm_f64(const double* A, double* L, int64_t n, int64_t batch, int64_t ld, const lgm_opts* opts,
                 lgm_report* rep, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!args_ok(A, n, batch, ld) || !L || !rep || (const void*)L == (const void*)A) return LGM_ERR_ARG;
  LgmParams P;
  fill_params(P, opts);
  if (P.max_k < 1 || P.max_k > LGM_K_MAX || P.maxiter_s < 0 || P.db_maxiter < 1 || P.est_itmax < 1)
    return LGM_ERR_ARG;
  if (P.cplx && (n & 1)) return LGM_ERR_ARG;  // a complex embedding is 2m x 2m
  if (batch == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  size_t need = 0;
  if (P.cplx) lgm_block_workspace_bytes(n, batch, &need);  // always the graph engine
  else lgm_workspace_bytes(n, batch, &need);
  if (!ws || ws_bytes < need) return LGM_ERR_WORKSPACE;
  if (n <= LGM_FUSED_MAX && !P.cplx) {
    // FULL instantiations (n == NMAX) carry n as a compile-time constant
    const bool full = (n == 32 || n == 64);
    if (n <= 32)
      return full ? launch_fused<32, true>(A, L, rep, ld, n, batch, ws, P, s)
                  : launch_fused<32, false>(A, L, rep, ld, n, batch, ws, P, s);
    return full ? launch_fused<64, true>(A, L, rep, ld, n, batch, ws, P, s)
                : launch_fused<64, false>(A, L, rep, ld, n, batch, ws, P, s);
  }
  note_grid_device();
  const int64_t ch = grid_chunk();
  for (int64_t b0 = 0; b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    const int rc = lgm_grid_logm(A + b0 * n * ld, L + b0 * n * ld, n, cnt, ld, P, rep + b0, ws, s);
    if (rc) return rc;
  }
  return 0;
}

#define LGM_DISPATCH_SMALL(KERNEL, ...)                                                                  \
  do {                                                                                                   \
    if (n <= 32) {                                                                                       \
      if (prep<32>(KERNEL<32>)) return LGM_ERR_CUDA;                                                     \
      lgm_count_launch(), KERNEL<32><<<(unsigned)batch, Cfg<32>::NT, Cfg<32>::SMEM_BYTES, (cudaStream_t)stream>>>(__VA_ARGS__); \
      return check_launch();                                                                             \
    }                                                                                                    \
    if (n <= 64) {                                                                                       \
      if (prep<64>(KERNEL<64>)) return LGM_ERR_CUDA;                                                     \
      lgm_count_launch(), KERNEL<64><<<(unsigned)batch, Cfg<64>::NT, Cfg<64>::SMEM_BYTES, (cudaStream_t)stream>>>(__VA_ARGS__); \
      return check_launch();                                                                             \
    }                                                                                                    \
  } while (0)

int lgm_sqrt_db_f64(const double* A, double* X, int64_t n, int64_t batch, int64_t ld, double tol, int32_t maxiter,
                    int32_t* iters, int32_t* status, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!args_ok(A, n, batch, ld) || !X || !iters || !status || maxiter < 1) return LGM_ERR_ARG;
  if (!block_ws_ok(n, batch, ws, ws_bytes)) return LGM_ERR_WORKSPACE;
  if (batch == 0) return 0;
  LgmParams P;
  fill_params(P, nullptr);
  LGM_DISPATCH_SMALL(sqrt_db_kernel, A, X, ld, (int)n, tol, maxiter, iters, status, P);
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    note_grid_device();
    const int rc = lgm_grid_sqrt_db(A + b0 * n * ld, X + b0 * n * ld, n, cnt, ld, tol, maxiter, iters + b0,
                                    status + b0, ws, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int lgm_est_power_norm_f64(const double* M, int64_t n, int64_t batch, int64_t ld, int32_t p, int32_t itmax,
                           double* est, int32_t* passes, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!args_ok(M, n, batch, ld) || !est || !passes || p < 1 || itmax < 1) return LGM_ERR_ARG;
  if (!block_ws_ok(n, batch, ws, ws_bytes)) return LGM_ERR_WORKSPACE;
  if (batch == 0) return 0;
  LgmParams P;
  fill_params(P, nullptr);
  LGM_DISPATCH_SMALL(est_kernel, M, p, (const double*)nullptr, ld, (int)n, itmax, 1, est, passes, P);
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    note_grid_device();
    const int rc = lgm_grid_est(M + b0 * n * ld, p, nullptr, n, cnt, ld, itmax, 1, est + b0, passes + b0, ws,
                                (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int lgm_est_product_norm_f64(const double* M1, int32_t p1, const double* M2, int64_t n, int64_t batch, int64_t ld,
                             int32_t itmax, double* est, int32_t* passes, void* ws, size_t ws_bytes,
                             lgm_stream_t stream) {
  if (!args_ok(M1, n, batch, ld) || !est || !passes || p1 < 1 || itmax < 1) return LGM_ERR_ARG;
  if (!block_ws_ok(n, batch, ws, ws_bytes)) return LGM_ERR_WORKSPACE;
  if (batch == 0) return 0;
  LgmParams P;
  fill_params(P, nullptr);
  LGM_DISPATCH_SMALL(est_kernel, M1, p1, M2, ld, (int)n, itmax, 0, est, passes, P);
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    note_grid_device();
    const int rc = lgm_grid_est(M1 + b0 * n * ld, p1, M2 ? M2 + b0 * n * ld : nullptr, n, cnt, ld, itmax, 0,
                                est + b0, passes + b0, ws, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int lgm_balance_f64(const double* A, double* B, double* scale, int64_t n, int64_t batch, int64_t ld,
                    int32_t max_sweeps, int32_t* sweeps, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!args_ok(A, n, batch, ld) || !B || !scale || !sweeps || max_sweeps < 1) return LGM_ERR_ARG;
  if (!block_ws_ok(n, batch, ws, ws_bytes)) return LGM_ERR_WORKSPACE;
  if (batch == 0) return 0;
  LgmParams P;
  fill_params(P, nullptr);
  LGM_DISPATCH_SMALL(balance_kernel, A, B, scale, ld, (int)n, max_sweeps, sweeps, P);
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    note_grid_device();
    const int rc = lgm_grid_balance(A + b0 * n * ld, B + b0 * n * ld, scale + b0 * n, n, cnt, ld, max_sweeps,
                                    sweeps + b0, ws, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

// eval_degopt for scheme k: the shipped coefficients, or (coef != NULL) the caller's scheme with
// k products in the same layout (lhs rows j = 0..k-1 with j + 2 entries, rhs rows, out k + 2),
// which takes the place of scheme k in the parameter block
static int degopt_impl(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld, int32_t k,
                       const double* coef, int32_t* products, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  if (!args_ok(X, n, batch, ld) || !Z || !products || k < 1 || k > LGM_K_MAX) return LGM_ERR_ARG;
  const bool fused = n <= LGM_FUSED_MAX && k <= 5;  // node storage of the fused kernel: P4..P6
  if (!block_ws_ok(n, batch, ws, ws_bytes, fused)) return LGM_ERR_WORKSPACE;
  if (batch == 0) return 0;
  LgmParams P;
  fill_params(P, nullptr);
  if (coef) {
    const int len = k * (k + 3) + k + 2;
    for (int i = 0; i < len; ++i)
      if (!std::isfinite(coef[i])) return LGM_ERR_ARG;
    std::memcpy(P.coef + P.coef_off[k - 1], coef, (size_t)len * sizeof(double));
  }
  if (fused && n <= 32) {
    if (prep<32>(degopt_kernel<32>, Cfg<32>::SMEM_BYTES_X)) return LGM_ERR_CUDA;
    lgm_count_launch(), degopt_kernel<32><<<(unsigned)batch, Cfg<32>::NT, Cfg<32>::SMEM_BYTES_X, (cudaStream_t)stream>>>(X, FP, Z, ld, (int)n,
                                                                                                  k, products, P);
    return check_launch();
  }
  if (fused) {
    if (prep<64>(degopt_kernel<64>, Cfg<64>::SMEM_BYTES_X)) return LGM_ERR_CUDA;
    lgm_count_launch(), degopt_kernel<64><<<(unsigned)batch, Cfg<64>::NT, Cfg<64>::SMEM_BYTES_X, (cudaStream_t)stream>>>(X, FP, Z, ld, (int)n,
                                                                                                  k, products, P);
    return check_launch();
  }
  for (int64_t b0 = 0, ch = grid_chunk(); b0 < batch; b0 += ch) {
    const int64_t cnt = batch - b0 < ch ? batch - b0 : ch;
    note_grid_device();
    const int rc = lgm_grid_degopt(X + b0 * n * ld, FP ? FP + b0 * n * ld : nullptr, Z + b0 * n * ld, n, cnt, ld, k,
                                   products + b0, P, ws, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int lgm_eval_degopt_f64(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld, int32_t k,
                        int32_t* products, void* ws, size_t ws_bytes, lgm_stream_t stream) {
  return degopt_impl(X, FP, Z, n, batch, ld, k, nullptr, products, ws, ws_bytes, stream);
}

int lgm_eval_degopt_scheme_f64(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld,
                               int32_t k, const double* coef, int32_t* products, void* ws, size_t ws_bytes,
                               lgm_stream_t stream) {
  if (!coef) return LGM_ERR_ARG;
  return degopt_impl(X, FP, Z, n, batch, ld, k, coef, products, ws, ws_bytes, stream);
}

// Diagnostics (LGM_WS_GUARD=1 only): the guard bands after every workspace region / slot.
// check = 0 fills them with the pattern (the library also does so before each call that uses
// the layout); check = 1 adds to *bad (device pointer) the number of guard bytes that no
// longer hold it, i.e. out-of-bounds writes by the calls since the fill.  layout 1: the
// lgm_logm_f64 workspace for n <= 64 (Engine F); 0: the Engine G / building-block workspace.
// Returns 1 if done, 0 if guards are off.
int lgm_debug_ws_guard(int64_t n, int64_t batch, int layout, void* ws, int check, unsigned long long* bad,
                       lgm_stream_t stream) {
  if (!lgm_ws_guard_bytes()) return 0;
  if (!ws || (check && !bad) || n < 1 || batch < 1) return LGM_ERR_ARG;
  if (layout == 1) {
    fused_guard_kernel<<<256, 256, 0, (cudaStream_t)stream>>>((unsigned long long*)ws, (long long)LGM_FUSED_WS * n * n,
                                                                fused_wst(n), batch, check, bad);
    return cudaGetLastError() == cudaSuccess ? 1 : LGM_ERR_CUDA;
  }
  const int rc = lgm_grid_ws_guard(n, batch < grid_chunk() ? batch : grid_chunk(), ws, check, bad, (cudaStream_t)stream);
  return rc < 0 ? rc : 1;
}

}  // extern "C"

#ifdef LGM_PHASE_PROF
extern "C" int lgm_debug_phase_cycles(unsigned long long* out8, int reset) {
  if (cudaMemcpyFromSymbol(out8, lgm::lgm_phase_cycles, 8 * sizeof(unsigned long long)) != cudaSuccess) return -2;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(lgm::lgm_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif
