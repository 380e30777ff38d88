// Engine G: Algorithm 1 for n > 64 as host-orchestrated batched kernels.
//
// Every matrix of the batch owns NBUF n x n slots of the caller's workspace.  The host
// runs the (uniform-across-matrices) control flow of oracle/driver.py in C++, keeping
// per-matrix decisions exactly as the restated Algorithm 1 and reading back only
// per-matrix scalars (norms, estimates, DB relative changes).  The O(n^3) work runs in
// batched kernels over the active matrices:
//   * gj_panel_kernel + gj_update_kernel: blocked pivoted Gauss-Jordan inversion (NB = 32
//     panels; trailing rank-NB updates on FP64 tensor cores, mma.sync m8n8k4 -> DMMA);
//   * db_update_kernel: fused scaled-DB update + column sums of |X'-X|, |X'|;
//   * est_*: the block 1-norm estimator (matcore.py:234-297) with on-device decisions;
//   * gemm_comb_kernel: graph-polynomial GEMMs with the left linear combination fused into
//     the A-tile load (schemes.py:91-126);
//   * balance_kernel / onenorm_kernel: numpy-order reductions (bit-identical decisions).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lgm_grid.cuh"

namespace {

constexpr int NB = 32;      // Gauss-Jordan panel width
#ifndef G2_RT
#define G2_RT 64            // rows per tile of the rank-64 combined pass (64: 4 warps; 128 measured equal)
#endif
constexpr int NBUF = 14;    // n x n slots per matrix (P8..P11: schemes k = 6..9; Q0/Q1: operand ping-pong)
static_assert(LGM_K_MAX <= 9, "node slots P2..P11 cover k <= 9");
enum { G_B = 0, G_Y, G_XI, G_YI, G_AP, G_AM, G_P6, G_P7, G_P8, G_P9, G_P10, G_P11, G_Q0, G_Q1 };

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "logmpoly_b200 grid: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return LGM_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

// G1 (one CTA per inversion) or G2 (per-panel kernels, rank-64 combined passes)?  Measured at
// config 4 (n = 512, 512 jobs per DB step): G2 with single-CTA panels 441 ms vs G1 452 ms;
// at n = 128 G1 (57 ms) beats G2 (81 ms).  By n only, so a matrix's arithmetic does not depend
// on the batch it is in.  LGM_G1_MAXN=<m> overrides: G1 exactly for n <= m (m <= 512).
bool use_g1(int n) {
  static const int v = [] {  // thread-safe once-init
    const char* e = std::getenv("LGM_G1_MAXN");
    return e ? std::min(512, std::max(0, std::atoi(e))) : -1;
  }();
  if (v >= 0) return n <= v;
  return n <= 256 || (n <= 512 && n % 64 != 0);
}

// Out-of-place inversion (the job reads its matrix from Src, no copy pass): G1, and G2 with
// single-CTA panels and rank-64 passes (n <= 512, n % 64 == 0) whose first pair reads the
// columns not yet written from Src.
bool inv_oop(int n) { return use_g1(n) || (n <= 512 && n % 64 == 0 && !(std::getenv("LGM_G2_RANK64") && std::getenv("LGM_G2_RANK64")[0] == '0')); }

// Cluster-resident estimator for EST_FUSED_MAXN < n <= 512, opt-in (LGM_EST_CLUSTER=1): bit-
// identical to the per-step kernels; at config 4 it measured 6.4 ms per 256-job estimate (round 1
// design: 14.8 ms) against 5.0 ms for the per-step kernels -- only 8 clusters of 16 CTAs run at
// once and each job's ~42 dependent thin products serialise on shared-memory bandwidth, DSMEM
// pushes and cluster barriers
bool est_cluster_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_EST_CLUSTER");
    return e && e[0] == '1';
  }();
  return on;
}

// G3 warp-specialised inverter (gj_inv_ws_kernel) for 256 < n <= 512, n % 64 == 0 (LGM_G3=0/1)
bool g3_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_G3");
    return e && e[0] == '1';
  }();
  return on;
}

// Lazy X^-1 on predicted-last DB iterations (LGM_LAZYX=0 disables; LGM_LAZYX_F = prediction
// factor f: predict when rel <= f sqrt(tol))
bool lazyx_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_LAZYX");
    return !(e && e[0] == '0');
  }();
  return on;
}
double lazyx_f() {
  static const double v = [] {
    const char* e = std::getenv("LGM_LAZYX_F");
    return e ? std::atof(e) : 1.0;
  }();
  return v;
}

// Single-K-half-slot combined pass (gj_update2s_kernel; LGM_UP2S=0 selects the one-shot kernel)
bool up2s_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_UP2S");
    return !(e && e[0] == '0');
  }();
  return on;
}

// G1 warp-level panels for n <= 128, n % 32 == 0 (gj_inv_cta_kernel<128, true>): opt-in with
// LGM_G1_WP=1.  Bit-identical to the block-level panels but measured slower (n = 128, 2048
// inversions: 1.44 vs 0.96 ms): one warp alone exposes every latency of its pivot steps.
bool g1_warp_panel_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_G1_WP");
    return e && e[0] == '1';
  }();
  return on;
}

#ifndef LGM_G1_PUBFIRST
#define LGM_G1_PUBFIRST 1
#endif
// Two-rows-per-thread pair panel for 256 < n <= 512 (gj_panel_pair2_kernel; LGM_PANEL2=0 selects
// the one-row-per-thread gj_panel_pair_kernel<512>; bit-identical results)
bool panel2_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_PANEL2");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One-launch estimator for n <= EST_FUSED_MAXN (LGM_EST_FUSED=0 selects the per-step kernels)
bool est_fused_on() {
  static const bool on = [] {  // thread-safe once-init
    const char* e = std::getenv("LGM_EST_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

__device__ __forceinline__ uint64_t dkey(double nonneg) { return (uint64_t)__double_as_longlong(nonneg) + 1ull; }

// Block-wide argmax of (key, index): max key, ties -> lowest index.  All threads get the result.
__device__ void block_argmax(uint64_t key, int idx, uint64_t* skey, int* sidx, uint64_t& kout, int& iout) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t k2 = __shfl_xor_sync(0xffffffffu, key, o);
    int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (k2 > key || (k2 == key && i2 < idx)) { key = k2; idx = i2; }
  }
  __syncthreads();
  if (lane == 0) { skey[warp] = key; sidx[warp] = idx; }
  __syncthreads();
  uint64_t kb = skey[0];
  int ib = sidx[0];
  for (int w = 1; w < nw; ++w) {
    if (skey[w] > kb || (skey[w] == kb && sidx[w] < ib)) { kb = skey[w]; ib = sidx[w]; }
  }
  kout = kb;
  iout = ib;
}

__device__ double block_sum(double v, double* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += sred[w];
  return s;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------------
// Shared DMMA tile core: C(64x64) += A(64x32, smem lda=36) * B(32x64, smem ldb=68).
// 4 warps; warp w owns rows (w/2)*32.., cols (w%2)*32..; acc[mi][ni][2] per lane.
constexpr int TM = 64, TN = 64, TK = 32, LDA_S = 36, LDB_S = 68;

__device__ __forceinline__ void tile_mma(const double* As, const double* Bs, double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 32, c0 = (warp & 1) * 32;
#pragma unroll
  for (int k = 0; k < TK; k += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = As[(r0 + mi * 8 + g) * LDA_S + k + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k + t) * LDB_S + c0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
}

// ------------------------------------------------------------------------------------------
// Batched pivoted Gauss-Jordan inversion.
struct InvJob {
  double* M;        // n x n row-major, inverted in place (storage permuted, see below)
  const double* Src;  // G1 only: if set, the first panel reads the matrix from here (M is
                      // written by then): out-of-place inversion without a copy pass
  int* piv;         // piv[k] = row chosen at step k
  int* rowstep;     // rowstep[i] = step at which row i became pivot (-1 = not yet)
  double* Wb;       // 6 NB x n buffers ("kinds") at stride wst: pivot-row snapshots W (kinds
  long long wst;    //  0/1: rank-32 look-ahead parities; rank-64 sets q: W1 = 3q, W2 = 3q+1)
                    //  and the first panel's multiplier copy A1 (n x NB, kind 3q+2)
  double* logdet;   // sum log|pivot|
  int* status;      // 0 ok, 1 exact zero pivot
};
__device__ __forceinline__ double* wkind(const InvJob& J, int k) { return J.Wb + (long long)k * J.wst; }
// After all panels, storage R satisfies R[piv[k]][j] = Minv[k][piv[j]], i.e.
// Minv[a][c] = R[piv[a]][rowstep[c]].

#ifdef LGM_PANEL_PROF
__device__ unsigned long long g_panel_cyc[12];  // load, stage-1, factor, store, CTAs; [6..8] panel2 step: search, publish, FMAs
#define PP_T(v) long long v = clock64()
#define PP_ADD(i, val) if (threadIdx.x == 0) atomicAdd(&g_panel_cyc[i], (unsigned long long)(val))
#else
#define PP_T(v)
#define PP_ADD(i, val)
#endif
// ------------------------------------------------------------------------------------------
// G1: the whole blocked Gauss-Jordan inversion of one matrix per CTA (64 < n <= NT <= 512).
// Thread `tid` owns row `tid` of the current 32-column panel in registers (static register
// indexing: the 32 pivot steps are unrolled); pivots by block argmax; the factored panel is
// staged in shared memory as the A operand of the trailing rank-32 update, which each warp
// applies to its 32 rows with DMMA (mma.sync m8n8k4 f64), column block by column block,
// with the pivot rows of the block snapshotted to shared memory first.  No host round trip
// or grid-level synchronisation per panel; one launch inverts every job of the batch.
constexpr int G1_LDA = 36;  // A panel row stride (bank-conflict free fragment loads)
constexpr int G1_LDW = 36;  // W chunk row stride

template <int NT>
struct G1Smem {
  static constexpr size_t A = 32 * (size_t)(NT + 4);  // doubles: panel stored transposed, row stride NT+4
  static constexpr size_t W = 2 * 32 * G1_LDW;  // double-buffered pivot-row snapshot
  static constexpr size_t PR = 2 * 40;
  static constexpr size_t bytes = (A + W + PR) * 8 + 2 * (size_t)NT * 4 + 64 * 16;
};

// G1 warp panel (n <= 128, n % 32 == 0; gj_inv_cta_kernel<128, true>): warp 0 factors the whole
// 32-column panel alone, lane l holding rows l, l + 32, l + 64, l + 96 of one 16-column half in
// registers.  The pivot search is a warp redux + shuffle -- no shared-memory exchange and no
// block barrier per pivot step (the block version spends ~1.7k cycles per step under load:
// two barriers, the key exchange, and the broadcast loads of a full 32-column pivot row per
// thread).  The 32 steps run as: 16 searched steps on columns 0-15 (multipliers g kept in
// shared memory), their replay on columns 16-31 (no search: stored g and pivot order), 16
// searched steps on columns 16-31, their replay on columns 0-15, then the deferred scaling of
// the panel's pivot rows.  Per element this is the block version's sequence of FMAs
// r <- fma(-g_k, p_k, r), k = 0..31, with the same g_k and pivot-row values: bit-identical.
// As: transposed panel As[c * lda + row]; Gs[16][128], pivval[128], rsc[128] live in the (idle)
// snapshot buffer.  Returns 1 on an exact zero pivot (warp-uniform).
__device__ __forceinline__ int g1_warp_panel(double* As, int lda, double* Gs, double* pivval, double* rsc, double* prow,
                                             int* rstep, int* piv, int n, int k0, int lane) {
  constexpr int H = 16;
  bool valid[4], used[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = lane + 32 * q;
    valid[q] = row < n;
    used[q] = valid[q] ? (rstep[row] >= 0) : true;
  }
  double x[4][H];
  auto load_half = [&](int h) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < H; ++j) x[q][j] = valid[q] ? As[(H * h + j) * lda + lane + 32 * q] : 0.0;
  };
  auto store_half = [&](int h) {  // with the deferred scaling of this panel's pivot rows
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!valid[q]) continue;
      const int row = lane + 32 * q;
      const int rs = rstep[row];
      const double sc = (rs >= k0 && rs < k0 + 32) ? rsc[row] : 1.0;
#pragma unroll
      for (int j = 0; j < H; ++j) As[(H * h + j) * lda + row] = (sc != 1.0) ? x[q][j] * sc : x[q][j];
    }
  };
  auto publish = [&](int slot, double* pw) {  // owner lane: its row `slot` of the live half
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (slot == q) {
#pragma unroll
        for (int j = 0; j < H; j += 2) *reinterpret_cast<double2*>(pw + j) = make_double2(x[q][j], x[q][j + 1]);
      }
  };
  auto replay = [&](int hs) {  // the 16 steps of half hs applied to the other half's columns (in x)
#pragma unroll 1
    for (int kk = 0; kk < H; ++kk) {
      const int p = piv[k0 + H * hs + kk];
      double* pw = prow + (kk & 1) * 40;
      if (lane == (p & 31)) publish(p >> 5, pw);
      __syncwarp();
      double g[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) g[q] = valid[q] ? Gs[kk * 128 + lane + 32 * q] : 0.0;
#pragma unroll
      for (int j = 0; j < H; j += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pw + j);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          x[q][j] = fma(-g[q], p2.x, x[q][j]);
          x[q][j + 1] = fma(-g[q], p2.y, x[q][j + 1]);
        }
      }
    }
  };
  auto search = [&](int h) -> int {  // 16 pivot steps on the live half (shift-in-FMA frame)
#pragma unroll 1
    for (int kk = 0; kk < H; ++kk) {
      double* pw = prow + (kk & 1) * 40;
      unsigned key = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double a = x[q][0];
        const bool cand = valid[q] && !used[q] && a != 0.0;
        const unsigned kq =
            cand ? ((((unsigned)__double2hiint(a) & 0x7fffffffu) & ~0x3ffu) | (unsigned)(1023 - (lane + 32 * q))) : 0u;
        key = kq > key ? kq : key;
      }
      const unsigned wk = __reduce_max_sync(0xffffffffu, key);
      if (wk == 0u) return 1;  // exact zero pivot (matcore.py:124-125)
      const int p = 1023 - (int)(wk & 0x3ffu);
      const int slot = p >> 5, ol = p & 31;
      const double asel = slot == 0 ? x[0][0] : (slot == 1 ? x[1][0] : (slot == 2 ? x[2][0] : x[3][0]));
      const double pv = __shfl_sync(0xffffffffu, asel, ol);
      if (lane == ol) {
        publish(slot, pw);
        rstep[p] = k0 + H * h + kk;
        piv[k0 + H * h + kk] = p;
        pivval[p] = pv;
      }
      const double rp = lgm_rcp(pv);
      if (lane == ol) rsc[p] = rp;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool own = (lane + 32 * q) == p;
        const double g = own ? 0.0 : x[q][0] * rp;
        const double last = own ? 1.0 : -g;
        if (valid[q]) Gs[kk * 128 + lane + 32 * q] = g;
        used[q] = used[q] || own;
#pragma unroll
        for (int c = 0; c < H; c += 2) {
          const double2 p2 = *reinterpret_cast<const double2*>(pw + c);
          if (c > 0) x[q][c - 1] = fma(-g, p2.x, x[q][c]);
          x[q][c] = fma(-g, p2.y, x[q][c + 1 < H ? c + 1 : c]);
        }
        x[q][H - 1] = last;
      }
    }
    return 0;
  };
  load_half(0);
  if (search(0)) return 1;
  // columns 0-15 wait (unscaled) in As for the second half's steps
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (valid[q]) {
#pragma unroll
      for (int j = 0; j < H; ++j) As[j * lda + lane + 32 * q] = x[q][j];
    }
  __syncwarp();
  load_half(1);
  replay(0);
  __syncwarp();  // replay's last reads of Gs before search overwrites it
  if (search(1)) return 1;
  __syncwarp();
  store_half(1);
  load_half(0);
  replay(1);
  store_half(0);
  return 0;
}

template <int NT, bool WP = false>
__global__ void __launch_bounds__(NT, WP ? 2 : 512 / NT) gj_inv_cta_kernel(const InvJob* jobs, int n) {
  extern __shared__ __align__(16) double g1sm[];
  double* As = g1sm;
  double* Ws = As + G1Smem<NT>::A;
  double* prow = Ws + G1Smem<NT>::W;                       // [2][40]: pivot row (32) + inv
  int* rstep = reinterpret_cast<int*>(prow + G1Smem<NT>::PR);  // [NT] rowstep
  int* piv = rstep + NT;                                   // [NT]
  unsigned long long* wkey = reinterpret_cast<unsigned long long*>(piv + NT);  // [2][16]
  double* wval = reinterpret_cast<double*>(wkey + 32);     // [2][16] exact signed pivot per warp
  unsigned* wkey32 = reinterpret_cast<unsigned*>(wkey);     // [2][16] per-warp best key

  const InvJob J = jobs[blockIdx.x];
  if (!J.M) return;  // unused slot of the device-built job table
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  double* M = J.M;
  for (int i = tid; i < NT; i += NT) rstep[i] = -1;
  if (tid < 80) prow[tid] = 0.0;  // pure-rotation steps read it with g = 0
  int my_step = -1;
  double mypiv = 1.0;   // this thread's pivot value (at most one); log|.| taken at the end
  int status = 0;
  __syncthreads();
  for (int k0 = 0; k0 < n && status == 0; k0 += 32) {
    const int nb = min(32, n - k0);
    double r[32];
    // (per-thread row loads: measured faster than staging through shared memory)
    // (the first panel reads the source matrix when inverting out of place: every element of
    // M is written during panel 0 -- K columns by the panel store, the rest by its update)
    const double* Mr = (k0 == 0 && J.Src) ? J.Src : M;
    PP_T(g0);
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      if (tid < n && c + 1 < nb && (n & 1) == 0) {
        const double2 v = *reinterpret_cast<const double2*>(&Mr[(size_t)tid * n + k0 + c]);
        r[c] = v.x;
        r[c + 1] = v.y;
      } else {
        r[c] = (tid < n && c < nb) ? Mr[(size_t)tid * n + k0 + c] : 0.0;
        r[c + 1] = (tid < n && c + 1 < nb) ? Mr[(size_t)tid * n + k0 + c + 1] : 0.0;
      }
    }
    double rowscale = 1.0;
    bool piv_here = false;
#ifdef LGM_PANEL_PROF
    long long g1 = clock64() + (__double_as_longlong(r[31]) & 0);
    PP_ADD(0, g1 - g0);
#endif
    if constexpr (WP) {
      // the panel moves to warp 0 through the transposed staging buffer and back
#pragma unroll
      for (int c = 0; c < 32; ++c) As[c * (NT + 4) + tid] = r[c];
      __syncthreads();
      if (warp == 0) {
        const int st = g1_warp_panel(As, NT + 4, Ws, Ws + 16 * 128, Ws + 17 * 128, prow, rstep, piv, n, k0, lane);
        if (lane == 0) wkey32[0] = (unsigned)st;
      }
      __syncthreads();
      if (wkey32[0]) status = 1;
      if (status == 0) {
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = As[c * (NT + 4) + tid];
        const int rs = rstep[tid];
        if (my_step < 0 && rs >= k0) {
          my_step = rs;
          mypiv = (Ws + 16 * 128)[tid];
        }
      }
    } else {
#pragma unroll 1
    for (int kk = 0; kk < 32; ++kk) {  // shift-in-FMA pivot frame: the pivot column is r[0]
      const int par = kk & 1;
      const double* pr = prow + par * 40;
      const double r0 = r[0];
      double g = 0.0, last = r0;       // kk >= nb: pure rotation
      if (kk < nb) {
        // single 32-bit key per level (see Engine F's gj_invert): high word of |r0| with its
        // 10 low bits replaced by 1023 - row -> threshold pivoting at 1 - 2^-10 (ties -> lowest
        // row); exact zeros excluded, so an all-zero key means a singular step
        const bool cand = (tid < n) && (my_step < 0) && r0 != 0.0;
        const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~0x3ffu) |
                                     (unsigned)(1023 - tid)) : 0u;
        const unsigned wk = __reduce_max_sync(0xffffffffu, key);
        const double wv = __shfl_sync(0xffffffffu, r0, (1023 - (int)(wk & 0x3ffu)) & 31);
        if (lane == 0) {
          wkey32[par * 16 + warp] = wk;
          wval[par * 16 + warp] = wv;
        }
        __syncthreads();
        // block max: lane w < NW holds warp w's key, one more redux
        const unsigned bk = __reduce_max_sync(0xffffffffu, lane < NW ? wkey32[par * 16 + lane] : 0u);
        if (bk == 0u) { status = 1; break; }  // exact zero pivot (matcore.py:124-125)
        const int p = 1023 - (int)(bk & 0x3ffu);
        double* pw = prow + par * 40;
        const bool own = (tid == p);
#if LGM_G1_PUBFIRST
        // the owner publishes first; the pivot's reciprocal (its slow-path call is a scheduling
        // barrier) follows, under the stores
        if (own) {
          my_step = k0 + kk;
          piv_here = true;
          mypiv = r0;
#pragma unroll
          for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r[c], r[c + 1]);
          rstep[tid] = k0 + kk;
          piv[k0 + kk] = tid;
        }
        const double rp = lgm_rcp(wval[par * 16 + (p >> 5)]);
        if (own) rowscale = rp;
        __syncthreads();
#else
        const double rp = lgm_rcp(wval[par * 16 + (p >> 5)]);
        if (own) {
          my_step = k0 + kk;
          piv_here = true;
          mypiv = r0;
          rowscale = rp;
#pragma unroll
          for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r[c], r[c + 1]);
          rstep[tid] = k0 + kk;
          piv[k0 + kk] = tid;
        }
        __syncthreads();
#endif
        g = own ? 0.0 : r0 * rp;
        last = own ? 1.0 : -g;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
        if (c > 0) r[c - 1] = fma(-g, p2.x, r[c]);
        r[c] = fma(-g, p2.y, r[c + 1]);
      }
      r[31] = last;
    }
    }  // !WP
#ifdef LGM_PANEL_PROF
    long long g2 = clock64() + (__double_as_longlong(r[30]) & 0);
    PP_ADD(2, g2 - g1);
#endif
    if (status) break;
    if (piv_here) {  // deferred scaling of this panel's pivot row
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] *= rowscale;
    }
    // factored panel -> global (K columns) and shared (A operand)
    if (tid < n) {
      if (nb == 32 && (n & 1) == 0) {  // 16-byte stores (row segment of 256 B per thread)
#pragma unroll
        for (int c = 0; c < 32; c += 2)
          *reinterpret_cast<double2*>(&M[(size_t)tid * n + k0 + c]) = make_double2(r[c], r[c + 1]);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nb) M[(size_t)tid * n + k0 + c] = r[c];
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) As[c * (NT + 4) + tid] = (c < nb) ? r[c] : 0.0;  // transposed: conflict-free
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) As[c * (NT + 4) + tid] = 0.0;
    }
    __syncthreads();
    // trailing update, column blocks of 32 outside the panel.  The pivot-row snapshot of
    // the next block is taken into the other half of Ws while the current block is updated
    // (one barrier per block); C fragments move as 16-byte accesses when n is even.
    const int g8 = lane >> 2, t4 = lane & 3;
    const int r0 = warp * 32;
    const bool vec = (n & 1) == 0;
    auto snap = [&](int jb, double* W) {
      for (int idx = tid; idx < 32 * 32; idx += NT) {
        const int c = idx >> 5, jj = idx & 31;
        W[c * G1_LDW + jj] = (c < nb && jb + jj < n) ? Mr[(size_t)piv[k0 + c] * n + jb + jj] : 0.0;
      }
    };
    // next block's snapshot: loads issued before the block's DMMA work, stored after it
    constexpr int SNP = (32 * 32 + NT - 1) / NT;
    auto snap_load = [&](int jb, double (&v)[SNP]) {
#pragma unroll
      for (int q = 0; q < SNP; ++q) {
        const int idx = tid + q * NT, c = idx >> 5, jj = idx & 31;
        v[q] = (idx < 1024 && c < nb && jb + jj < n) ? Mr[(size_t)piv[k0 + c] * n + jb + jj] : 0.0;
      }
    };
    auto snap_store = [&](const double (&v)[SNP], double* W) {
#pragma unroll
      for (int q = 0; q < SNP; ++q) {
        const int idx = tid + q * NT;
        if (idx < 1024) W[(idx >> 5) * G1_LDW + (idx & 31)] = v[q];
      }
    };
    int jcur = (k0 == 0) ? 32 : 0;
    int buf = 0;
    if (jcur < n) snap(jcur, Ws);
    __syncthreads();
    PP_T(g3);
    PP_ADD(3, g3 - g2);
    while (jcur < n) {
      int jnext = jcur + 32;
      if (jnext == k0) jnext += 32;
      double sv[SNP];
      if (jnext < n) snap_load(jnext, sv);
      const double* Wc = Ws + buf * 32 * G1_LDW;
      const int j0 = jcur;
      if (r0 < n) {
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int i = r0 + mi * 8 + g8;
          const int rs = (i < n) ? rstep[i] : -1;
          const bool live_row = i < n && !(rs >= k0 && rs < k0 + nb);
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int j = j0 + ni * 8 + 2 * t4;
            if (vec && live_row && j + 1 < n) {
              const double2 v = *reinterpret_cast<const double2*>(&Mr[(size_t)i * n + j]);
              acc[mi][ni][0] = v.x;
              acc[mi][ni][1] = v.y;
            } else {
#pragma unroll
              for (int e = 0; e < 2; ++e) acc[mi][ni][e] = (live_row && j + e < n) ? Mr[(size_t)i * n + j + e] : 0.0;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          double a[4], b[4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) a[mi] = As[(k + t4) * (NT + 4) + r0 + mi * 8 + g8];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) b[ni] = Wc[(k + t4) * G1_LDW + ni * 8 + g8];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int i = r0 + mi * 8 + g8;
          if (i >= n) continue;
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int j = j0 + ni * 8 + 2 * t4;
            if (vec && j + 1 < n) {
              *reinterpret_cast<double2*>(&M[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            } else {
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (j + e < n) M[(size_t)i * n + j + e] = acc[mi][ni][e];
            }
          }
        }
      }
      if (jnext < n) snap_store(sv, Ws + (buf ^ 1) * 32 * G1_LDW);
      __syncthreads();
      jcur = jnext;
      buf ^= 1;
    }
    PP_T(g4);
    PP_ADD(1, g4 - g3);
    PP_ADD(4, 1);
  }
  // publish pivots, log|det|, status
  for (int i = tid; i < n; i += NT) { J.piv[i] = piv[i]; J.rowstep[i] = rstep[i]; }
  double s = my_step >= 0 ? log(fabs(mypiv)) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __syncthreads();
  double* red = reinterpret_cast<double*>(prow);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < NW; ++w) tot += red[w];
    *J.logdet = tot;
    *J.status = status;
  }
}

__global__ void gj_init_kernel(const InvJob* jobs, int n) {
  const InvJob J = jobs[blockIdx.y];
  if (!J.M) return;  // unused slot of the device-built job table (its status reads 1)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) J.rowstep[i] = -1;
  if (blockIdx.x == 0 && threadIdx.x == 0) { *J.logdet = 0.0; *J.status = 0; }
}

// Factor the panel columns [k0, k0+nb) of every job: GJ elimination of the panel over all
// rows with partial pivoting among rows not yet used (ties -> lowest row).  The panel
// lives in shared memory (row stride NB+1) when it fits, else is updated in place.
// G2 panel (n > 512): one 8-CTA thread-block cluster per inversion.  CTA q of the cluster
// owns rows [q*rpc, (q+1)*rpc) of the 32-column panel, one row per thread in registers
// (shift-in-FMA pivot frame as in Engine F).  Per pivot step: block argmax, each CTA
// publishes its candidate (key, row values) in its own shared memory, one cluster barrier,
// every CTA reads the 8 candidates over DSMEM and applies the winner.  No grid-wide sync.
constexpr int CL = 8;
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(512, 1)
    gj_panel_cluster_kernel(const InvJob* jobs, int n, int k0, int nb) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ unsigned long long s_key[2];   // this CTA's best packed key per step parity
  __shared__ double s_cand[2][34];          // its candidate row (32) + exact pivot value
  __shared__ double s_prow[2][34];          // the cluster winner's row, local copy
  __shared__ unsigned long long s_wkey[2][16];
  __shared__ double s_red[16];
  __shared__ double s_tot;
  const int part = (int)cl.block_rank();
  const InvJob J = jobs[blockIdx.x / CL];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rpc = (n + CL - 1) / CL;
  const int row = part * rpc + tid;
  const bool valid = tid < rpc && row < n;
  const int st0 = *J.status;
  if (tid < 2 * 34) (&s_prow[0][0])[tid] = 0.0;  // pure-rotation steps read it with g = 0
  cl.sync();
  if (st0) return;  // whole cluster = this job: uniform
  PP_T(t0);
  double r[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) r[c] = (valid && c < nb) ? J.M[(size_t)row * n + k0 + c] : 0.0;
  bool used = valid ? (J.rowstep[row] >= 0) : true;
  bool piv_here = false;
#ifdef LGM_PANEL_PROF
  long long t1 = clock64() + (__double_as_longlong(r[31]) & 0);
  PP_ADD(0, t1 - t0);
#endif
  double rowscale = 1.0, mypiv = 1.0;
  int status = 0;
  // packed pivot key: high word of |r0|; low word with its 12 low bits replaced by 4095 - row
  // (ties and values equal to within 2^-40 go to the lowest row); exact zeros excluded
  auto pack = [&](double v, bool cand) -> unsigned long long {
    if (!cand || v == 0.0) return 0ull;
    const unsigned hi = (unsigned)__double2hiint(v) & 0x7fffffffu;
    const unsigned lo = ((unsigned)__double2loint(v) & ~0xfffu) | (unsigned)(4095 - row);
    return ((unsigned long long)hi << 32) | lo;
  };
  auto warp_max = [&](unsigned long long k) -> unsigned long long {
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
    return ((unsigned long long)hi << 32) | lo;
  };
#pragma unroll 1
  for (int kk = 0; kk < 32; ++kk) {
    const double r0 = r[0];
    double g = 0.0, last = r0;
    const int par = kk & 1;
    const double* pr = s_prow[par];
    if (kk < nb) {
      // block argmax: warp redux, then every warp reduces the 16 warp keys itself
      PP_T(ta);
      const unsigned long long wk = warp_max(pack(r0, valid && !used));
      if (lane == 0) s_wkey[par][warp] = wk;
      __syncthreads();
      PP_T(tb);
      PP_ADD(6, tb - ta);
      const unsigned long long bk = warp_max(lane < 16 ? s_wkey[par][lane] : 0ull);
      const int brow = 4095 - (int)(bk & 0xfffu);
      if (tid == 0) s_key[par] = bk;
      if (bk != 0ull && valid && row == brow) {  // publish this CTA's candidate row
#pragma unroll
        for (int c = 0; c < 32; ++c) s_cand[par][c] = r[c];
      }
      PP_T(tc0);
      cl.sync();
      PP_T(tc);
      PP_ADD(9, tc0 - tb);
      PP_ADD(7, tc - tc0);
      // cluster winner: lanes q < CL of every warp read CTA q's key over DSMEM
      const unsigned long long ck = warp_max(lane < CL ? *cl.map_shared_rank(&s_key[par], lane) : 0ull);
      if (ck == 0ull) { status = 1; break; }  // exact zero pivot (matcore.py:124-125)
      const int p = 4095 - (int)(ck & 0xfffu);
      if (tid < 32) s_prow[par][tid] = cl.map_shared_rank(&s_cand[par][0], p / rpc)[tid];
      __syncthreads();
      PP_T(td);
      PP_ADD(10, td - tc);
      const double rp = lgm_rcp(pr[0]);  // the winner's exact pivot (its row in its frame)
      const bool own = valid && (row == p);  // (idle threads' row ids alias other CTAs' rows)
      if (own) {
        used = true;
        piv_here = true;
        rowscale = rp;
        mypiv = r0;
        J.rowstep[row] = k0 + kk;
        J.piv[k0 + kk] = row;
      }
      g = own ? 0.0 : r0 * rp;
      last = own ? 1.0 : -g;
    }
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const double x = pr[j], y = pr[j + 1];
      if (j > 0) r[j - 1] = fma(-g, x, r[j]);
      r[j] = fma(-g, y, r[j + 1]);
    }
    r[31] = last;
  }
#ifdef LGM_PANEL_PROF
  long long t2 = clock64() + (__double_as_longlong(r[30]) & 0);
  PP_ADD(2, t2 - t1);
#endif
  if (status) {
    if (part == 0 && tid == 0) *J.status = 1;
    cl.sync();
    return;
  }
  // log|det| contribution of this panel's pivots: one log per pivot row, CTA sum, one atomic
  double lg = piv_here ? log(fabs(mypiv)) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
  if (lane == 0) s_red[warp] = lg;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 16; ++w) t += s_red[w];
    s_tot = t;
  }
  if (piv_here) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] *= rowscale;
  }
  if (valid) {
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < nb) J.M[(size_t)row * n + k0 + c] = r[c];
  }
  cl.sync();  // partial sums visible; peers' shared memory alive for the DSMEM reads
  if (part == 0 && tid == 0) {  // deterministic: CTA order
    double t = 0.0;
    for (int q = 0; q < CL; ++q) t += *cl.map_shared_rank(&s_tot, q);
    *J.logdet += t;
  }
  cl.sync();
#ifdef LGM_PANEL_PROF
  PP_T(t3);
  PP_ADD(3, t3 - t2);
  PP_ADD(4, 1);
#endif
}

// G2 panel for n <= 512 (many jobs): one CTA of NT >= n threads per inversion, row `tid`
// of the 32-column panel in registers, the pivot rule and shift-in-FMA frame of G1
// (gj_inv_cta_kernel).  No cluster: with hundreds of jobs the 8-CTA cluster panel's
// per-step cluster barriers serialise into many waves.
// s1_a1kind >= 0 (P2 of a rank-64 pair): the stage-1 update of P2's columns by P1 is applied
// to the loaded rows first (r <- z1 r + A1 W1[:, P2], FMA chain in c' order), replacing the
// narrow gj_update_kernel launch and its snapshot.
struct PanelSmem {
  double prow[2][40];
  unsigned wkey32[2][16];
  double wval[2][16];
  double red[16];
  int piv_s[32];
  double w1s[32][34];
#ifdef LGM_PANEL_1BAR
  double cand[2][16][32];  // every warp's candidate pivot row (one barrier per pivot step)
#endif
};
// Returns false when the panel hit an exact zero pivot (status set).
template <int NT>
__device__ __forceinline__ bool panel_body(const InvJob& J, int n, int k0, int nb, int a1_kind, int s1_a1kind,
                                           PanelSmem& ps, double* ptile) {
  constexpr int NW = NT / 32;
  auto& prow = ps.prow;
  auto& wkey32 = ps.wkey32;
  auto& wval = ps.wval;
  auto& red = ps.red;
  auto& piv_s = ps.piv_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 80) (&prow[0][0])[tid] = 0.0;  // pure-rotation steps read it with g = 0
  PP_T(t0);
  bool used = tid < n ? (J.rowstep[tid] >= 0) : true;
  double r[32];
  double* M = J.M;
  // out-of-place first pair: columns not yet written in M are read from Src
  const double* Mi = (J.Src && k0 < 2 * NB) ? J.Src : M;
  // full panels move through a per-warp 32 x 33 shared tile: the warp reads / writes its 32
  // rows' 256-byte segments coalesced (one row per instruction) instead of one strided
  // 256-byte segment per lane
  double* T = ptile + warp * 32 * 33;
  const bool tiled = nb == 32 && (n & 31) == 0;
  if (tiled) {
    if (warp * 32 < n) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) r[rr] = Mi[(size_t)(warp * 32 + rr) * n + k0 + lane];  // all in flight
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) T[rr * 33 + lane] = r[rr];
      __syncwarp();
      if (s1_a1kind < 0) {  // (with a stage-1 update the rows stay in T for the DMMA below)
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = T[lane * 33 + c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = 0.0;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      if (tid < n && c + 1 < nb && (n & 1) == 0) {
        const double2 v = *reinterpret_cast<const double2*>(&Mi[(size_t)tid * n + k0 + c]);
        r[c] = v.x;
        r[c + 1] = v.y;
      } else {
        r[c] = (tid < n && c < nb) ? Mi[(size_t)tid * n + k0 + c] : 0.0;
        r[c + 1] = (tid < n && c + 1 < nb) ? Mi[(size_t)tid * n + k0 + c + 1] : 0.0;
      }
    }
  }
  __syncthreads();
  PP_T(t1);
  PP_ADD(0, t1 - t0);
  if (s1_a1kind >= 0) {
    auto& w1s = ps.w1s;
    const int p1 = k0 - NB;
    for (int idx = tid; idx < 32 * 32; idx += NT) {
      const int c1 = idx >> 5, c = idx & 31;
      w1s[c1][c] = Mi[(size_t)J.piv[p1 + c1] * n + k0 + c];
    }
    __syncthreads();
    if (tiled) {  // on the tensor cores: per warp C(32 x 32) = z1 T + A1 W1 (8 k-steps of DMMA)
      if (warp * 32 < n) {
        const int g = lane >> 2, t4 = lane & 3;
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int rs = J.rowstep[warp * 32 + mi * 8 + g];
          const bool z1 = !(rs >= p1 && rs < k0);  // P1 pivot rows restart from zero
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[mi][ni][e] = z1 ? T[(mi * 8 + g) * 33 + ni * 8 + 2 * t4 + e] : 0.0;
        }
        const double* a1 = wkind(J, s1_a1kind) + (size_t)(warp * 32) * NB;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          double a[4], b[4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) a[mi] = a1[(size_t)(mi * 8 + g) * NB + k + t4];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) b[ni] = w1s[k + t4][ni * 8 + g];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
        }
        __syncwarp();
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) T[(mi * 8 + g) * 33 + ni * 8 + 2 * t4 + e] = acc[mi][ni][e];
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = T[lane * 33 + c];
      }
    } else if (tid < n) {
      const int rs = J.rowstep[tid];
      if (rs >= p1 && rs < k0) {  // P1 pivot row: z1 = 0
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = 0.0;
      }
      const double* a1 = wkind(J, s1_a1kind) + (size_t)tid * NB;
#pragma unroll 1
      for (int c1 = 0; c1 < 32; c1 += 4) {
        const double2 x01 = *reinterpret_cast<const double2*>(a1 + c1);
        const double2 x23 = *reinterpret_cast<const double2*>(a1 + c1 + 2);
        const double av[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const double2 w = *reinterpret_cast<const double2*>(&w1s[c1 + u][c]);
            r[c] = fma(av[u], w.x, r[c]);
            r[c + 1] = fma(av[u], w.y, r[c + 1]);
          }
      }
    }
  }
  double rowscale = 1.0, mypiv = 1.0;
  int my_step = -1;  // pivots kept on chip in the loop, published at the end (no live global pointers)
  __syncthreads();
  PP_T(t2);
  PP_ADD(1, t2 - t1);
#pragma unroll 1
  for (int kk = 0; kk < 32; ++kk) {
    const int par = kk & 1;
    const double* pr = prow[par];
    const double r0 = r[0];
    double g = 0.0, last = r0;  // kk >= nb: pure rotation
    if (kk < nb) {
      const bool cand = (tid < n) && !used && r0 != 0.0;
      const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~0x3ffu) | (unsigned)(1023 - tid)) : 0u;
      const unsigned wk = __reduce_max_sync(0xffffffffu, key);
      const double wv = __shfl_sync(0xffffffffu, r0, (1023 - (int)(wk & 0x3ffu)) & 31);
      if (lane == 0) {
        wkey32[par][warp] = wk;
        wval[par][warp] = wv;
      }
#ifdef LGM_PANEL_1BAR
      if (wk != 0u && lane == ((1023 - (int)(wk & 0x3ffu)) & 31)) {  // this warp's candidate row
        double* cw = ps.cand[par][warp];
#pragma unroll
        for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(cw + c) = make_double2(r[c], r[c + 1]);
      }
#endif
      __syncthreads();
      const unsigned bk = __reduce_max_sync(0xffffffffu, lane < NW ? wkey32[par][lane] : 0u);
      if (bk == 0u) {  // exact zero pivot (matcore.py:124-125)
        if (tid == 0) *J.status = 1;
        return false;
      }
      const int p = 1023 - (int)(bk & 0x3ffu);
      const double rp = lgm_rcp(wval[par][p >> 5]);
      const bool own = (tid == p);
#ifdef LGM_PANEL_1BAR
      pr = ps.cand[par][p >> 5];
      if (own) {
        used = true;
        mypiv = r0;
        rowscale = rp;
        my_step = k0 + kk;
        piv_s[kk] = tid;
      }
#else
      if (own) {
        used = true;
        mypiv = r0;
        rowscale = rp;
        double* pw = prow[par];
#pragma unroll
        for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r[c], r[c + 1]);
        my_step = k0 + kk;
        piv_s[kk] = tid;
      }
      __syncthreads();
#endif
      g = own ? 0.0 : r0 * rp;
      last = own ? 1.0 : -g;
    }
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
      if (c > 0) r[c - 1] = fma(-g, p2.x, r[c]);
      r[c] = fma(-g, p2.y, r[c + 1]);
    }
    r[31] = last;
  }
#ifdef LGM_PANEL_1BAR
  __syncthreads();  // the last steps' piv_s entries (no second barrier per step)
#endif
  const bool piv_here = my_step >= 0;
  if (piv_here) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] *= rowscale;
    J.rowstep[tid] = my_step;
  }
  if (tid < nb) J.piv[k0 + tid] = piv_s[tid];
  PP_T(t3);
  PP_ADD(2, t3 - t2);
  if (tiled) {
    if (warp * 32 < n) {
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 32; ++c) T[lane * 33 + c] = r[c];
      __syncwarp();
      double* A1 = a1_kind >= 0 ? wkind(J, a1_kind) : nullptr;  // rank-64 pair: P1's multipliers
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const double v = T[rr * 33 + lane];
        M[(size_t)(warp * 32 + rr) * n + k0 + lane] = v;
        if (A1) A1[(size_t)(warp * 32 + rr) * NB + lane] = v;
      }
    }
  } else if (tid < n) {
    if (nb == 32 && (n & 1) == 0) {
#pragma unroll
      for (int c = 0; c < 32; c += 2)
        *reinterpret_cast<double2*>(&M[(size_t)tid * n + k0 + c]) = make_double2(r[c], r[c + 1]);
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nb) M[(size_t)tid * n + k0 + c] = r[c];
    }
    if (a1_kind >= 0) {  // rank-64 pair: P1's multipliers also go to A1 (gj_copy_a1_kernel's layout)
      double* A1 = wkind(J, a1_kind) + (size_t)tid * NB;
#pragma unroll
      for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(A1 + c) = make_double2(r[c], r[c + 1]);
    }
  }
  // log|det| of this panel's pivots, CTA sum in warp order, one update per panel
  double lg = piv_here ? log(fabs(mypiv)) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
  if (lane == 0) red[warp] = lg;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += red[w];
    *J.logdet += t;
  }
  PP_T(t4);
  PP_ADD(3, t4 - t3);
  PP_ADD(4, 1);
  return true;
}

template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) gj_panel_cta_kernel(const InvJob* jobs, int n, int k0, int nb, int a1_kind,
                                                                   int s1_a1kind) {
  __shared__ __align__(16) PanelSmem ps;
  extern __shared__ __align__(16) double ptile[];
  const InvJob J = jobs[blockIdx.x];
  if (*J.status) return;  // uniform per CTA
  panel_body<NT>(J, n, k0, nb, a1_kind, s1_a1kind, ps, ptile);
}

// Both panels of a rank-64 pair in one launch (one CTA per job): P1 [k0, k0+NB) writing its
// multiplier copy A1 (kind a1_kind), then P2 [k0+NB, k0+2NB) with P1's stage-1 update fused
// (the same CTA wrote everything P2 reads: a block-scope fence orders it).  One wave tail and
// one launch per pair instead of two.
template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) gj_panel_pair_kernel(const InvJob* jobs, int n, int k0, int a1_kind) {
  __shared__ __align__(16) PanelSmem ps;
  extern __shared__ __align__(16) double ptile[];
  const InvJob J = jobs[blockIdx.x];
  if (*J.status) return;
  if (!panel_body<NT>(J, n, k0, NB, a1_kind, -1, ps, ptile)) return;
  __threadfence_block();
  __syncthreads();
  panel_body<NT>(J, n, k0 + NB, NB, -1, a1_kind, ps, ptile);
}

// Two rows per thread (256 < n <= 512, n % 32 == 0, full 32-column panels): the pivot loop of
// panel_body is bound by the shared-memory return path, not by latency -- every thread reads
// the whole 256-byte pivot row each step (512 threads x 256 B = 128 KB = 1024 cycles at 128
// B/clk/SM, the measured ~1.1k cycles per step), four times the FP64 pipe's 256 cycles.  Here
// thread `tid` of 256 owns rows tid and tid + 256, so one set of pivot-row loads feeds two
// rows' FMAs (64 KB per step).  Pivot rule, FMA chains, stage-1 DMMA products and the order
// of the log|det| sum are those of panel_body<512>: results are bit-identical.
struct Panel2Smem {
  double prow[2][40];
  unsigned wkey32[2][8];
  double wval[2][8];
  double red[16];
  int piv_s[32];
  double w1s[32][34];
};
__device__ __forceinline__ bool panel2_body(const InvJob& J, int n, int k0, int a1_kind, int s1_a1kind, Panel2Smem& ps,
                                            double* ptile) {
  constexpr int NT2 = 256, NW = 8;
  auto& prow = ps.prow;
  auto& wkey32 = ps.wkey32;
  auto& wval = ps.wval;
  auto& red = ps.red;
  auto& piv_s = ps.piv_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  PP_T(t0);
  const int row0 = tid, row1 = tid + NT2;
  const int base0 = warp * 32, base1 = NT2 + warp * 32;  // the warp's 32 rows in slot 0 / slot 1
  const bool v1 = base1 < n;                            // warp-uniform (n % 32 == 0); slot 0 is always valid
  bool used0 = J.rowstep[row0] >= 0;
  bool used1 = v1 ? (J.rowstep[row1] >= 0) : true;
  double r0[32], r1[32];
  double* M = J.M;
  const double* Mi = (J.Src && k0 < 2 * NB) ? J.Src : M;
  double* T = ptile + warp * 32 * 33;
  // both slots' global loads in flight first (r0 / r1 as transposed temporaries)
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) r0[rr] = Mi[(size_t)(base0 + rr) * n + k0 + lane];
  if (v1) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) r1[rr] = Mi[(size_t)(base1 + rr) * n + k0 + lane];
  }
  if (s1_a1kind >= 0) {
    auto& w1s = ps.w1s;
    const int p1 = k0 - NB;
    for (int idx = tid; idx < 32 * 32; idx += NT2) {
      const int c1 = idx >> 5, c = idx & 31;
      w1s[c1][c] = Mi[(size_t)J.piv[p1 + c1] * n + k0 + c];
    }
    __syncthreads();
  }
  // per slot: transpose through the warp's tile (with P1's stage-1 update on DMMA for P2)
  auto stage = [&](double (&r)[32], int base) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) T[rr * 33 + lane] = r[rr];
    __syncwarp();
    if (s1_a1kind >= 0) {
      auto& w1s = ps.w1s;
      const int p1 = k0 - NB;
      const int g = lane >> 2, t4 = lane & 3;
      double acc[4][4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int rs = J.rowstep[base + mi * 8 + g];
        const bool z1 = !(rs >= p1 && rs < k0);  // P1 pivot rows restart from zero
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[mi][ni][e] = z1 ? T[(mi * 8 + g) * 33 + ni * 8 + 2 * t4 + e] : 0.0;
      }
      const double* a1 = wkind(J, s1_a1kind) + (size_t)base * NB;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = a1[(size_t)(mi * 8 + g) * NB + k + t4];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = w1s[k + t4][ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
      __syncwarp();
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) T[(mi * 8 + g) * 33 + ni * 8 + 2 * t4 + e] = acc[mi][ni][e];
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = T[lane * 33 + c];
    __syncwarp();
  };
  stage(r0, base0);
  if (v1) {
    stage(r1, base1);
  } else {
#pragma unroll
    for (int c = 0; c < 32; ++c) r1[c] = 0.0;
  }
  double rowscale0 = 1.0, rowscale1 = 1.0, mypiv0 = 1.0, mypiv1 = 1.0;
  int my_step0 = -1, my_step1 = -1;
  __syncthreads();
  PP_T(t2);
  PP_ADD(0, t2 - t0);
#pragma unroll 1
  for (int kk = 0; kk < 32; ++kk) {
    PP_T(ta);
    const int par = kk & 1;
    const double* pr = prow[par];
    const double a0 = r0[0], a1 = r1[0];
    const bool cand0 = !used0 && a0 != 0.0;
    const bool cand1 = !used1 && a1 != 0.0;
    const unsigned key0 =
        cand0 ? ((((unsigned)__double2hiint(a0) & 0x7fffffffu) & ~0x3ffu) | (unsigned)(1023 - row0)) : 0u;
    const unsigned key1 =
        cand1 ? ((((unsigned)__double2hiint(a1) & 0x7fffffffu) & ~0x3ffu) | (unsigned)(1023 - row1)) : 0u;
    const unsigned wk = __reduce_max_sync(0xffffffffu, key0 > key1 ? key0 : key1);
    const int wrow = 1023 - (int)(wk & 0x3ffu);  // the warp's winning row (warp-uniform)
    const double wv = __shfl_sync(0xffffffffu, wrow >= NT2 ? a1 : a0, wrow & 31);
    if (lane == 0) {
      wkey32[par][warp] = wk;
      wval[par][warp] = wv;
    }
    __syncthreads();
    PP_T(tb);
    PP_ADD(6, tb - ta);
    const unsigned bk = __reduce_max_sync(0xffffffffu, lane < NW ? wkey32[par][lane] : 0u);
    if (bk == 0u) {  // exact zero pivot (matcore.py:124-125)
      if (tid == 0) *J.status = 1;
      return false;
    }
    const int p = 1023 - (int)(bk & 0x3ffu);
    // the owner publishes its raw row first: the reciprocal's slow-path call is a scheduling
    // barrier, and in source order after it the stores would wait for the whole Newton chain
    // (measured: reciprocal after the barrier 7.41 ms per 512-inversion step, before the
    // publish 7.31 ms)
    const bool own0 = (row0 == p), own1 = (row1 == p);
    if (own0) {
      used0 = true;
      mypiv0 = a0;
      double* pw = prow[par];
#pragma unroll
      for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r0[c], r0[c + 1]);
      my_step0 = k0 + kk;
      piv_s[kk] = p;
    }
    if (own1) {
      used1 = true;
      mypiv1 = a1;
      double* pw = prow[par];
#pragma unroll
      for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r1[c], r1[c + 1]);
      my_step1 = k0 + kk;
      piv_s[kk] = p;
    }
    const double rp = lgm_rcp(wval[par][(p & (NT2 - 1)) >> 5]);  // under the owner's stores
    if (own0) rowscale0 = rp;
    if (own1) rowscale1 = rp;
    __syncthreads();
    PP_T(tc);
    PP_ADD(7, tc - tb);
    const double g0 = own0 ? 0.0 : a0 * rp, g1 = own1 ? 0.0 : a1 * rp;
    const double last0 = own0 ? 1.0 : -g0, last1 = own1 ? 1.0 : -g1;
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
      if (c > 0) {
        r0[c - 1] = fma(-g0, p2.x, r0[c]);
        r1[c - 1] = fma(-g1, p2.x, r1[c]);
      }
      r0[c] = fma(-g0, p2.y, r0[c + 1]);
      r1[c] = fma(-g1, p2.y, r1[c + 1]);
    }
    r0[31] = last0;
    r1[31] = last1;
#ifdef LGM_PANEL_PROF
    if (tid == 0) {  // the step's FMAs: wait for the last result before reading the clock
      const long long td = clock64() + (long long)(__double_as_longlong(r0[30]) & 0);
      atomicAdd(&g_panel_cyc[8], (unsigned long long)(td - tc));
    }
#endif
  }
  PP_T(t3);
  PP_ADD(2, t3 - t2);
  const bool ph0 = my_step0 >= 0, ph1 = my_step1 >= 0;
  if (ph0) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r0[c] *= rowscale0;
    J.rowstep[row0] = my_step0;
  }
  if (ph1) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r1[c] *= rowscale1;
    J.rowstep[row1] = my_step1;
  }
  if (tid < 32) J.piv[k0 + tid] = piv_s[tid];
  double* A1 = a1_kind >= 0 ? wkind(J, a1_kind) : nullptr;  // rank-64 pair: P1's multipliers
  auto unstage = [&](const double (&r)[32], int base) {
#pragma unroll
    for (int c = 0; c < 32; ++c) T[lane * 33 + c] = r[c];
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const double v = T[rr * 33 + lane];
      M[(size_t)(base + rr) * n + k0 + lane] = v;
      if (A1) A1[(size_t)(base + rr) * NB + lane] = v;
    }
    __syncwarp();
  };
  unstage(r0, base0);
  if (v1) unstage(r1, base1);
  // log|det| of this panel's pivots: per 32-row group a butterfly sum, groups added in row
  // order (panel_body<512>'s warp order), one update per panel
  double lg0 = ph0 ? log(fabs(mypiv0)) : 0.0, lg1 = ph1 ? log(fabs(mypiv1)) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lg0 += __shfl_xor_sync(0xffffffffu, lg0, o);
    lg1 += __shfl_xor_sync(0xffffffffu, lg1, o);
  }
  if (lane == 0) {
    red[warp] = lg0;
    red[NW + warp] = lg1;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 2 * NW; ++w) t += red[w];
    *J.logdet += t;
  }
  PP_T(t4);
  PP_ADD(3, t4 - t3);
  PP_ADD(4, 1);
  return true;
}

__global__ void __launch_bounds__(256, 1) gj_panel_pair2_kernel(const InvJob* jobs, int n, int k0, int a1_kind) {
  __shared__ __align__(16) Panel2Smem ps;
  extern __shared__ __align__(16) double ptile[];
  const InvJob J = jobs[blockIdx.x];
  if (*J.status) return;
  if (threadIdx.x < 80) (&ps.prow[0][0])[threadIdx.x] = 0.0;
  if (!panel2_body(J, n, k0, a1_kind, -1, ps, ptile)) return;
  __threadfence_block();
  __syncthreads();
  panel2_body(J, n, k0 + NB, -1, a1_kind, ps, ptile);
}

__global__ void __launch_bounds__(512) gj_panel_kernel(const InvJob* jobs, int n, int k0, int nb, int in_smem) {
  extern __shared__ __align__(16) double psm[];
  __shared__ uint64_t skey[16];
  __shared__ int sidx[16];
  __shared__ double prow[NB];
  __shared__ int s_stop;
  const InvJob J = jobs[blockIdx.x];
  if (*J.status) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* S;
  int lds;
  if (in_smem) {
    S = psm;
    lds = NB + 1;
    for (int idx = tid; idx < n * nb; idx += nt) {
      int i = idx / nb, c = idx - i * nb;
      S[i * lds + c] = J.M[(size_t)i * n + k0 + c];
    }
  } else {
    S = J.M + k0;
    lds = n;
  }
  if (tid == 0) s_stop = 0;
  __syncthreads();
  for (int kk = 0; kk < nb; ++kk) {
    // pivot search among unused rows
    uint64_t key = 0ull;
    int idx = 0x7fffffff;
    for (int i = tid; i < n; i += nt) {
      if (J.rowstep[i] < 0) {
        uint64_t kq = dkey(fabs(S[(size_t)i * lds + kk]));
        if (kq > key) { key = kq; idx = i; }
      }
    }
    uint64_t kmax;
    int p;
    block_argmax(key, idx, skey, sidx, kmax, p);
    if (kmax <= 1ull) {  // exact zero pivot (matcore.py:124-125)
      if (tid == 0) *J.status = 1;
      return;
    }
    const double pv = S[(size_t)p * lds + kk];
    const double inv = 1.0 / pv;
    if (tid < nb) prow[tid] = S[(size_t)p * lds + tid];
    __syncthreads();
    if (tid == 0) {
      J.rowstep[p] = k0 + kk;
      J.piv[k0 + kk] = p;
      *J.logdet += log(fabs(pv));
    }
    for (int idx2 = tid; idx2 < n * nb; idx2 += nt) {
      int i = idx2 / nb, c = idx2 - i * nb;
      double* e = &S[(size_t)i * lds + c];
      if (i == p) {
        *e = (c == kk) ? inv : prow[c] * inv;
      } else {
        const double g = S[(size_t)i * lds + kk] * inv;
        if (c != kk) *e = fma(-g, prow[c], *e);
      }
    }
    __syncthreads();
    // the pivot column last (its old values were the multipliers above)
    for (int i = tid; i < n; i += nt)
      if (i != p) S[(size_t)i * lds + kk] = -S[(size_t)i * lds + kk] * inv;
    __syncthreads();
  }
  if (in_smem) {
    for (int idx = tid; idx < n * nb; idx += nt) {
      int i = idx / nb, c = idx - i * nb;
      J.M[(size_t)i * n + k0 + c] = S[i * lds + c];
    }
  }
  (void)s_stop;
}

// Snapshot the pivot rows of panel k0 (their values outside the panel are the B operand of
// the trailing update and get overwritten by it).
__global__ void gj_snapshot_kernel(const InvJob* jobs, int n, int k0, int nb, int kind, int jlo, int jhi) {
  const InvJob J = jobs[blockIdx.y];
  if (*J.status) return;
  double* W = wkind(J, kind);
  const int w = jhi - jlo;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nb * w; idx += gridDim.x * blockDim.x) {
    int c = idx / w, j = jlo + (idx - c * w);
    W[(size_t)c * n + j] = J.M[(size_t)J.piv[k0 + c] * n + j];
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Trailing update for every column j outside the panel:
//   M[i][j] <- (i pivot of this panel ? 0 : M[i][j]) + sum_c M[i][k0+c] * W[c][j].
// grid: (ceil(n/64) col tiles, ceil(n/64) row tiles, jobs); 128 threads; DMMA core.
// Columns written: [col_lo, col_hi) minus the panel minus [ex_lo, ex_hi); tile x covers
// [col_base + x*TN, +TN).  W parity `wpar` selects the snapshot buffer.
__global__ void __launch_bounds__(128) gj_update_kernel(const InvJob* jobs, int n, int k0, int nb, int col_base,
                                                        int col_lo, int col_hi, int ex_lo, int ex_hi, int wpar) {
  __shared__ __align__(16) double As[TM * LDA_S];
  __shared__ __align__(16) double Bs[TK * LDB_S];
  const InvJob J = jobs[blockIdx.z];
  if (*J.status) return;
  const int col0 = col_base + blockIdx.x * TN, row0 = blockIdx.y * TM;
  // skip tiles with no writable column
  if (col0 >= col_hi || col0 + TN <= col_lo) return;
  if (col0 >= k0 && col0 + TN <= k0 + nb) return;
  if (col0 >= ex_lo && col0 + TN <= ex_hi) return;
  const double* Wp = wkind(J, wpar);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  const bool vec = (n & 1) == 0;
  // C fragments first (their latency overlaps the A / W staging below); pivot rows of this
  // panel start from zero, panel columns are left alone
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    const int rs = (i < n) ? J.rowstep[i] : -1;
    const bool live = i < n && !(rs >= k0 && rs < k0 + nb);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;
      if (vec && live && j + 1 < n) {
        const double2 v = *reinterpret_cast<const double2*>(&J.M[(size_t)i * n + j]);
        acc[mi][ni][0] = v.x;
        acc[mi][ni][1] = v.y;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[mi][ni][e] = (live && j + e < n) ? J.M[(size_t)i * n + j + e] : 0.0;
      }
    }
  }
  // A (panel multipliers) and W (pivot-row snapshot) tiles: cp.async straight into shared
  // memory (no staging registers while the C fragments are held), scalar fallback at the
  // edges / odd n
  for (int idx = tid; idx < TM * (TK / 2); idx += 128) {
    const int r = idx / (TK / 2), c = (idx - r * (TK / 2)) * 2;
    const int i = row0 + r;
    if (i < n && vec && c + 1 < nb) {
      cp_async16(&As[r * LDA_S + c], &J.M[(size_t)i * n + k0 + c]);
    } else {
      As[r * LDA_S + c] = (i < n && c < nb) ? J.M[(size_t)i * n + k0 + c] : 0.0;
      As[r * LDA_S + c + 1] = (i < n && c + 1 < nb) ? J.M[(size_t)i * n + k0 + c + 1] : 0.0;
    }
  }
  for (int idx = tid; idx < TK * (TN / 2); idx += 128) {
    const int c = idx / (TN / 2), jj = (idx - c * (TN / 2)) * 2;
    const int j = col0 + jj;
    if (c < nb && vec && j + 1 < n) {
      cp_async16(&Bs[c * LDB_S + jj], &Wp[(size_t)c * n + j]);
    } else {
      Bs[c * LDB_S + jj] = (c < nb && j < n) ? Wp[(size_t)c * n + j] : 0.0;
      Bs[c * LDB_S + jj + 1] = (c < nb && j + 1 < n) ? Wp[(size_t)c * n + j + 1] : 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  tile_mma(As, Bs, acc);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;
      const bool in0 = j >= col_lo && j < col_hi && !(j >= k0 && j < k0 + nb) && !(j >= ex_lo && j < ex_hi);
      const bool in1 = j + 1 >= col_lo && j + 1 < col_hi && !(j + 1 >= k0 && j + 1 < k0 + nb) &&
                       !(j + 1 >= ex_lo && j + 1 < ex_hi);
      if (vec && in0 && in1) {
        *reinterpret_cast<double2*>(&J.M[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (in0) J.M[(size_t)i * n + j] = acc[mi][ni][0];
        if (in1) J.M[(size_t)i * n + j + 1] = acc[mi][ni][1];
      }
    }
  }
}

// ---- rank-64 delayed update (G2, n % 64 == 0) ---------------------------------------------
// Two consecutive 32-column panels P1 = [k0, k0+32), P2 = [k0+32, k0+64) are applied to the
// rest of the matrix in ONE pass (half the HBM traffic of two rank-32 passes).  With z1/z2 = 0
// on the pivot rows of P1/P2, A1 = P1's multipliers (copied before the pass overwrites P1),
// W1 = P1's pivot rows before any update, A2 = P2's multipliers and W2 = P2's pivot rows
// after P1's update, the two Gauss-Jordan stages compose to
//   j in P1:          M[i][j] <- z2 M[i][j] + sum_c A2[i][c] W2[c][j]           (M holds A1)
//   j outside P1, P2: M[i][j] <- z1 z2 M[i][j] + sum_c z2 A1[i][c] W1[c][j] + sum_c A2[i][c] W2[c][j]
// where W2[c][j] = M[p2_c][j] + sum_c' A1[p2_c][c'] W1[c'][j] (P2's pivot rows are not P1
// pivots) and W2[c][j in P1] = A1[p2_c][j - k0].  P2's columns are left alone.

__global__ void gj_copy_a1_kernel(const InvJob* jobs, int n, int k0, int ka1) {
  const InvJob J = jobs[blockIdx.y];
  if (*J.status) return;
  double* A1 = wkind(J, ka1);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * NB; idx += gridDim.x * blockDim.x) {
    const int i = idx / NB, c = idx - i * NB;
    A1[idx] = J.M[(size_t)i * n + k0 + c];
  }
}

// W2 (into J.W2) from the unmodified pivot rows of P2, A1 and W1 (= J.W); then W1's P1 columns
// are zeroed for the combined pass.  One thread per column j, the 32 x 32 block A1[p2_c][:] in
// shared memory.
// snap = 1: W1 is not snapshotted beforehand -- its rows are read from M (P1's pivot rows,
// not yet touched by the pass) and written here (one kernel instead of snapshot + W2).
__global__ void __launch_bounds__(128) gj_w2_kernel(const InvJob* jobs, int n, int k0, int q, int snap) {
  __shared__ __align__(16) double a1s[NB][NB + 2];
  __shared__ int p2s[NB];
  const InvJob J = jobs[blockIdx.y];
  if (*J.status) return;
  double* W1 = wkind(J, 3 * q);
  double* W2 = wkind(J, 3 * q + 1);
  const double* A1 = wkind(J, 3 * q + 2);
  const int tid = threadIdx.x;
  if (tid < NB) p2s[tid] = J.piv[k0 + NB + tid];
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    const int c = idx / NB, cc = idx - c * NB;
    a1s[c][cc] = A1[(size_t)p2s[c] * NB + cc];
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + tid;
  if (j >= n) return;
  if (j >= k0 && j < k0 + NB) {
#pragma unroll 4
    for (int c = 0; c < NB; ++c) W2[(size_t)c * n + j] = a1s[c][j - k0];
#pragma unroll 4
    for (int c = 0; c < NB; ++c) W1[(size_t)c * n + j] = 0.0;
    return;
  }
  if (j >= k0 + NB && j < k0 + 2 * NB) {
#pragma unroll 4
    for (int c = 0; c < NB; ++c) W2[(size_t)c * n + j] = 0.0;
    return;
  }
  double w[NB];
  if (snap) {
#pragma unroll
    for (int cc = 0; cc < NB; ++cc) {
      w[cc] = J.M[(size_t)J.piv[k0 + cc] * n + j];
      W1[(size_t)cc * n + j] = w[cc];
    }
  } else {
#pragma unroll
    for (int cc = 0; cc < NB; ++cc) w[cc] = W1[(size_t)cc * n + j];
  }
#pragma unroll 2
  for (int c = 0; c < NB; ++c) {
    double acc = J.M[(size_t)p2s[c] * n + j];
#pragma unroll
    for (int cc = 0; cc < NB; cc += 2) {  // 16-byte broadcast loads, same FMA order
      const double2 a = *reinterpret_cast<const double2*>(&a1s[c][cc]);
      acc = fma(a.x, w[cc], acc);
      acc = fma(a.y, w[cc + 1], acc);
    }
    W2[(size_t)c * n + j] = acc;
  }
}

// W1 snapshot + W2 on DMMA (the cta-panel path, n % 64 == 0): CTA = 64 columns of one job,
// W2[c][j] = M[p2_c][j] + sum_cc A1[p2_c][cc] W1[cc][j] as a 32 x 64 x 32 product (warp w:
// all 32 rows c, columns 16w..16w+15), W1[cc][j] = M[p1_cc][j] read once (not snapshotted
// beforehand).  P1 columns: W1 = 0, W2 = A1[p2_c][j - k0]; P2 columns: W2 = 0.
// wt = 1: W1 / W2 stored transposed (n x NB per kind) for gj_update2_tma_kernel's TMA tiles
__global__ void __launch_bounds__(128) gj_w2_mma_kernel(const InvJob* jobs, int n, int k0, int q, int wt) {
  __shared__ __align__(16) double a1s[NB][NB + 4];
  __shared__ __align__(16) double w1s[NB][64 + 4];
  __shared__ int p1s[NB], p2s[NB];
  const InvJob J = jobs[blockIdx.y];
  if (*J.status) return;
  double* W1 = wkind(J, 3 * q);
  double* W2 = wkind(J, 3 * q + 1);
  const double* A1 = wkind(J, 3 * q + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j0 = blockIdx.x * 64;
  if (tid < NB) p1s[tid] = J.piv[k0 + tid];
  else if (tid < 2 * NB) p2s[tid - NB] = J.piv[k0 + tid];
  __syncthreads();
  // the accumulators' P2 rows need only p2s: issued with the A1 / W1 staging loads (one global
  // round trip less per CTA)
  const int g8 = lane >> 2, t4 = lane & 3, wc = warp * 16;
  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int jc = j0 + wc + ni * 8 + 2 * t4;
      const double* Ms = (J.Src && k0 == 0 && jc >= 2 * NB) ? J.Src : J.M;
      const double2 v = *reinterpret_cast<const double2*>(&Ms[(size_t)p2s[mi * 8 + g8] * n + jc]);
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
    }
  for (int idx = tid; idx < NB * NB; idx += 128) {
    const int c = idx >> 5, cc = idx & 31;
    a1s[c][cc] = A1[(size_t)p2s[c] * NB + cc];
  }
  for (int idx = tid; idx < NB * 32; idx += 128) {  // W1 rows, 16-byte chunks
    const int cc = idx >> 5, jj = (idx & 31) * 2;
    const int j = j0 + jj;
    const double* Ms = (J.Src && k0 == 0 && j >= 2 * NB) ? J.Src : J.M;  // out-of-place first pair
    double2 v = *reinterpret_cast<const double2*>(&Ms[(size_t)p1s[cc] * n + j]);
    if (j >= k0 && j < k0 + NB) v = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(&w1s[cc][jj]) = v;
    if (!wt) *reinterpret_cast<double2*>(&W1[(size_t)cc * n + j]) = v;
  }
  __syncthreads();
  if (wt) {  // transposed: the 64 x NB block W1T[j0 .. j0+64) is contiguous
    for (int idx = tid; idx < 64 * NB; idx += 128) {
      const int jj = idx >> 5, cc = idx & 31;
      W1[(size_t)(j0 + jj) * NB + cc] = w1s[cc][jj];
    }
  }
#pragma unroll
  for (int k = 0; k < NB; k += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = a1s[mi * 8 + g8][k + t4];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = w1s[k + t4][wc + ni * 8 + g8];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
  if (wt) __syncthreads();  // every warp is done reading w1s before it stages W2
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int c = mi * 8 + g8;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int j = j0 + wc + ni * 8 + 2 * t4;  // j, j + 1 on the same side of 32-aligned bounds
      double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      if (j >= k0 && j < k0 + NB) v = make_double2(a1s[c][j - k0], a1s[c][j + 1 - k0]);
      else if (j >= k0 + NB && j < k0 + 2 * NB) v = make_double2(0.0, 0.0);
      if (wt) {  // staged (w1s is free now) for a contiguous transposed store
        w1s[c][j - j0] = v.x;
        w1s[c][j + 1 - j0] = v.y;
      } else {
        *reinterpret_cast<double2*>(&W2[(size_t)c * n + j]) = v;
      }
    }
  }
  if (wt) {
    __syncthreads();
    for (int idx = tid; idx < 64 * NB; idx += 128) {
      const int jj = idx >> 5, cc = idx & 31;
      W2[(size_t)(j0 + jj) * NB + cc] = w1s[cc][jj];
    }
  }
}

template <int RT>  // RT = output tile rows (64: 4 warps, 128: 8 warps); 64 columns
constexpr size_t up2_smem() { return (size_t)(2 * RT * LDA_S + 2 * TK * LDB_S + TK) * 8; }

// Combined pass (see above).  Tile x covers [col_base + x*TN, +TN); columns written:
// [col_lo, col_hi) minus P2 minus [ex_lo, ex_hi).
template <int RT>
__global__ void __launch_bounds__(2 * RT) gj_update2_kernel(const InvJob* jobs, int n, int k0, int col_base,
                                                         int col_lo, int col_hi, int ex_lo, int ex_hi, int q) {
  extern __shared__ __align__(16) double u2sm[];
  double* As1 = u2sm;
  double* As2 = As1 + RT * LDA_S;
  double* Bs1 = As2 + RT * LDA_S;
  double* Bs2 = Bs1 + TK * LDB_S;
  double* Zs = Bs2 + TK * LDB_S;  // a zero row: the A1 operand of P2's pivot rows (z2 = 0)
  // consecutive pairs traverse the jobs in opposite orders (L2 reuse across passes)
  const InvJob J = jobs[(q & 1) ? gridDim.z - 1 - blockIdx.z : blockIdx.z];
  if (*J.status) return;  // (checked first: moving this load after the tile loads measured 7% slower)
  const double* W1 = wkind(J, 3 * q);
  const double* W2 = wkind(J, 3 * q + 1);
  const double* A1 = wkind(J, 3 * q + 2);
  const int col0 = col_base + blockIdx.x * TN, row0 = blockIdx.y * RT;
  const int p1lo = k0, p2lo = k0 + NB, p2hi = k0 + 2 * NB;
  if (col0 >= col_hi || col0 + TN <= col_lo) return;
  if (col0 >= p2lo && col0 + TN <= p2hi) return;
  if (col0 >= ex_lo && col0 + TN <= ex_hi) return;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  // stage A1 / A2 / W1 / W2 (cp.async; n % 64 == 0 so every 16-byte chunk is in range)
  for (int idx = tid; idx < RT * (TK / 2); idx += 2 * RT) {
    const int r = idx / (TK / 2), c = (idx - r * (TK / 2)) * 2;
    cp_async16(&As1[r * LDA_S + c], &A1[(size_t)(row0 + r) * NB + c]);
    cp_async16(&As2[r * LDA_S + c], &J.M[(size_t)(row0 + r) * n + p2lo + c]);
  }
  for (int idx = tid; idx < TK * (TN / 2); idx += 2 * RT) {
    const int c = idx / (TN / 2), jj = (idx - c * (TN / 2)) * 2;
    cp_async16(&Bs1[c * LDB_S + jj], &W1[(size_t)c * n + col0 + jj]);
    cp_async16(&Bs2[c * LDB_S + jj], &W2[(size_t)c * n + col0 + jj]);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  if (tid < TK) Zs[tid] = 0.0;
  // C fragments while the tiles land; z1 / z2 masks per row
  double acc[4][4][2];
  bool z2r[4];
  // out-of-place first pair: columns beyond the pair are still only in Src
  const double* Cs = (J.Src && k0 == 0 && c0 >= 2 * NB) ? J.Src : J.M;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    const int rs = J.rowstep[i];
    const bool z1 = !(rs >= p1lo && rs < p2lo), z2 = !(rs >= p2lo && rs < p2hi);
    z2r[mi] = z2;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;  // j, j+1 on the same side of every 32-aligned boundary
      const bool keep = (j >= p1lo && j < p2lo) ? z2 : (z1 && z2);
      const double2 v = *reinterpret_cast<const double2*>(&Cs[(size_t)i * n + j]);
      acc[mi][ni][0] = keep ? v.x : 0.0;
      acc[mi][ni][1] = keep ? v.y : 0.0;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int lr0 = (warp >> 1) * 32, lc0 = (warp & 1) * 32;
  int aoff[4];  // A1 rows, or the zero row where z2 = 0 (offsets into the shared array: LDS,
                // no select in the k loop)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) aoff[mi] = z2r[mi] ? (lr0 + mi * 8 + g) * LDA_S : (int)(Zs - u2sm);
#pragma unroll
  for (int k = 0; k < TK; k += 4) {  // + z2 A1 W1
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = u2sm[aoff[mi] + k + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs1[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
#pragma unroll
  for (int k = 0; k < TK; k += 4) {  // + A2 W2
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = As2[(lr0 + mi * 8 + g) * LDA_S + k + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs2[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;
      const bool in = j >= col_lo && j < col_hi && !(j >= p2lo && j < p2hi) && !(j >= ex_lo && j < ex_hi);
      if (in) *reinterpret_cast<double2*>(&J.M[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
  }
}

// The same combined pass with one K-half slot in shared memory (A1 / W1, products, then A2 / W2
// into the same slot, products): 36 KB per CTA instead of 72, so 4 CTAs (16 warps) per SM hide
// the loads of each other's halves -- the one-shot kernel above holds 3.  Per output element the
// accumulation order is unchanged (C, + z2 A1 W1 in k order, + A2 W2 in k order): bit-identical.
#ifndef UP2S_MINB
#define UP2S_MINB 4
#endif
template <int RT>
constexpr size_t up2s_smem() { return (size_t)(RT * LDA_S + TK * LDB_S + TK) * 8; }
template <int RT>
__global__ void __launch_bounds__(2 * RT, UP2S_MINB) gj_update2s_kernel(const InvJob* jobs, int n, int k0, int col_base,
                                                         int col_lo, int col_hi, int ex_lo, int ex_hi, int q) {
  extern __shared__ __align__(16) double u2sm[];
  double* As = u2sm;               // one K-half slot: A1 / W1, then A2 / W2
  double* Bs = As + RT * LDA_S;
  double* Zs = Bs + TK * LDB_S;  // a zero row: the A1 operand of P2's pivot rows (z2 = 0)
  // consecutive pairs traverse the jobs in opposite orders (L2 reuse across passes)
  const InvJob J = jobs[(q & 1) ? gridDim.z - 1 - blockIdx.z : blockIdx.z];
  if (*J.status) return;  // (checked first: moving this load after the tile loads measured 7% slower)
  const double* W1 = wkind(J, 3 * q);
  const double* W2 = wkind(J, 3 * q + 1);
  const double* A1 = wkind(J, 3 * q + 2);
  const int col0 = col_base + blockIdx.x * TN, row0 = blockIdx.y * RT;
  const int p1lo = k0, p2lo = k0 + NB, p2hi = k0 + 2 * NB;
  if (col0 >= col_hi || col0 + TN <= col_lo) return;
  if (col0 >= p2lo && col0 + TN <= p2hi) return;
  if (col0 >= ex_lo && col0 + TN <= ex_hi) return;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  // stage A1 / A2 / W1 / W2 (cp.async; n % 64 == 0 so every 16-byte chunk is in range)
  auto stage = [&](const double* Ag, size_t lda, size_t aoff0, const double* Wg) {
    for (int idx = tid; idx < RT * (TK / 2); idx += 2 * RT) {
      const int r = idx / (TK / 2), c = (idx - r * (TK / 2)) * 2;
      cp_async16(&As[r * LDA_S + c], &Ag[(size_t)(row0 + r) * lda + aoff0 + c]);
    }
    for (int idx = tid; idx < TK * (TN / 2); idx += 2 * RT) {
      const int c = idx / (TN / 2), jj = (idx - c * (TN / 2)) * 2;
      cp_async16(&Bs[c * LDB_S + jj], &Wg[(size_t)c * n + col0 + jj]);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  stage(A1, NB, 0, W1);  // K-half 1: A1 / W1 (A2 / W2 reuse the slot after the first products)
  if (tid < TK) Zs[tid] = 0.0;
  // C fragments while the tiles land; z1 / z2 masks per row
  double acc[4][4][2];
  bool z2r[4];
  // out-of-place first pair: columns beyond the pair are still only in Src
  const double* Cs = (J.Src && k0 == 0 && c0 >= 2 * NB) ? J.Src : J.M;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    const int rs = J.rowstep[i];
    const bool z1 = !(rs >= p1lo && rs < p2lo), z2 = !(rs >= p2lo && rs < p2hi);
    z2r[mi] = z2;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;  // j, j+1 on the same side of every 32-aligned boundary
      const bool keep = (j >= p1lo && j < p2lo) ? z2 : (z1 && z2);
      const double2 v = *reinterpret_cast<const double2*>(&Cs[(size_t)i * n + j]);
      acc[mi][ni][0] = keep ? v.x : 0.0;
      acc[mi][ni][1] = keep ? v.y : 0.0;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int lr0 = (warp >> 1) * 32, lc0 = (warp & 1) * 32;
  int aoff[4];  // A1 rows, or the zero row where z2 = 0 (offsets into the shared array: LDS,
                // no select in the k loop)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) aoff[mi] = z2r[mi] ? (lr0 + mi * 8 + g) * LDA_S : (int)(Zs - u2sm);
#pragma unroll
  for (int k = 0; k < TK; k += 4) {  // + z2 A1 W1
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = u2sm[aoff[mi] + k + t];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
  __syncthreads();  // every warp is done with A1 / W1
  stage(J.M, (size_t)n, (size_t)p2lo, W2);  // K-half 2: P2's multipliers / W2
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < TK; k += 4) {  // + A2 W2
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
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;
      const bool in = j >= col_lo && j < col_hi && !(j >= p2lo && j < p2hi) && !(j >= ex_lo && j < ex_hi);
      if (in) *reinterpret_cast<double2*>(&J.M[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// G3: the whole inversion of one job per CTA with warp specialisation (256 < n <= 512,
// n % 64 == 0).  16 panel warps (P: row `tid` of the current 32-column panel in registers,
// G1's pivot rule and shift-in-FMA frame) factor pair p+1 while 8 update warps (U) apply pair
// p's delayed rank-64 update (G2's combined pass: C <- z C + z2 A1 W1 + A2 W2) to the rest of
// the matrix, 64 x 64 tiles through a 2-stage cp.async pipeline -- so the latency-bound pivot
// steps run under DMMA work instead of owning an SM, and there is no per-panel launch.  Per pair:
//   U: wait PANEL_DONE(p) -> form W1 / W2 of pair p -> the tiles of pair p+1's columns ->
//      arrive NARROW_DONE(p) -> every other tile;
//   P: wait NARROW_DONE(p) -> factor pair p+1 (P2's stage-1 by P1 as FMA chains, as G2's
//      untiled panel path) -> arrive PANEL_DONE(p+1).
// Persistent: gridDim.x CTAs walk the job table.  Named barriers: 1 = P (512), 2 = U (256),
// 3 = PANEL_DONE (P arrive, U sync), 4 = NARROW_DONE (U arrive, P sync).
constexpr int G3_THREADS = 768, G3_P = 512, G3_U = 256;
#ifdef LGM_G3_PROF  // clock64 phase sums (thread 0 of each role): see lgm_debug_g3_cycles
__device__ unsigned long long g_g3_cyc[8];  // P: wait narrow, panels; U: wait panel, W, narrow tiles, rest tiles
#define G3T(v) long long v = clock64()
#define G3ADD(i, a, b) if ((threadIdx.x & (G3_P - 1)) == 0 || threadIdx.x == G3_P) atomicAdd(&g_g3_cyc[i], (unsigned long long)((b) - (a)))
#define G3SET(a, b) a = b
#else
#define G3SET(a, b)
#define G3T(v)
#define G3ADD(i, a, b)
#endif
constexpr int G3_LDC = 72;  // C tile row stride (conflict-free 16-byte fragment reads)
constexpr size_t G3_STAGE = (size_t)2 * 64 * LDA_S + 2 * TK * LDB_S + 64 * G3_LDC;  // doubles
struct G3Smem {
  double prow[2][40];
  unsigned wkey32[2][16];
  double wval[2][16];
  double red[16];
  double w1s[32][34];   // P2's stage-1 operand (pivot rows of P1 in P2's columns)
  double zs[32];        // zero row (A1 operand of P2's pivot rows in the update)
  int piv_s[64];        // the current pair's pivots
  int rstep[512];       // rowstep of every row
  int abort_;           // exact zero pivot: the job stops
};
constexpr size_t g3_smem() { return 2 * G3_STAGE * 8; }

__device__ __forceinline__ void g3_bar(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void g3_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

// P warps: one 32-column panel [kp, kp+32) of the job (row = tid < n).  s1_kind >= 0: the
// previous panel's stage-1 update first (multipliers in kind s1_kind); a1_kind >= 0: the
// output also goes to that multiplier copy.  Returns false on an exact zero pivot.
__device__ __forceinline__ bool g3_panel(const InvJob& J, int n, int kp, int pofs, int a1_kind, int s1_kind, G3Smem& gs,
                                         bool& used, double& mypiv, int& my_step) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Mi = (J.Src && kp < 2 * NB) ? J.Src : J.M;  // out-of-place first pair
  const bool row_ok = tid < n;
  double r[32];
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    double2 v = make_double2(0.0, 0.0);
    if (row_ok) v = *reinterpret_cast<const double2*>(&Mi[(size_t)tid * n + kp + c]);
    r[c] = v.x;
    r[c + 1] = v.y;
  }
  if (s1_kind >= 0) {  // r <- z1 r + A1[row] W1[:, this panel] (FMA chains in c1 order)
    const int p1 = kp - NB;
    for (int idx = tid; idx < 32 * 32; idx += G3_P) {
      const int c1 = idx >> 5, c = idx & 31;
      gs.w1s[c1][c] = Mi[(size_t)J.piv[p1 + c1] * n + kp + c];
    }
    g3_bar(1, G3_P);
    if (row_ok) {
      const int rs = gs.rstep[tid];
      if (rs >= p1 && rs < kp) {
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = 0.0;
      }
      const double* a1 = wkind(J, s1_kind) + (size_t)tid * NB;
#pragma unroll 1
      for (int c1 = 0; c1 < 32; c1 += 4) {
        const double2 x01 = *reinterpret_cast<const double2*>(a1 + c1);
        const double2 x23 = *reinterpret_cast<const double2*>(a1 + c1 + 2);
        const double av[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const double2 w = *reinterpret_cast<const double2*>(&gs.w1s[c1 + u][c]);
            r[c] = fma(av[u], w.x, r[c]);
            r[c + 1] = fma(av[u], w.y, r[c + 1]);
          }
      }
    }
  }
  double rowscale = 1.0;
#pragma unroll 1
  for (int kk = 0; kk < 32; ++kk) {
    const int par = kk & 1;
    const double r0 = r[0];
    const bool cand = row_ok && !used && r0 != 0.0;
    const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~0x3ffu) | (unsigned)(1023 - tid)) : 0u;
    const unsigned wk = __reduce_max_sync(0xffffffffu, key);
    const double wv = __shfl_sync(0xffffffffu, r0, (1023 - (int)(wk & 0x3ffu)) & 31);
    if (lane == 0) {
      gs.wkey32[par][warp] = wk;
      gs.wval[par][warp] = wv;
    }
    g3_bar(1, G3_P);
    const unsigned bk = __reduce_max_sync(0xffffffffu, lane < 16 ? gs.wkey32[par][lane] : 0u);
    if (bk == 0u) return false;  // exact zero pivot (matcore.py:124-125), uniform
    const int p = 1023 - (int)(bk & 0x3ffu);
    const double rp = lgm_rcp(gs.wval[par][p >> 5]);
    const bool own = (tid == p);
    if (own) {
      used = true;
      mypiv = r0;
      rowscale = rp;
      double* pw = gs.prow[par];
#pragma unroll
      for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(pw + c) = make_double2(r[c], r[c + 1]);
      my_step = kp + kk;
      gs.piv_s[pofs + kk] = tid;
      gs.rstep[tid] = kp + kk;
    }
    g3_bar(1, G3_P);
    const double g = own ? 0.0 : r0 * rp;
    const double last = own ? 1.0 : -g;
    const double* pr = gs.prow[par];
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      const double2 p2 = *reinterpret_cast<const double2*>(pr + c);
      if (c > 0) r[c - 1] = fma(-g, p2.x, r[c]);
      r[c] = fma(-g, p2.y, r[c + 1]);
    }
    r[31] = last;
  }
  if (my_step >= kp && my_step < kp + 32) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] *= rowscale;
  }
  if (row_ok) {
#pragma unroll
    for (int c = 0; c < 32; c += 2)
      *reinterpret_cast<double2*>(&J.M[(size_t)tid * n + kp + c]) = make_double2(r[c], r[c + 1]);
    if (a1_kind >= 0) {
      double* A1 = wkind(J, a1_kind) + (size_t)tid * NB;
#pragma unroll
      for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(A1 + c) = make_double2(r[c], r[c + 1]);
    }
  }
  if (tid < 32) J.piv[kp + tid] = gs.piv_s[pofs + tid];
  g3_bar(1, G3_P);  // P1's outputs (global, piv_s) before P2's stage-1 reads them
  return true;
}

__global__ void __launch_bounds__(G3_THREADS, 1) gj_inv_ws_kernel(const InvJob* jobs, int nj, int n) {
  extern __shared__ __align__(16) double g3sm[];
  __shared__ __align__(16) G3Smem gs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool is_p = tid < G3_P;
  const int npairs = n / (2 * NB);
  for (int jb = blockIdx.x; jb < nj; jb += gridDim.x) {
    const InvJob J = jobs[jb];
    if (!J.M) continue;  // unused slot of the device-built job table (uniform)
    for (int i = tid; i < 512; i += G3_THREADS) gs.rstep[i] = i < n ? -1 : 0x3fffffff;
    if (tid < 32) gs.zs[tid] = 0.0;
    if (tid == 0) gs.abort_ = 0;
    __syncthreads();
    if (is_p) {
      // ================================================================ P warps
      bool used = false;
      double mypiv = 1.0;
      int my_step = -1;
      bool ok = true;
      for (int pp = 0; pp < npairs && ok; ++pp) {
        const int kp = pp * 2 * NB, q = pp & 1;
        G3T(ta);
        if (pp > 0) g3_bar(4, G3_THREADS);  // NARROW_DONE(pp - 1): this pair's columns are updated
        G3T(tb);
        ok = g3_panel(J, n, kp, 0, 3 * q + 2, -1, gs, used, mypiv, my_step) &&
             g3_panel(J, n, kp + NB, NB, -1, 3 * q + 2, gs, used, mypiv, my_step);
        G3T(tc);
        G3ADD(0, ta, tb);
        G3ADD(1, tb, tc);
        if (!ok && tid == 0) gs.abort_ = 1;
        __threadfence_block();
        g3_arrive(3, G3_THREADS);  // PANEL_DONE(pp)
      }
      // publish rowstep, log|det| (warp-order CTA sum over the P warps)
      if (tid < n) J.rowstep[tid] = my_step;
      double lg = my_step >= 0 ? log(fabs(mypiv)) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
      if (lane == 0) gs.red[warp] = lg;
      g3_bar(1, G3_P);
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 16; ++w) t += gs.red[w];
        *J.logdet = t;
        *J.status = ok ? 0 : 1;
      }
    } else {
      // ================================================================ U warps
      const int ut = tid - G3_P, uw = ut >> 5;  // 0..255, warp 0..7
      const int g = lane >> 2, t = lane & 3;
      for (int pp = 0; pp < npairs; ++pp) {
        G3T(ua);
        g3_bar(3, G3_THREADS);  // PANEL_DONE(pp)
        G3T(ub);
        G3ADD(2, ua, ub);
        if (*(volatile int*)&gs.abort_) break;
        const int k0 = pp * 2 * NB, q = pp & 1;
        const int p1lo = k0, p2lo = k0 + NB, p2hi = k0 + 2 * NB;
        const bool next = pp + 1 < npairs;
        const int kn = k0 + 2 * NB;
        double* W1 = wkind(J, 3 * q);
        double* W2 = wkind(J, 3 * q + 1);
        const double* A1 = wkind(J, 3 * q + 2);
        // ---- W1 / W2 of this pair (gj_w2_mma_kernel's arithmetic), two 64-column blocks at a time
        {
          double* a1s = g3sm;                  // [32][LDA_S]
          double* w1s = a1s + 32 * LDA_S;      // [2][32][LDB_S]
          for (int idx = ut; idx < NB * NB; idx += G3_U) {
            const int c = idx >> 5, cc = idx & 31;
            a1s[c * LDA_S + cc] = A1[(size_t)gs.piv_s[NB + c] * NB + cc];
          }
          const int half = uw >> 2, wc = (uw & 3) * 16;
          for (int jb2 = 0; jb2 < n; jb2 += 128) {
            for (int idx = ut; idx < 2 * NB * 32; idx += G3_U) {  // W1 rows of both blocks, 16-byte chunks
              const int h = idx / (NB * 32), rem = idx - h * (NB * 32);
              const int cc = rem >> 5, jj = (rem & 31) * 2, j = jb2 + h * 64 + jj;
              if (j >= n) continue;  // n % 128 == 64: the last pair of blocks has one
              const double* Ms = (J.Src && k0 == 0 && j >= 2 * NB) ? J.Src : J.M;
              double2 v = *reinterpret_cast<const double2*>(&Ms[(size_t)gs.piv_s[cc] * n + j]);
              if (j >= k0 && j < k0 + NB) v = make_double2(0.0, 0.0);
              *reinterpret_cast<double2*>(&w1s[(h * 32 + cc) * LDB_S + jj]) = v;
              *reinterpret_cast<double2*>(&W1[(size_t)cc * n + j]) = v;
            }
            g3_bar(2, G3_U);
            const int j0 = jb2 + half * 64;
            const double* wsh = w1s + half * 32 * LDB_S;
            if (j0 < n) {  // (warp-uniform)
            double acc[4][2][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) {
                const int jc = j0 + wc + ni * 8 + 2 * t;
                const double* Ms = (J.Src && k0 == 0 && jc >= 2 * NB) ? J.Src : J.M;
                const double2 v = *reinterpret_cast<const double2*>(&Ms[(size_t)gs.piv_s[NB + mi * 8 + g] * n + jc]);
                acc[mi][ni][0] = v.x;
                acc[mi][ni][1] = v.y;
              }
#pragma unroll
            for (int k = 0; k < NB; k += 4) {
              double a[4], b[2];
#pragma unroll
              for (int mi = 0; mi < 4; ++mi) a[mi] = a1s[(mi * 8 + g) * LDA_S + k + t];
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) b[ni] = wsh[(k + t) * LDB_S + wc + ni * 8 + g];
#pragma unroll
              for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              const int c = mi * 8 + g;
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) {
                const int j = j0 + wc + ni * 8 + 2 * t;
                double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
                if (j >= k0 && j < k0 + NB) v = make_double2(a1s[c * LDA_S + j - k0], a1s[c * LDA_S + j + 1 - k0]);
                else if (j >= k0 + NB && j < k0 + 2 * NB) v = make_double2(0.0, 0.0);
                *reinterpret_cast<double2*>(&W2[(size_t)c * n + j]) = v;
              }
            }
            }
            g3_bar(2, G3_U);  // w1s reused by the next blocks
          }
          __threadfence_block();
          g3_bar(2, G3_U);  // W1 / W2 (global) complete before the tiles read them
        }
        G3T(uc);
        G3ADD(3, ub, uc);
        // ---- the combined rank-64 update, 64 x 64 tiles: next pair's columns first
        const int nrb = n / 64, nct = n / 64;
        const int cx_next = next ? kn / 64 : -1;
        const int ntile = next ? nrb * nct : nrb * nct;  // every (rb, cx); next pair's column first
        auto tile_of = [&](int i, int& rb, int& cx) {
          if (next) {
            if (i < nrb) { rb = i; cx = cx_next; return; }
            const int r = i - nrb;  // the remaining (nct - 1) columns
            rb = r / (nct - 1);
            const int c = r - rb * (nct - 1);
            cx = c < cx_next ? c : c + 1;
          } else {
            rb = i / nct;
            cx = i - rb * nct;
          }
        };
        const int nt = next ? nrb * nct : nrb * nct;
        (void)ntile;
        auto issue = [&](int i, int stg) {
          int rb, cx;
          tile_of(i, rb, cx);
          double* S = g3sm + stg * G3_STAGE;
          double* As1 = S;
          double* As2 = As1 + 64 * LDA_S;
          double* Bs1 = As2 + 64 * LDA_S;
          double* Bs2 = Bs1 + TK * LDB_S;
          double* Cs = Bs2 + TK * LDB_S;
          const int row0 = rb * 64, col0 = cx * 64;
          for (int idx = ut; idx < 64 * (TK / 2); idx += G3_U) {
            const int r = idx / (TK / 2), c = (idx - r * (TK / 2)) * 2;
            cp_async16(&As1[r * LDA_S + c], &A1[(size_t)(row0 + r) * NB + c]);
            cp_async16(&As2[r * LDA_S + c], &J.M[(size_t)(row0 + r) * n + p2lo + c]);
          }
          for (int idx = ut; idx < TK * 32; idx += G3_U) {
            const int c = idx >> 5, jj = (idx & 31) * 2;
            cp_async16(&Bs1[c * LDB_S + jj], &W1[(size_t)c * n + col0 + jj]);
            cp_async16(&Bs2[c * LDB_S + jj], &W2[(size_t)c * n + col0 + jj]);
          }
          for (int idx = ut; idx < 64 * 32; idx += G3_U) {
            const int r = idx >> 5, jj = (idx & 31) * 2, j = col0 + jj;
            const double* Csrc = (J.Src && k0 == 0 && j >= 2 * NB) ? J.Src : J.M;
            cp_async16(&Cs[r * G3_LDC + jj], &Csrc[(size_t)(row0 + r) * n + j]);
          }
          asm volatile("cp.async.commit_group;\n" ::);
        };
        const int lr0 = (uw >> 2) * 32, lc0 = (uw & 3) * 16;
        issue(0, 0);
        for (int i = 0; i < nt; ++i) {
          if (i + 1 < nt) {
            issue(i + 1, (i + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
          } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
          }
          g3_bar(2, G3_U);
          int rb, cx;
          tile_of(i, rb, cx);
          const double* S = g3sm + (i & 1) * G3_STAGE;
          const double* As1 = S;
          const double* As2 = As1 + 64 * LDA_S;
          const double* Bs1 = As2 + 64 * LDA_S;
          const double* Bs2 = Bs1 + TK * LDB_S;
          const double* Cs = Bs2 + TK * LDB_S;
          const int r0 = rb * 64 + lr0, c0 = cx * 64 + lc0;
          double acc[4][2][2];
          const double* aptr[4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int rs = gs.rstep[r0 + mi * 8 + g];
            const bool z1 = !(rs >= p1lo && rs < p2lo), z2 = !(rs >= p2lo && rs < p2hi);
            aptr[mi] = z2 ? As1 + (lr0 + mi * 8 + g) * LDA_S : gs.zs;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              const int j = c0 + ni * 8 + 2 * t;
              const bool keep = (j >= p1lo && j < p2lo) ? z2 : (z1 && z2);
              const double2 v = *reinterpret_cast<const double2*>(&Cs[(lr0 + mi * 8 + g) * G3_LDC + lc0 + ni * 8 + 2 * t]);
              acc[mi][ni][0] = keep ? v.x : 0.0;
              acc[mi][ni][1] = keep ? v.y : 0.0;
            }
          }
#pragma unroll
          for (int k = 0; k < TK; k += 4) {  // + z2 A1 W1
            double a[4], b[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = aptr[mi][k + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) b[ni] = Bs1[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
          }
#pragma unroll
          for (int k = 0; k < TK; k += 4) {  // + A2 W2
            double a[4], b[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As2[(lr0 + mi * 8 + g) * LDA_S + k + t];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) b[ni] = Bs2[(k + t) * LDB_S + lc0 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int ii = r0 + mi * 8 + g;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              const int j = c0 + ni * 8 + 2 * t;
              if (!(j >= p2lo && j < p2hi))
                *reinterpret_cast<double2*>(&J.M[(size_t)ii * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            }
          }
          if (next && i == nrb - 1) {  // the next pair's columns are complete
            __threadfence_block();
            g3_bar(2, G3_U);
            g3_arrive(4, G3_THREADS);  // NARROW_DONE(pp)
            G3T(ud);
            G3ADD(4, uc, ud);
            G3SET(uc, ud);
          } else {
            g3_bar(2, G3_U);  // stage (i & 1) is refilled at i + 2
          }
        }
        G3T(ue);
        G3ADD(5, uc, ue);
      }
    }
    __syncthreads();  // job end: every role done (the next job reuses the shared state)
  }
}

// ------------------------------------------------------------------------------------------
// TMA-pipelined combined rank-64 pass (n <= 512 with single-CTA panels, n % 64 == 0).
// One CTA owns a 64-row block of one job and walks its column tiles: the A operands (A1 and
// P2's multipliers) are staged once, the W1 / W2 column tiles stream through a 2-stage ring
// filled by TMA (cp.async.bulk.tensor, 128-byte swizzle, mbarrier complete_tx) from a producer
// warp, and each tile's C fragments are prefetched into registers one tile ahead.  W1 / W2 are
// stored transposed (n x NB per kind, written by gj_w2_mma_kernel) so the swizzled B-fragment
// reads are bank-conflict free.
#ifndef UT_STAGES_DEF
#define UT_STAGES_DEF 3
#endif
#ifndef UT_NWR
#define UT_NWR 2
#endif
constexpr int UT_STAGES = UT_STAGES_DEF;
constexpr int UT_ROWS = 64 * UT_NWR;                  // rows per CTA (4 compute warps per 64)
constexpr int UT_THREADS = 128 * UT_NWR;              // thread 0 also issues the TMA loads
constexpr int UT_BOX = 64 * 16 * 8;                 // one TMA box: 64 W rows (columns of M) x 16 k
constexpr int UT_STAGE_BYTES = 4 * UT_BOX;           // W1 (2 boxes) + W2 (2 boxes)
constexpr size_t ut_smem() { return 1024 + (size_t)UT_STAGES * UT_STAGE_BYTES + (size_t)(2 * UT_ROWS * LDA_S + 32) * 8 + 64; }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c_inner, int c_row, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c_inner), "r"(c_row), "r"(smem_u32(bar))
      : "memory");
}
// element (row r, k) of a 64 x 16 box stored with the 128-byte swizzle
__device__ __forceinline__ int swz(int r, int k) { return r * 16 + ((((k >> 1) ^ (r & 7)) << 1) | (k & 1)); }

#ifndef UT_MINB
#define UT_MINB 1
#endif
__global__ void __launch_bounds__(UT_THREADS, UT_MINB) gj_update2_tma_kernel(const InvJob* jobs, int n, int k0, int col_base,
                                                                 int col_lo, int col_hi, int ex_lo, int ex_hi, int q,
                                                                 const double* Wbase,
                                                                 const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ __align__(16) unsigned char utsm_raw[];
  // 1024-byte aligned ring (128-byte swizzle), then A1 / A2 tiles, the zero row, barriers
  unsigned char* base = (unsigned char*)(((uintptr_t)utsm_raw + 1023) & ~(uintptr_t)1023);
  double* ring = reinterpret_cast<double*>(base);
  double* As1 = ring + UT_STAGES * UT_STAGE_BYTES / 8;
  double* As2 = As1 + UT_ROWS * LDA_S;
  double* Zs = As2 + UT_ROWS * LDA_S;
  uint64_t* full = reinterpret_cast<uint64_t*>(Zs + 32);
  uint64_t* empty = full + UT_STAGES;
  const InvJob J = jobs[blockIdx.y];
  if (*J.status) return;  // uniform per CTA (unused table slots read the always-1 status)
  const int row0 = blockIdx.x * UT_ROWS;
  const int p1lo = k0, p2lo = k0 + NB, p2hi = k0 + 2 * NB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NCW = 4 * UT_NWR;  // compute warps
  // the column tiles this CTA writes, in order
  const int ntile_all = (col_hi - col_base + 63) / 64;
  auto tile_ok = [&](int t) {
    const int c0 = col_base + t * 64;
    if (c0 >= col_hi || c0 + 64 <= col_lo) return false;
    if (c0 >= p2lo && c0 + 64 <= p2hi) return false;
    if (c0 >= ex_lo && c0 + 64 <= ex_hi) return false;
    return true;
  };
  // W row index of (kind, column j): rows of the transposed W region, NB doubles each
  const long long w1row = (long long)(wkind(J, 3 * q) - Wbase) / NB;
  const long long w2row = (long long)(wkind(J, 3 * q + 1) - Wbase) / NB;
  if (tid == 0) {
    for (int s = 0; s < UT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // A1 rows and P2's multipliers (M columns [p2lo, p2hi)) of this row block, once
  {
    const double* A1 = wkind(J, 3 * q + 2);
    for (int idx = tid; idx < UT_ROWS * (NB / 2); idx += UT_THREADS) {
      const int r = idx / (NB / 2), c = (idx - r * (NB / 2)) * 2;
      if (row0 + r >= n) break;  // last row block of n % UT_ROWS != 0 (n % 64 == 0)
      cp_async16(&As1[r * LDA_S + c], &A1[(size_t)(row0 + r) * NB + c]);
      cp_async16(&As2[r * LDA_S + c], &J.M[(size_t)(row0 + r) * n + p2lo + c]);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (tid < 32) Zs[tid] = 0.0;
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  // consumers: warp w owns rows (w/2)*32.., columns (w%2)*32.. of each UT_ROWS x 64 tile
  const int g = lane >> 2, t4 = lane & 3;
  const int lr0 = (warp >> 1) * 32, lc0 = (warp & 1) * 32;
  const int r0 = row0 + lr0;
  const bool rows_ok = r0 < n;  // (a warp's 32 rows are all in range or all out: n % 64 == 0)
  bool z1r[4], z2r[4];
  int aoff[4];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int rs = rows_ok ? J.rowstep[r0 + mi * 8 + g] : -1;
    z1r[mi] = !(rs >= p1lo && rs < p2lo);
    z2r[mi] = !(rs >= p2lo && rs < p2hi);
    aoff[mi] = z2r[mi] ? (lr0 + mi * 8 + g) * LDA_S : (int)(Zs - As1);
  }
  auto load_c = [&](int c0, double (&cv)[4][4][2]) {
    if (!rows_ok) return;
    const double* Cs = (J.Src && k0 == 0 && c0 + lc0 >= 2 * NB) ? J.Src : J.M;  // out-of-place first pair
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const double2 v = *reinterpret_cast<const double2*>(&Cs[(size_t)(r0 + mi * 8 + g) * n + c0 + lc0 + ni * 8 + 2 * t4]);
        cv[mi][ni][0] = v.x;
        cv[mi][ni][1] = v.y;
      }
  };
  // TMA issue (thread 0): the ring runs UT_STAGES tiles ahead of the consumers
  int tiss = 0, sis = 0;
  unsigned phis = 0;
  auto issue_next = [&]() {
    while (tiss < ntile_all && !tile_ok(tiss)) ++tiss;
    if (tiss >= ntile_all) return;
    const int c0 = col_base + tiss * 64;
    mbar_wait(&empty[sis], phis ^ 1u);
    mbar_expect_tx(&full[sis], UT_STAGE_BYTES);
    double* st = ring + (size_t)sis * (UT_STAGE_BYTES / 8);
    tma_load_2d(st, &wmap, 0, (int)(w1row + c0), &full[sis]);
    tma_load_2d(st + UT_BOX / 8, &wmap, 16, (int)(w1row + c0), &full[sis]);
    tma_load_2d(st + 2 * UT_BOX / 8, &wmap, 0, (int)(w2row + c0), &full[sis]);
    tma_load_2d(st + 3 * UT_BOX / 8, &wmap, 16, (int)(w2row + c0), &full[sis]);
    ++tiss;
    if (++sis == UT_STAGES) { sis = 0; phis ^= 1u; }
  };
  if (tid == 0)
    for (int s0 = 0; s0 < UT_STAGES; ++s0) issue_next();
  int tcur = 0;
  while (tcur < ntile_all && !tile_ok(tcur)) ++tcur;
  if (tcur >= ntile_all) return;
  double acc[4][4][2] = {};
  load_c(col_base + tcur * 64, acc);
  int stage = 0;
  unsigned ph = 0;
  while (tcur < ntile_all) {
    int tnext = tcur + 1;
    while (tnext < ntile_all && !tile_ok(tnext)) ++tnext;
    const int c0 = col_base + tcur * 64;
    double cn[4][4][2] = {};
    if (tnext < ntile_all) load_c(col_base + tnext * 64, cn);  // in flight during this tile's MMAs
    // masks: P1 columns keep z2; other columns keep z1 && z2 (the applied panels' pivot rows)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int j = c0 + lc0 + ni * 8 + 2 * t4;
        const bool keep = (j >= p1lo && j < p2lo) ? z2r[mi] : (z1r[mi] && z2r[mi]);
        if (!keep) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
    mbar_wait(&full[stage], ph);
    const double* st = ring + (size_t)stage * (UT_STAGE_BYTES / 8);
#pragma unroll
    for (int k = 0; k < NB; k += 4) {  // + z2 A1 W1
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As1[aoff[mi] + k + t4];
      const double* bx = st + ((k >> 4) * UT_BOX / 8);
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = bx[swz(lc0 + ni * 8 + g, (k & 15) + t4)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
#pragma unroll
    for (int k = 0; k < NB; k += 4) {  // + A2 W2
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As2[(lr0 + mi * 8 + g) * LDA_S + k + t4];
      const double* bx = st + ((2 + (k >> 4)) * UT_BOX / 8);
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = bx[swz(lc0 + ni * 8 + g, (k & 15) + t4)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == UT_STAGES) { stage = 0; ph ^= 1u; }
    if (tid == 0) issue_next();  // refill the slot just released (waits for every warp)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = r0 + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int j = c0 + lc0 + ni * 8 + 2 * t4;
        const bool in = rows_ok && j >= col_lo && j < col_hi && !(j >= p2lo && j < p2hi) && !(j >= ex_lo && j < ex_hi);
        if (in) *reinterpret_cast<double2*>(&J.M[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    }
    if (tnext < ntile_all) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          acc[mi][ni][0] = cn[mi][ni][0];
          acc[mi][ni][1] = cn[mi][ni][1];
        }
    }
    tcur = tnext;
  }
}

// ------------------------------------------------------------------------------------------
// Elementwise / reduction kernels over a list of matrices (index list `ids`).
struct Slots {
  double* ws;       // base of the n x n slots
  int n;
  size_t st;        // slot stride in doubles: n^2 (+ a guard band under LGM_WS_GUARD=1)
  __device__ __host__ double* buf(int b, int k) const { return ws + ((size_t)b * NBUF + k) * st; }
};

// Device-built matrix lists: ids[0 .. *cnt) (ascending matrix indices), capacity = batch.
// The list kernels below stride over (entry, element) with a grid sized for the device, so a
// short or empty list costs one small launch whatever the capacity.
struct DList {
  const int* ids;
  const int* cnt;
};
constexpr int EW_BLOCKS = 148 * 8;  // grid of the element-wise list kernels

#define LIST_LOOP(L, nn)                                                                                    \
  const size_t per_ = (nn);                                                                                \
  const size_t tot_ = (size_t)(*(L).cnt) * per_;                                                           \
  for (size_t g_ = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g_ < tot_; g_ += (size_t)gridDim.x * blockDim.x) { \
    const int e_ = (int)(g_ / per_);                                                                       \
    const size_t idx = g_ - (size_t)e_ * per_;                                                             \
    const int b = (L).ids[e_];

__global__ void load_kernel(const double* const* Ap, const long long* ldp, Slots S, DList L, int* bad) {
  const int n = S.n;
  const double* A = *Ap;
  const long long ld = *ldp;
  LIST_LOOP(L, (size_t)n * n)
    int i = idx / n, j = idx - (size_t)i * n;
    double v = A[(size_t)b * n * ld + (size_t)i * ld + j];
    S.buf(b, G_B)[idx] = v;
    if (!isfinite(v)) bad[b] = 1;
  }
}

// dst = src - I (op 0), copy (op 1), identity (op 2), dst = src - 2*src2 + I (op 3, A_I2),
// dst = I - src (op 4)
__global__ void ew_kernel(Slots S, DList L, int op, int dk, int sk, int s2k) {
  const int n = S.n;
  LIST_LOOP(L, (size_t)n * n)
    double* D = S.buf(b, dk);
    const double* X = S.buf(b, sk);
    const double* X2 = S.buf(b, s2k);
    int i = idx / n, j = idx - (size_t)i * n;
    double v;
    switch (op) {
      case 0: v = X[idx]; if (i == j) v = v - 1.0; break;
      case 1: v = X[idx]; break;
      case 2: v = (i == j) ? 1.0 : 0.0; break;
      case 3: v = X[idx] - 2.0 * X2[idx]; if (i == j) v = v + 1.0; break;
      default: v = X[idx]; v = (i == j) ? 1.0 - v : -v; break;
    }
    D[idx] = v;
  }
}

// onenorm exactly as numpy (column sums accumulated over rows in order), max via atomicMax
// into out[b] (zeroed beforehand).
// Complex embeddings (P->cplx): the norm of Z, |z_ij| = hypot(E[i][j], E[i+m][j]) over the
// m x m complex entries (numpy's abs of complex128, then the same row-order column sums).
__global__ void onenorm_kernel(Slots S, DList L, int k, double* out, const LgmParams* P) {
  const int n = S.n;
  const bool cx = P && P->cplx;
  const int m = cx ? n / 2 : n;
  LIST_LOOP(L, (size_t)m)
    const double* M = S.buf(b, k);
    const int j = (int)idx;
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
      const double v = cx ? hypot(M[(size_t)i * n + j], M[(size_t)(i + m) * n + j]) : fabs(M[(size_t)i * n + j]);
      acc = (i == 0) ? v : acc + v;
    }
    atomic_max_nonneg(&out[b], acc);
  }
}

// numpy pairwise sum (n < 8: sequential; n <= 128: 8 accumulators; else split n/2 - (n/2)%8)
// of |p[i*stride]|.  Leaves (<= 128 terms) are summed by different threads, then combined
// in the recursion's order by thread 0.
__device__ int pw_leaves(int n, int off, int* loff, int* llen, int cnt) {
  if (n <= 128) { loff[cnt] = off; llen[cnt] = n; return cnt + 1; }
  int n2 = n / 2;
  n2 -= n2 % 8;
  cnt = pw_leaves(n2, off, loff, llen, cnt);
  return pw_leaves(n - n2, off + n2, loff, llen, cnt);
}
// The same recursion flattened once into a post-order program (1 = next leaf, 0 = add the
// top two: left + right), evaluated without recursion per balancing step.
__device__ int pw_tokens(int n, signed char* tok, int cnt) {
  if (n <= 128) { tok[cnt] = 1; return cnt + 1; }
  int n2 = n / 2;
  n2 -= n2 % 8;
  cnt = pw_tokens(n2, tok, cnt);
  cnt = pw_tokens(n - n2, tok, cnt);
  tok[cnt] = 0;
  return cnt + 1;
}
__device__ __forceinline__ double pw_eval(const signed char* tok, int ntok, const double* leaf) {
  double st[16];  // depth <= log2(number of leaves) + 1
  int sp = 0, pos = 0;
  for (int t = 0; t < ntok; ++t) {
    if (tok[t]) {
      st[sp++] = leaf[pos++];
    } else {
      const double b = st[--sp];
      st[sp - 1] = st[sp - 1] + b;
    }
  }
  return st[0];
}
__device__ double pw_block(const double* p, size_t stride, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += fabs(p[i * stride]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = fabs(p[q * stride]);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] += fabs(p[(i + q) * stride]);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += fabs(p[i * stride]);
  return res;
}

// Osborne radix-2 balancing (matcore.py:180-215), one CTA per matrix, bit-identical to numpy.
// number of pairwise-summation leaves of length n (same recursion as pw_leaves)
static int host_pw_leaves(int n) {
  if (n <= 128) return 1;
  int n2 = n / 2;
  n2 -= n2 % 8;
  return host_pw_leaves(n2) + host_pw_leaves(n - n2);
}
// launch shape of balance_kernel_g: 64 threads for n <= 256 (one leaf pair per row / column:
// more CTAs per SM), else 256 / 1024; dynamic smem = the (leaf, accumulator) partials
static int bal_threads(int n) { return n <= 256 ? 64 : (n >= 2048 ? 1024 : 256); }
static size_t bal_smem(int n) { return (size_t)2 * host_pw_leaves(n) * 8 * sizeof(double); }

// Complex embeddings (P->cplx): Osborne on Z (m x m, |z| = hypot of the two blocks' entries),
// each scaling applied to the embedding's rows / columns i and i + m.
__global__ void __launch_bounds__(1024) balance_kernel_g(Slots S, DList L, double* scale, int* sweeps_out,
                                                        int max_sweeps, double* margin, const int* enable,
                                                        const int* max_sweeps_p, const LgmParams* P) {
  if (blockIdx.x >= *L.cnt || (enable && !*enable)) return;
  if (max_sweeps_p) max_sweeps = *max_sweeps_p;
  const int b = L.ids[blockIdx.x];
  const int nfull = S.n;
  const bool cx = P && P->cplx;
  const int n = cx ? nfull / 2 : nfull;  // the matrix balanced (Z's order for an embedding)
  const size_t imoff = (size_t)n * nfull;  // offset of Im(z_ij) from Re(z_ij) in the embedding
  auto absv = [&](const double* p, size_t off) { return cx ? hypot(p[off], p[off + imoff]) : fabs(p[off]); };
  double* B = S.buf(b, G_B);
  double* sc = scale + (size_t)b * nfull;
  __shared__ int loff[128], llen[128];
  __shared__ double lsum[2][128];
  extern __shared__ double lacc_dyn[];  // [2][nleaf * 8] (sized by the host: bal_smem)
  __shared__ int s_nleaf, s_do, s_ntok;
  __shared__ double s_f, s_mm;
  __shared__ signed char tok[256];
  if (threadIdx.x == 0) {
    s_nleaf = pw_leaves(n, 0, loff, llen, 0);
    s_ntok = pw_tokens(n, tok, 0);
    s_mm = margin[b];
  }
  for (int i = threadIdx.x; i < nfull; i += blockDim.x) sc[i] = 1.0;
  __syncthreads();
  const int nleaf = s_nleaf;
  int sweeps = 0;
  for (int sw = 0; sw < max_sweeps; ++sw) {
    sweeps++;
    bool moved = false;
    for (int i = 0; i < n; ++i) {
      // leaf sums in numpy's order, split over (leaf, accumulator) so all loads are in
      // flight at once: accumulator a of a leaf sums elements a, a+8, ... (pairwise_sum's
      // 8-way unrolled block), then one thread per leaf combines them and adds the tail
      for (int t = threadIdx.x; t < 2 * nleaf * 8; t += blockDim.x) {
        const int which = t / (nleaf * 8), rem = t - which * nleaf * 8, q = rem >> 3, a = rem & 7;
        const int len = llen[q];
        if (len < 8) continue;
        const double* p = which == 0 ? B + (size_t)loff[q] * nfull + i : B + (size_t)i * nfull + loff[q];
        const size_t stride = which == 0 ? (size_t)nfull : 1;
        const int m8 = len - len % 8;
        double r;
        if (m8 == 128) {  // full leaf: all 16 loads in flight, then the in-order sum
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = absv(p, (a + 8 * u) * stride);
          r = v[0];
#pragma unroll
          for (int u = 1; u < 16; ++u) r += v[u];
        } else {
          r = absv(p, a * stride);
          for (int k = 8 + a; k < m8; k += 8) r += absv(p, k * stride);
        }
        lacc_dyn[which * nleaf * 8 + rem] = r;
      }
      __syncthreads();
      for (int l = threadIdx.x; l < 2 * nleaf; l += blockDim.x) {
        const int which = l / nleaf, q = l - which * nleaf;
        const int len = llen[q];
        const double* p = which == 0 ? B + (size_t)loff[q] * nfull + i : B + (size_t)i * nfull + loff[q];
        const size_t stride = which == 0 ? (size_t)nfull : 1;
        double res;
        if (len < 8) {
          res = 0.0;
          for (int k = 0; k < len; ++k) res += absv(p, k * stride);
        } else {
          const double* r = &lacc_dyn[which * nleaf * 8 + q * 8];
          res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
          for (int k = len - len % 8; k < len; ++k) res += absv(p, k * stride);
        }
        lsum[which][q] = res;
      }
      __syncthreads();
      // column (lane 0) and row (lane 1) sums combined in the recursion's order, in parallel
      double cr = 0.0, rr = 0.0;
      if (threadIdx.x < 2) {
        cr = pw_eval(tok, s_ntok, lsum[threadIdx.x]);
        rr = __shfl_sync(0x3u, cr, 1);
      }
      if (threadIdx.x == 0) {
        double dg = absv(B, (size_t)i * nfull + i);
        double c = cr - dg;
        double r = rr - dg;
        double mm = s_mm;
        int go = 0;
        double f = 1.0;
        if (!(c == 0.0 || r == 0.0)) {
          double tot = c + r;
          auto note = [&](double x, double thr) { double d = fabs(thr); mm = fmin(mm, d > 0 ? fabs(x - thr) / d : fabs(x - thr)); };
          while (true) { note(c, r / 2.0); if (!(c < r / 2.0)) break; c *= 2.0; r /= 2.0; f *= 2.0; }
          while (true) { note(c, r * 2.0); if (!(c >= r * 2.0)) break; c /= 2.0; r *= 2.0; f /= 2.0; }
          note(c + r, 0.95 * tot);
          go = (c + r < 0.95 * tot && 1e-300 < f && f < 1e300) ? 1 : 0;
        }
        s_mm = mm;
        s_do = go;
        s_f = f;
      }
      __syncthreads();
      if (s_do) {
        const double f = s_f, inv = 1.0 / f;
        for (int q = threadIdx.x; q < nfull; q += blockDim.x) {
          B[(size_t)q * nfull + i] *= f;
          if (cx) B[(size_t)q * nfull + i + n] *= f;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nfull; q += blockDim.x) {
          B[(size_t)i * nfull + q] *= inv;
          if (cx) B[(size_t)(i + n) * nfull + q] *= inv;
        }
        if (threadIdx.x == 0) {
          sc[i] *= f;
          if (cx) sc[i + n] = sc[i];
        }
        moved = true;
      }
      __syncthreads();
    }
    if (!moved) break;
  }
  if (threadIdx.x == 0) { sweeps_out[b] = sweeps; margin[b] = s_mm; }
}

__device__ unsigned long long g_exec_nodes;  // kernel nodes executed inside graphs (lgm_launch_count)

__device__ __forceinline__ void count_nodes(int nodes) {
  if (threadIdx.x == 0) atomicAdd(&g_exec_nodes, (unsigned long long)nodes);
}

// per-matrix Algorithm-1 state (oracle/driver.py _State + the running root / request)
static_assert(2 * 14 + 2 <= 32, "estimate cache covers powers up to m_K + 1");
struct MDev {
  int status, s, db_iters, nest, passes, products, k, plateau, sweeps;
  int finish, have_ai2, post_fail;
  int dbit, dbst, dbplat;           // running square root: iterations, status, plateau tests
  int dbpred;                       // this iteration is predicted to be the root's last (lazy X^-1)
  int dbskip;                       // X inversions skipped by the lazy order (whole call)
  int jcur, max_in;                 // select sweep
  int am, need1, need2, adone;      // alpha request (power m) and its progress
  unsigned cvalid;                  // estimate cache validity bits, by power
  double dbmm;                      // running root's margin
  double th, t1, Pm, t2, aout;      // alpha request threshold and terms
  double alpha_loop, mm, nA, nI2, cert, cert_max;
  double cache[32];  // estimates by power m (<= m_K + 1 = 29 with k = 9)
  __device__ void note(double x, double thr) {
    const double d = fabs(thr);
    mm = fmin(mm, d > 0 ? fabs(x - thr) / d : fabs(x - thr));
  }
  __device__ bool le(double x, double thr) { note(x, thr); return x <= thr; }
};

// ------------------------------------------------------------------------------------------
// Scaled DB update (sqrtm.py:57-67) fused with the column sums of |X'-X| and |X'|.
struct DbArgs {
  Slots S;
  DList L;
  const int* xpiv;   // [b][n] pivot rows of the X inversion (piv)
  const int* xstep;  // [b][n] rowstep of the X inversion
  const int* ypiv;
  const int* ystep;
  const double* xlog;  // [b]
  const double* ylog;
  const int* scaling;  // [b]
  int first;           // iteration 1: Y = I, Y^-1 = I
  double* change;      // [b] (max over columns, atomicMax; zeroed by host)
  double* size;
  const int* istat;    // [2][b] singular flags of this iteration's X / Y inversions
  int batch;
  MDev* ms;            // dbpred: X' goes to slot xn_slot, Y is left for the fix-up (lazy X^-1)
  int xn_slot;
  const LgmParams* P;  // P->cplx: change / size are the complex 1-norms of Z's m x m block
};

__global__ void __launch_bounds__(128) db_update_kernel(DbArgs a) {
  if (blockIdx.y >= *a.L.cnt) return;
  const int b = a.L.ids[blockIdx.y];
  const int n = a.S.n;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (a.istat[b] || (!a.first && a.istat[a.batch + b])) return;  // singular iterate: X, Y kept
  const bool cx = a.P && a.P->cplx;
  const int m = cx ? n / 2 : n;
  if (!a.first && a.ms[b].dbpred) {  // predicted last iteration: X' (no X^-1 needed) to a spare slot
    const double* X = a.S.buf(b, G_B);
    double* Xn = a.S.buf(b, a.xn_slot);
    const double* RY = a.S.buf(b, G_YI);
    const int* yp = a.ypiv + (size_t)b * n;
    const int qyc = a.ystep[(size_t)b * n + c];
    double mu = 1.0;
    if (a.scaling[b]) mu = fmin(fmax(exp(-(a.xlog[b] + a.ylog[b]) / (2.0 * n)), LGM_MU_MIN), LGM_MU_MAX);
    const double inv_mu = 1.0 / mu;
    double dsum = 0.0, ssum = 0.0;
    if (cx) {  // rows r and r + m together: the complex entry of row r (column c < m)
      for (int r = 0; r < m; ++r) {
        const size_t e = (size_t)r * n + c, e2 = (size_t)(r + m) * n + c;
        const double xo = X[e], xo2 = X[e2];
        const double xn = 0.5 * (mu * xo + RY[(size_t)yp[r] * n + qyc] * inv_mu);
        const double xn2 = 0.5 * (mu * xo2 + RY[(size_t)yp[r + m] * n + qyc] * inv_mu);
        Xn[e] = xn;
        Xn[e2] = xn2;
        if (c < m) {
          const double d = hypot(xn - xo, xn2 - xo2), sz = hypot(xn, xn2);
          dsum = (r == 0) ? d : dsum + d;
          ssum = (r == 0) ? sz : ssum + sz;
        }
      }
      if (c < m) {
        atomic_max_nonneg(&a.change[b], dsum);
        atomic_max_nonneg(&a.size[b], ssum);
      }
      return;
    }
    constexpr int U = 8;
    int r = 0;
    for (; r + U <= n; r += U) {
      double yi[U], xo[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        yi[u] = RY[(size_t)yp[r + u] * n + qyc];
        xo[u] = X[(size_t)(r + u) * n + c];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double xn = 0.5 * (mu * xo[u] + yi[u] * inv_mu);
        Xn[(size_t)(r + u) * n + c] = xn;
        dsum = (r + u == 0) ? fabs(xn - xo[u]) : dsum + fabs(xn - xo[u]);
        ssum = (r + u == 0) ? fabs(xn) : ssum + fabs(xn);
      }
    }
    for (; r < n; ++r) {
      const double xo = X[(size_t)r * n + c];
      const double xn = 0.5 * (mu * xo + RY[(size_t)yp[r] * n + qyc] * inv_mu);
      Xn[(size_t)r * n + c] = xn;
      dsum = (r == 0) ? fabs(xn - xo) : dsum + fabs(xn - xo);
      ssum = (r == 0) ? fabs(xn) : ssum + fabs(xn);
    }
    atomic_max_nonneg(&a.change[b], dsum);
    atomic_max_nonneg(&a.size[b], ssum);
    return;
  }
  double* X = a.S.buf(b, G_B);
  double* Y = a.S.buf(b, G_Y);
  const double* RX = a.S.buf(b, G_XI);
  const double* RY = a.S.buf(b, G_YI);
  const int* xp = a.xpiv + (size_t)b * n;
  const int* yp = a.ypiv + (size_t)b * n;
  const int qxc = a.xstep[(size_t)b * n + c];
  const int qyc = a.first ? 0 : a.ystep[(size_t)b * n + c];
  double mu = 1.0;
  if (a.scaling[b]) mu = fmin(fmax(exp(-(a.xlog[b] + a.ylog[b]) / (2.0 * n)), LGM_MU_MIN), LGM_MU_MAX);
  const double inv_mu = 1.0 / mu;
  double dsum = 0.0, ssum = 0.0;
  if (cx) {  // rows r and r + m together: the complex entry of row r (column c < m)
    for (int r = 0; r < m; ++r) {
      double xn2[2], xo2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = r + h * m;
        const size_t e = (size_t)rr * n + c;
        const double xi = RX[(size_t)xp[rr] * n + qxc];
        const double yi = a.first ? ((rr == c) ? 1.0 : 0.0) : RY[(size_t)yp[rr] * n + qyc];
        xo2[h] = X[e];
        xn2[h] = 0.5 * (mu * xo2[h] + yi * inv_mu);
        X[e] = xn2[h];
        Y[e] = 0.5 * (mu * Y[e] + xi * inv_mu);
      }
      if (c < m) {
        const double d = hypot(xn2[0] - xo2[0], xn2[1] - xo2[1]), sz = hypot(xn2[0], xn2[1]);
        dsum = (r == 0) ? d : dsum + d;
        ssum = (r == 0) ? sz : ssum + sz;
      }
    }
    if (c < m) {
      atomic_max_nonneg(&a.change[b], dsum);
      atomic_max_nonneg(&a.size[b], ssum);
    }
    return;
  }
  // rows in chunks of 8 with every load of the chunk issued before the (row-ordered) sums:
  // the permuted-storage gathers are scattered, so their latency needs overlapping when
  // few columns (threads) are in flight (small batches at large n)
  constexpr int U = 8;
  int r = 0;
  for (; r + U <= n; r += U) {
    double xi[U], yi[U], xo[U], yo[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t e = (size_t)(r + u) * n + c;
      xi[u] = RX[(size_t)xp[r + u] * n + qxc];
      yi[u] = a.first ? ((r + u == c) ? 1.0 : 0.0) : RY[(size_t)yp[r + u] * n + qyc];
      xo[u] = X[e];
      yo[u] = Y[e];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t e = (size_t)(r + u) * n + c;
      const double xn = 0.5 * (mu * xo[u] + yi[u] * inv_mu);
      const double yn = 0.5 * (mu * yo[u] + xi[u] * inv_mu);
      X[e] = xn;
      Y[e] = yn;
      dsum = (r + u == 0) ? fabs(xn - xo[u]) : dsum + fabs(xn - xo[u]);
      ssum = (r + u == 0) ? fabs(xn) : ssum + fabs(xn);
    }
  }
  for (; r < n; ++r) {
    const size_t e = (size_t)r * n + c;
    const double xinv = RX[(size_t)xp[r] * n + qxc];
    const double yinv = a.first ? ((r == c) ? 1.0 : 0.0) : RY[(size_t)yp[r] * n + qyc];
    const double xo = X[e];
    const double xn = 0.5 * (mu * xo + yinv * inv_mu);
    const double yn = 0.5 * (mu * Y[e] + xinv * inv_mu);
    X[e] = xn;
    Y[e] = yn;
    dsum = (r == 0) ? fabs(xn - xo) : dsum + fabs(xn - xo);
    ssum = (r == 0) ? fabs(xn) : ssum + fabs(xn);
  }
  atomic_max_nonneg(&a.change[b], dsum);
  atomic_max_nonneg(&a.size[b], ssum);
}

// Lazy X^-1 fix-up (matrices of LS_PMISS: predicted last, not converged): Y' from the X^-1 just
// formed (db_update_kernel's formula), X <- X' from the spare slot.  An exactly singular X
// ends the root as the eager order would have (status SINGULAR, that iteration not counted).
__global__ void __launch_bounds__(128) db_fix_kernel(DbArgs a, int nodes) {
  if (blockIdx.x == 0 && blockIdx.y == 0) count_nodes(nodes);
  if (blockIdx.y >= *a.L.cnt) return;
  const int b = a.L.ids[blockIdx.y];
  const int n = a.S.n;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (a.istat[b]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.ms[b].dbst = LGM_SINGULAR;
      a.ms[b].dbit -= 1;
    }
    return;
  }
  if (c >= n) return;
  double* X = a.S.buf(b, G_B);
  double* Y = a.S.buf(b, G_Y);
  const double* Xn = a.S.buf(b, a.xn_slot);
  const double* RX = a.S.buf(b, G_XI);
  const int* xp = a.xpiv + (size_t)b * n;
  const int qxc = a.xstep[(size_t)b * n + c];
  double mu = 1.0;
  if (a.scaling[b]) mu = fmin(fmax(exp(-(a.xlog[b] + a.ylog[b]) / (2.0 * n)), LGM_MU_MIN), LGM_MU_MAX);
  const double inv_mu = 1.0 / mu;
  for (int r = 0; r < n; ++r) {
    const size_t e = (size_t)r * n + c;
    Y[e] = 0.5 * (mu * Y[e] + RX[(size_t)xp[r] * n + qxc] * inv_mu);
    X[e] = Xn[e];
  }
}

// ------------------------------------------------------------------------------------------
// Block 1-norm estimator, batched.  Vectors are column-major n x 2 per job.
struct EstJob {
  const double* M1;
  const double* M2;   // nullable: operator M1^p1 * M2
  int p1;
  int live;           // slot in use (device-built tables are capacity-sized)
  int zchk;           // est_power_norm's zero-matrix shortcut applies (matcore.py:309-310)
  int nzf;            // set by est_nz_kernel when M1 has a nonzero entry
  int owner, key;     // matrix index and cache key (power) of the request
  int cplx;           // vectors are complex embeddings [Re; Im] of length n = 2m (decisions on Z)
  double* V0;         // ping
  double* V1;         // pong
  double* part;       // adjoint partial sums [splits][2][n]
  int* hist;          // [16]
  // state
  double est;
  int best_j, ncols, done, nhist, passes, total;
  double mm;
};

// initial block X (matcore.py:265-271): ones / m and the normalised alternating ramp, m = the
// operator's order (Z's for a complex embedding: [Re; Im] with zero imaginary parts)
__device__ __forceinline__ int est_x0(const EstJob& J, int n, double rsum, double rsum_c, int i0, int step) {
  const bool cx = J.cplx;
  const int m = cx ? n / 2 : n;
  const double rs = cx ? rsum_c : rsum;
  const int t = m < 2 ? m : 2;
  for (int i = i0; i < n; i += step) {
    const bool re = i < m;
    J.V0[i] = re ? 1.0 / m : 0.0;
    if (t > 1) J.V0[n + i] = re ? (((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(m > 1 ? m - 1 : 1))) / rs : 0.0;
  }
  return t;
}
__global__ void est_init_kernel(EstJob* jobs, int n, double rsum, double rsum_c) {
  EstJob& J = jobs[blockIdx.y];
  if (!J.live) {  // unused slot of a device-built table (its vectors are not assigned)
    if (blockIdx.x == 0 && threadIdx.x == 0) J.done = 1;
    return;
  }
  const int t = est_x0(J, n, rsum, rsum_c, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    J.est = 0.0; J.best_j = 0; J.ncols = t; J.nhist = 0; J.passes = 0; J.mm = INFINITY;
    J.total = J.p1 + (J.M2 ? 1 : 0);
    J.done = (!J.live || (J.zchk && !J.nzf)) ? 1 : 0;
  }
}

// est_power_norm's zero shortcut: flag jobs whose M1 has a nonzero entry (CTAs skip the scan
// once the flag is set)
__global__ void est_nz_kernel(EstJob* jobs, int n) {
  EstJob& J = jobs[blockIdx.y];
  if (!J.live || !J.zchk || *(volatile int*)&J.nzf) return;
  bool nz = false;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)n * n; idx += (size_t)gridDim.x * blockDim.x)
    nz |= J.M1[idx] != 0.0;
  if (__syncthreads_or(nz) && threadIdx.x == 0) J.nzf = 1;
}

// One thin product for every job still running: step q of the forward (trans=0) or adjoint
// (trans=1) application.  Forward: q = 0 is M2 (if present), then M1; adjoint: M1^T p1
// times then M2^T.  src = V[q%2], dst = V[(q+1)%2].
#ifndef EST_FWD_R
#define EST_FWD_R 4
#endif
// Job order alternates between consecutive thin products (boustrophedon): the matrices read
// last by one product are read first by the next, while they are still L2 resident.
__device__ __forceinline__ int est_job(int q, int flip, unsigned bi, unsigned nb) {
  return ((q ^ flip) & 1) ? (int)(nb - 1 - bi) : (int)bi;
}
__global__ void __launch_bounds__(256) est_fwd_kernel(EstJob* jobs, int n, int q) {
  EstJob& J = jobs[est_job(q, 0, blockIdx.y, gridDim.y)];
  if (J.done || q >= J.total) return;
  const double* M = (J.M2 && q == 0) ? J.M2 : J.M1;
  const double* x = (q & 1) ? J.V1 : J.V0;
  double* y = (q & 1) ? J.V0 : J.V1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // EST_FWD_R rows per warp (each row accumulated in the plain lane-strided order): the x
  // loads are shared by the warp's rows and each lane keeps EST_FWD_R row streams in flight
  const int i0 = (blockIdx.x * 8 + warp) * EST_FWD_R;
  if (i0 >= n) return;
  const int nc = J.ncols;
  double a0[EST_FWD_R], a1[EST_FWD_R];
#pragma unroll
  for (int q = 0; q < EST_FWD_R; ++q) a0[q] = a1[q] = 0.0;
  const double* Mr = M + (size_t)i0 * n;
  const int nr = min(EST_FWD_R, n - i0);
  for (int j = lane; j < n; j += 32) {
    const double x0 = x[j], x1 = nc > 1 ? x[n + j] : 0.0;
#pragma unroll
    for (int q = 0; q < EST_FWD_R; ++q) {
      if (q < nr) {
        const double m = Mr[(size_t)q * n + j];
        a0[q] = fma(m, x0, a0[q]);
        if (nc > 1) a1[q] = fma(m, x1, a1[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < EST_FWD_R; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0[q] += __shfl_xor_sync(0xffffffffu, a0[q], o);
      a1[q] += __shfl_xor_sync(0xffffffffu, a1[q], o);
    }
    if (lane == 0 && q < nr) {
      y[i0 + q] = a0[q];
      if (nc > 1) y[n + i0 + q] = a1[q];
    }
  }
}

constexpr int ADJ_ROWS = 64;
// z = M^T x: thread per column, a 64-row slab per CTA (partials reduced in fixed order by
// est_adj_reduce_kernel), 4 independent accumulators per column.
__global__ void __launch_bounds__(128) est_adj_kernel(EstJob* jobs, int n, int q, int flip) {
  EstJob& J = jobs[est_job(q, flip, blockIdx.z, gridDim.z)];
  if (J.done || q >= J.total) return;
  const double* M = (q < J.p1) ? J.M1 : J.M2;
  const double* x = (q & 1) ? J.V1 : J.V0;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int r0 = blockIdx.y * ADJ_ROWS, r1 = min(n, r0 + ADJ_ROWS);
  if (j >= n) return;
  const bool two = J.ncols > 1;
  double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
  int r = r0;
  for (; r + 3 < r1; r += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double m = M[(size_t)(r + u) * n + j];
      a0[u] = fma(m, x[r + u], a0[u]);
      if (two) a1[u] = fma(m, x[n + r + u], a1[u]);
    }
  }
  for (; r < r1; ++r) {
    const double m = M[(size_t)r * n + j];
    a0[0] = fma(m, x[r], a0[0]);
    if (two) a1[0] = fma(m, x[n + r], a1[0]);
  }
  J.part[((size_t)blockIdx.y * 2 + 0) * n + j] = (a0[0] + a0[1]) + (a0[2] + a0[3]);
  J.part[((size_t)blockIdx.y * 2 + 1) * n + j] = (a1[0] + a1[1]) + (a1[2] + a1[3]);
}

// Even n: two adjacent columns per thread (16-byte loads: twice the bytes per request of the
// kernel above, same per-column accumulation order, so the same partial sums).
__global__ void __launch_bounds__(128) est_adj2_kernel(EstJob* jobs, int n, int q, int flip) {
  EstJob& J = jobs[est_job(q, flip, blockIdx.z, gridDim.z)];
  if (J.done || q >= J.total) return;
  const double* M = (q < J.p1) ? J.M1 : J.M2;
  const double* x = (q & 1) ? J.V1 : J.V0;
  const int j = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int r0 = blockIdx.y * ADJ_ROWS, r1 = min(n, r0 + ADJ_ROWS);
  if (j >= n) return;
  const bool two = J.ncols > 1;
  double a0[2][4] = {}, a1[2][4] = {};
  int r = r0;
  for (; r + 3 < r1; r += 4) {
    double2 m[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) m[u] = *reinterpret_cast<const double2*>(&M[(size_t)(r + u) * n + j]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double xa = x[r + u];
      a0[0][u] = fma(m[u].x, xa, a0[0][u]);
      a0[1][u] = fma(m[u].y, xa, a0[1][u]);
      if (two) {
        const double xb = x[n + r + u];
        a1[0][u] = fma(m[u].x, xb, a1[0][u]);
        a1[1][u] = fma(m[u].y, xb, a1[1][u]);
      }
    }
  }
  for (; r < r1; ++r) {
    const double2 m = *reinterpret_cast<const double2*>(&M[(size_t)r * n + j]);
    a0[0][0] = fma(m.x, x[r], a0[0][0]);
    a0[1][0] = fma(m.y, x[r], a0[1][0]);
    if (two) {
      a1[0][0] = fma(m.x, x[n + r], a1[0][0]);
      a1[1][0] = fma(m.y, x[n + r], a1[1][0]);
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    J.part[((size_t)blockIdx.y * 2 + 0) * n + j + e] = (a0[e][0] + a0[e][1]) + (a0[e][2] + a0[e][3]);
    J.part[((size_t)blockIdx.y * 2 + 1) * n + j + e] = (a1[e][0] + a1[e][1]) + (a1[e][2] + a1[e][3]);
  }
}

__global__ void est_adj_reduce_kernel(EstJob* jobs, int n, int q, int splits) {
  EstJob& J = jobs[blockIdx.y];
  if (J.done || q >= J.total) return;
  double* y = (q & 1) ? J.V0 : J.V1;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a0 = 0.0, a1 = 0.0;
  for (int s = 0; s < splits; ++s) {
    a0 += J.part[((size_t)s * 2 + 0) * n + j];
    a1 += J.part[((size_t)s * 2 + 1) * n + j];
  }
  y[j] = a0;
  if (J.ncols > 1) y[n + j] = a1;
}

__device__ __forceinline__ void mgap(double& mm, double a, double b) {
  double den = fmax(fabs(a), fabs(b));
  mm = fmin(mm, den > 0.0 ? fabs(a - b) / den : 0.0);
}

// After the forward application: column 1-norms, argmax, estimate update, S = sign(Y).
// (CTA-wide body: 256 threads per job, shared by the per-step kernels and est_fused_kernel)
template <bool CXT>
__device__ void est_after_fwd_impl(EstJob& J, int n, int sweep, double* sred) {
  if (J.done) return;
  double* Yv = (J.total & 1) ? J.V1 : J.V0;
  const int nc = J.ncols;
  constexpr bool cx = CXT;
  const int m = cx ? n / 2 : n;  // Z's order; an entry's Im part sits m below its Re part
  double cn[2] = {0.0, 0.0};
  for (int c = 0; c < nc; ++c) {
    double v = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) v += cx ? hypot(Yv[c * n + i], Yv[c * n + i + m]) : fabs(Yv[c * n + i]);
    cn[c] = block_sum(v, sred);
  }
  const int j = (nc > 1 && cn[1] > cn[0]) ? 1 : 0;
  double mm = J.mm;
  if (nc > 1) mgap(mm, cn[0], cn[1]);
  const double cand = cn[j];
  if (J.est > 0.0) mgap(mm, cand, J.est);
  bool stop = false;
  double est = J.est;
  int best = J.best_j;
  if (cand > est) { est = cand; best = j; }
  else if (sweep > 0) stop = true;
  __syncthreads();
  if (threadIdx.x == 0) {
    J.est = est; J.best_j = best; J.mm = mm; J.passes += J.total;
    if (stop) J.done = 1;
  }
  if (!stop) {  // S = sign(Y) in place (matcore.py:226-231); the adjoint reads it as step 0 input
    double* D = (J.total & 1) ? J.V0 : Yv;  // adjoint starts from V0: move if Y landed in V1
    for (int c = 0; c < nc; ++c)
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        if (cx) {  // complex sign: y / |y|, 1 where y = 0
          const double re = Yv[c * n + i], im = Yv[c * n + i + m];
          const double a = hypot(re, im);
          D[c * n + i] = a == 0.0 ? 1.0 : re / a;
          D[c * n + i + m] = a == 0.0 ? 0.0 : im / a;
        } else {
          D[c * n + i] = (Yv[c * n + i] >= 0.0) ? 1.0 : -1.0;
        }
      }
  }
}
__device__ void est_after_fwd_body(EstJob& J, int n, int sweep, double* sred) {
  if (J.cplx) est_after_fwd_impl<true>(J, n, sweep, sred);
  else est_after_fwd_impl<false>(J, n, sweep, sred);
}
template <bool CX>
__global__ void __launch_bounds__(256) est_after_fwd_kernel(EstJob* jobs, int n, int sweep) {
  __shared__ double sred[8];
  est_after_fwd_impl<CX>(jobs[blockIdx.x], n, sweep, sred);
}

// After the adjoint: h = row max |Z|, top-(4t+1) order, picks, stopping test, next X.
constexpr int ETK_PER = 16;  // rows per lane of the warp top-k (m <= 512)
struct EstAdjSmem {
  uint64_t skey[8];
  int sidx[8];
  int order[9];
  double hval[9];
};
template <bool CXT>
__device__ void est_after_adj_impl(EstJob& J, int n, int sweep, EstAdjSmem& sa) {
  uint64_t* skey = sa.skey;
  int* sidx = sa.sidx;
  int* order = sa.order;
  double* hval = sa.hval;
  if (J.done) return;
  const double* Z = (J.total & 1) ? J.V1 : J.V0;
  const int nc = J.ncols;
  constexpr bool cx = CXT;
  const int m = cx ? n / 2 : n;  // Z's order (complex embeddings: Im parts m below)
  auto zabs = [&](int off) { return cx ? hypot(Z[off], Z[off + m]) : fabs(Z[off]); };
  const int t = m < 2 ? m : 2;
  const int ntop = m < 4 * t + 1 ? m : 4 * t + 1;
  if (m <= 32 * ETK_PER) {
    // warp 0: lane l keeps the keys of rows l + 32 e in registers; ntop rounds of a warp
    // argmax (max key, ties -> lowest row), the winner's key cleared -- the same order as the
    // repeated block argmax below, without a block barrier per round
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint64_t kk[ETK_PER];
#pragma unroll
      for (int e = 0; e < ETK_PER; ++e) {
        const int i = lane + 32 * e;
        uint64_t k = 0ull;
        if (i < m) {
          double h = zabs(i);
          if (nc > 1) h = fmax(h, zabs(n + i));
          k = dkey(h);
        }
        kk[e] = k;
      }
      for (int qq = 0; qq < ntop; ++qq) {
        uint64_t key = 0ull;
        int idx = 0x7fffffff;
#pragma unroll
        for (int e = 0; e < ETK_PER; ++e)
          if (kk[e] > key) { key = kk[e]; idx = lane + 32 * e; }  // rows ascend with e: ties keep the lowest
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t k2 = __shfl_xor_sync(0xffffffffu, key, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
          if (k2 > key || (k2 == key && i2 < idx)) { key = k2; idx = i2; }
        }
        if ((idx & 31) == lane) {
#pragma unroll
          for (int e = 0; e < ETK_PER; ++e)
            if (lane + 32 * e == idx) kk[e] = 0ull;
        }
        if (lane == 0) { order[qq] = idx; hval[qq] = __longlong_as_double((long long)(key - 1ull)); }
      }
    }
    __syncthreads();
  } else {
    // repeated block argmax over h with exclusion of already taken rows
    for (int qq = 0; qq < ntop; ++qq) {
      uint64_t key = 0ull;
      int idx = 0x7fffffff;
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        bool taken = false;
        for (int u = 0; u < qq; ++u) taken |= (order[u] == i);
        if (taken) continue;
        double h = zabs(i);
        if (nc > 1) h = fmax(h, zabs(n + i));
        uint64_t kq = dkey(h);
        if (kq > key) { key = kq; idx = i; }
      }
      uint64_t kmax;
      int p;
      block_argmax(key, idx, skey, sidx, kmax, p);
      if (threadIdx.x == 0) { order[qq] = p; hval[qq] = __longlong_as_double((long long)(kmax - 1ull)); }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    double mm = J.mm;
    for (int a = 0; a + 1 < ntop && a < 4 * t; ++a) mgap(mm, hval[a], hval[a + 1]);
    int picks[2], np = 0;
    const int lim = ntop < 4 * t ? ntop : 4 * t;
    for (int qq = 0; qq < lim && np < t; ++qq) {
      int i = order[qq];
      bool seen = false;
      for (int u = 0; u < J.nhist; ++u) seen |= (J.hist[u] == i);
      if (!seen) picks[np++] = i;
    }
    auto hrow = [&](int i) { double h = zabs(i); if (nc > 1) h = fmax(h, zabs(n + i)); return h; };
    const double h0 = hval[0], hb = hrow(J.best_j);
    if (sweep > 0 && order[0] != J.best_j) mgap(mm, h0, hb);
    J.mm = mm;
    J.passes += J.total;
    if (np == 0 || (sweep > 0 && h0 <= hb)) {
      J.done = 1;
    } else {
      for (int c = 0; c < np; ++c) J.hist[J.nhist++] = picks[c];
      J.ncols = np;
      order[0] = picks[0];
      order[1] = np > 1 ? picks[1] : -1;
    }
  }
  __syncthreads();
  if (J.done) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    J.V0[i] = (i == order[0]) ? 1.0 : 0.0;
    J.V0[n + i] = (i == order[1]) ? 1.0 : 0.0;
  }
}
__device__ void est_after_adj_body(EstJob& J, int n, int sweep, EstAdjSmem& sa) {
  if (J.cplx) est_after_adj_impl<true>(J, n, sweep, sa);
  else est_after_adj_impl<false>(J, n, sweep, sa);
}
template <bool CX>
__global__ void __launch_bounds__(256) est_after_adj_kernel(EstJob* jobs, int n, int sweep) {
  __shared__ EstAdjSmem sa;
  est_after_adj_impl<CX>(jobs[blockIdx.x], n, sweep, sa);
}

// The whole estimate for one job per CTA (256 threads), M1 resident in shared memory
// (n <= EST_FUSED_MAXN): one launch instead of 1 + itmax (2 total + 2) per-step launches.
// Every reduction reproduces the per-step kernels' order exactly (forward: warp per row,
// lane-strided FMAs + butterfly; adjoint: thread per column, 64-row slabs with 4 accumulators,
// slab partials summed in order; the after-bodies are shared), so the two paths agree bit for bit.
constexpr int EST_FUSED_MAXN = 160;
#ifndef EST_FUSED_V2
#define EST_FUSED_V2 1
#endif
#if EST_FUSED_V2
constexpr int ESTF_THREADS = 512;
#else
constexpr int ESTF_THREADS = 256;
#endif
#if EST_FUSED_V2
// Version 2 (default; -DEST_FUSED_V2=0 builds the first version): the same sums in the same
// order, arranged for the single CTA that runs them --
//  * the job state and the two ping-pong vectors live in shared memory (a shared EstJob copy
//    whose V0 / V1 point at shared buffers; the shared after-bodies work on it unchanged) and
//    the state is written back once at the end: no L2 round trip per dependent step;
//  * forward: a warp accumulates 16 of its rows at a time (lane-strided FMAs, one x load per
//    16 rows) and reduces them with a butterfly reduce-scatter (stages 16, 8, 4, 2, then the
//    final xor 1): per row the additions pair the same lane subsets in the same order as the
//    plain butterfly, with 32 shuffles per 16 rows instead of 160;
//  * adjoint: two threads per column, thread h forming (a_2h + a_2h+1) of each 64-row slab
//    (rows = 2h, 2h + 1 mod 4; the remainder rows join a_0 as in est_adj_kernel), the column
//    owner adding the halves and the slabs in order.
// ESTF_NT threads (512 for n > ESTF_SMALL_N, else 256): the thread count only adds zero terms to
// the after-bodies' block sums (n <= 160 < 256), so every variant gives the same bits
constexpr int ESTF_SMALL_N = 96;
template <bool CX, int ESTF_NT = 512>
__global__ void __launch_bounds__(ESTF_NT) est_fused_kernel(EstJob* jobs, int n, double rsum, double rsum_c, int itmax) {
  extern __shared__ __align__(16) double Ms[];
  __shared__ double sred[ESTF_NT / 32];
  __shared__ EstAdjSmem sa;
  __shared__ EstJob Js;
  __shared__ __align__(16) double Vs[2][2 * EST_FUSED_MAXN];
  constexpr int MAXSPL = (EST_FUSED_MAXN + ADJ_ROWS - 1) / ADJ_ROWS;
  __shared__ double parts[MAXSPL][2][EST_FUSED_MAXN];  // adjoint slab partials (est_adj_reduce_kernel's inputs)
  EstJob& Jg = jobs[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = ESTF_NT / 32;
  if (!Jg.live) {  // unused slot of a device-built table
    if (tid == 0) Jg.done = 1;
    return;
  }
  const bool skip = Jg.zchk && !Jg.nzf;  // (uniform: set before the launch)
  if (tid == 0) {
    Js = Jg;
    Js.V0 = Vs[0];
    Js.V1 = Vs[1];
  }
  __syncthreads();
  EstJob& J = Js;
  {  // est_init_kernel
    const int t = est_x0(J, n, rsum, rsum_c, tid, ESTF_NT);
    if (tid == 0) {
      J.est = 0.0; J.best_j = 0; J.ncols = t; J.nhist = 0; J.passes = 0; J.mm = INFINITY;
      J.total = J.p1 + (J.M2 ? 1 : 0);
      J.done = skip ? 1 : 0;
    }
  }
  auto write_back = [&]() {
    __syncthreads();
    if (tid == 0) {
      Jg.est = J.est; Jg.best_j = J.best_j; Jg.ncols = J.ncols; Jg.done = J.done; Jg.nhist = J.nhist;
      Jg.passes = J.passes; Jg.total = J.total; Jg.mm = J.mm;
    }
  };
  if (skip) { write_back(); return; }
  for (int idx = tid; idx < n * n; idx += ESTF_NT) Ms[idx] = J.M1[idx];
  __syncthreads();
  const int total = J.p1 + (J.M2 ? 1 : 0);
  const int splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
  const int cblocks = (n + 15) / 16;
  for (int sweep = 0; sweep < itmax; ++sweep) {
    if (J.done) break;
    const int nc = J.ncols;
    for (int q = 0; q < total; ++q) {  // forward (est_fwd_kernel's sums)
      const double* M = (J.M2 && q == 0) ? J.M2 : Ms;
      const double* x = (q & 1) ? Vs[1] : Vs[0];
      double* y = (q & 1) ? Vs[0] : Vs[1];
      for (int ib = warp; ib < n; ib += NW * 8) {  // rows ib + NW r, r = 0..7
        double a0[8], a1[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a0[r] = a1[r] = 0.0;
        for (int j = lane; j < n; j += 32) {
          const double x0 = x[j], x1 = nc > 1 ? x[n + j] : 0.0;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int i = ib + NW * r;
            const double m = i < n ? M[(size_t)i * n + j] : 0.0;
            a0[r] = fma(m, x0, a0[r]);
            a1[r] = fma(m, x1, a1[r]);
          }
        }
        // reduce-scatter with offsets 16, 8, 4 (lane l then holds row r = 4 b4 + 2 b3 + b2, b_k =
        // bit k of l), then the plain xor-2 and xor-1 stages: the butterfly's pairings in its order
#pragma unroll
        for (int off = 16, len = 8; off >= 4; off >>= 1, len >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (r < len / 2) {
              const double s0 = up ? a0[r] : a0[r + len / 2], k0 = up ? a0[r + len / 2] : a0[r];
              const double s1 = up ? a1[r] : a1[r + len / 2], k1 = up ? a1[r + len / 2] : a1[r];
              a0[r] = k0 + __shfl_xor_sync(0xffffffffu, s0, off);
              a1[r] = k1 + __shfl_xor_sync(0xffffffffu, s1, off);
            }
          }
        }
#pragma unroll
        for (int off = 2; off >= 1; off >>= 1) {
          a0[0] += __shfl_xor_sync(0xffffffffu, a0[0], off);
          a1[0] += __shfl_xor_sync(0xffffffffu, a1[0], off);
        }
        const int i = ib + NW * (lane >> 2);
        if ((lane & 3) == 0 && i < n) {
          y[i] = a0[0];
          if (nc > 1) y[n + i] = a1[0];
        }
      }
      __syncthreads();
    }
    est_after_fwd_impl<CX>(J, n, sweep, sred);
    __syncthreads();
    if (J.done) break;
    const bool two = J.ncols > 1;
    for (int q = 0; q < total; ++q) {  // adjoint (est_adj_kernel + est_adj_reduce_kernel's sums)
      const double* M = (q < J.p1) ? Ms : J.M2;
      const double* x = (q & 1) ? Vs[1] : Vs[0];
      double* y = (q & 1) ? Vs[0] : Vs[1];
      // one warp task = (64-row slab, 16 columns): lanes 0-15 form a0 + a1 of their column over the
      // slab, lanes 16-31 a2 + a3 (each half-warp reads one contiguous 128-byte row segment)
      for (int task = warp; task < splits * cblocks; task += NW) {
        const int sl = task / cblocks, j = (task - sl * cblocks) * 16 + (lane & 15), h = lane >> 4;
        const int r0 = sl * ADJ_ROWS, r1 = min(n, r0 + ADJ_ROWS);
        double b0[2] = {0.0, 0.0}, b1[2] = {0.0, 0.0};
        if (j < n) {
          int r = r0;
          for (; r + 3 < r1; r += 4) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int rr = r + 2 * h + u;
              const double m = M[(size_t)rr * n + j];
              b0[u] = fma(m, x[rr], b0[u]);
              if (two) b1[u] = fma(m, x[n + rr], b1[u]);
            }
          }
          if (h == 0) {
            for (; r < r1; ++r) {
              const double m = M[(size_t)r * n + j];
              b0[0] = fma(m, x[r], b0[0]);
              if (two) b1[0] = fma(m, x[n + r], b1[0]);
            }
          }
        }
        const double p0 = b0[0] + b0[1], p1 = b1[0] + b1[1];
        const double o0 = __shfl_xor_sync(0xffffffffu, p0, 16), o1 = __shfl_xor_sync(0xffffffffu, p1, 16);
        if (h == 0 && j < n) {
          parts[sl][0][j] = p0 + o0;  // (a0 + a1) + (a2 + a3)
          parts[sl][1][j] = p1 + o1;
        }
      }
      __syncthreads();  // partials complete; every thread has read x before y (the other buffer) is written
      if (tid < n) {
        double s0 = 0.0, s1 = 0.0;
        for (int sl = 0; sl < splits; ++sl) {
          s0 += parts[sl][0][tid];
          s1 += parts[sl][1][tid];
        }
        y[tid] = s0;
        if (two) y[n + tid] = s1;
      }
      __syncthreads();
    }
    est_after_adj_impl<CX>(J, n, sweep, sa);
    __syncthreads();
  }
  write_back();
}
#else
template <bool CX>
__global__ void __launch_bounds__(256) est_fused_kernel(EstJob* jobs, int n, double rsum, double rsum_c, int itmax) {
  extern __shared__ __align__(16) double Ms[];
  __shared__ double sred[8];
  __shared__ EstAdjSmem sa;
  EstJob& J = jobs[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!J.live) {  // unused slot of a device-built table
    if (tid == 0) J.done = 1;
    return;
  }
  {  // est_init_kernel
    const int t = est_x0(J, n, rsum, rsum_c, tid, 256);
    if (tid == 0) {
      J.est = 0.0; J.best_j = 0; J.ncols = t; J.nhist = 0; J.passes = 0; J.mm = INFINITY;
      J.total = J.p1 + (J.M2 ? 1 : 0);
      J.done = (!J.live || (J.zchk && !J.nzf)) ? 1 : 0;
    }
  }
  if (!J.live || (J.zchk && !J.nzf)) return;  // (uniform: set before the launch)
  for (int idx = tid; idx < n * n; idx += 256) Ms[idx] = J.M1[idx];
  __syncthreads();
  const int total = J.p1 + (J.M2 ? 1 : 0);
  const int splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
  for (int sweep = 0; sweep < itmax; ++sweep) {
    if (J.done) break;
    const int nc = J.ncols;
    for (int q = 0; q < total; ++q) {  // forward (est_fwd_kernel)
      const double* M = (J.M2 && q == 0) ? J.M2 : Ms;
      const double* x = (q & 1) ? J.V1 : J.V0;
      double* y = (q & 1) ? J.V0 : J.V1;
      for (int i = warp; i < n; i += 8) {
        double a0 = 0.0, a1 = 0.0;
        const double* Mr = M + (size_t)i * n;
        for (int j = lane; j < n; j += 32) {
          const double m = Mr[j];
          a0 = fma(m, x[j], a0);
          if (nc > 1) a1 = fma(m, x[n + j], a1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a0 += __shfl_xor_sync(0xffffffffu, a0, o);
          a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        if (lane == 0) {
          y[i] = a0;
          if (nc > 1) y[n + i] = a1;
        }
      }
      __syncthreads();
    }
    est_after_fwd_impl<CX>(J, n, sweep, sred);
    __syncthreads();
    if (J.done) break;
    const bool two = J.ncols > 1;
    for (int q = 0; q < total; ++q) {  // adjoint (est_adj_kernel + est_adj_reduce_kernel)
      const double* M = (q < J.p1) ? Ms : J.M2;
      const double* x = (q & 1) ? J.V1 : J.V0;
      double* y = (q & 1) ? J.V0 : J.V1;
      const int j = tid;
      double s0 = 0.0, s1 = 0.0;
      if (j < n) {
        for (int sl = 0; sl < splits; ++sl) {
          const int r0 = sl * ADJ_ROWS, r1 = min(n, r0 + ADJ_ROWS);
          double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
          int r = r0;
          for (; r + 3 < r1; r += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double m = M[(size_t)(r + u) * n + j];
              a0[u] = fma(m, x[r + u], a0[u]);
              if (two) a1[u] = fma(m, x[n + r + u], a1[u]);
            }
          }
          for (; r < r1; ++r) {
            const double m = M[(size_t)r * n + j];
            a0[0] = fma(m, x[r], a0[0]);
            if (two) a1[0] = fma(m, x[n + r], a1[0]);
          }
          s0 += (a0[0] + a0[1]) + (a0[2] + a0[3]);
          s1 += (a1[0] + a1[1]) + (a1[2] + a1[3]);
        }
      }
      __syncthreads();  // every thread has read x before y (the other buffer) is written
      if (j < n) {
        y[j] = s0;
        if (two) y[n + j] = s1;
      }
      __syncthreads();
    }
    est_after_adj_impl<CX>(J, n, sweep, sa);
    __syncthreads();
  }
}

#endif  // EST_FUSED_V2

// ------------------------------------------------------------------------------------------
// The whole estimate of one job per thread-block cluster (EST_FUSED_MAXN < n <= 512), M1
// resident in the cluster's shared memory for every thin product of every sweep instead of
// streamed from HBM once per product.  The cluster has CL = 2 ceil(n / 64) CTAs (<= 16): CTA
// q = 2 s + h holds the rows of the per-step adjoint's 64-row slab s whose residue u (mod 4)
// inside the slab's full 4-row groups is 2h or 2h + 1, plus (h = 0) the slab's remainder rows,
// so every reduction is the per-step kernels' own (bit-identical estimates):
//  * forward y = M x: a warp per row, lane-strided FMAs + butterfly (est_fwd_kernel); the row
//    results are pushed into every CTA's copy of y (DSMEM stores), one cluster barrier;
//  * adjoint z = M^T x: per column the CTA forms its two interleaved accumulators of the slab
//    (a_2h, a_2h+1, remainder rows into a_0) and their sum -- half of est_adj_kernel's
//    (a0 + a1) + (a2 + a3) -- and pushes it to the column's owner CTA; barrier; the owner adds
//    the slab halves and the slabs in order (est_adj_reduce_kernel) and pushes the column into
//    every CTA's y; barrier.
// The after-bodies (norms, argmax, top-k, history, stop tests) run redundantly on every CTA's
// identical local copy of the vectors and job state (one barrier after each, so no push of
// the next product lands in a vector a slower peer still reads); rank 0 publishes the result.
constexpr int ECL_NT = 256;
constexpr int ECL_MAXR = 32;   // rows per CTA
constexpr int ECL_MAXC = 32;   // adjoint columns owned per CTA
constexpr int ECL_MAXCL = 16;
struct EclSmem {
  EstJob S;           // this CTA's copy of the job state (V0 / V1 / hist point into shared)
  double sred[8];
  EstAdjSmem sa;
  int hist[16];
  int grow[ECL_MAXR];                 // local row -> global row
  double own[2][ECL_MAXC];            // owned adjoint columns (both vectors)
};
inline int ecl_cl(int n) { return 2 * ((n + 63) / 64); }
inline size_t ecl_smem(int n) {
  return ((size_t)ECL_MAXR * n + 4 * (size_t)n + (size_t)ECL_MAXCL * 2 * ECL_MAXC) * 8;
}
// forward rows lr0 .. lr0 + nr - 1 of the cluster estimator (est_fwd_kernel's per-row order):
// from shared memory (M1) or, for the product form's first step, from M2 in global memory
template <bool GM>
__device__ __forceinline__ void ecl_fwd_rows(const double* M2, const int* grow, const double* Ms, int n, int lr0,
                                             int nr, int nc, const double* x, int lane, double (&a0)[4],
                                             double (&a1)[4]) {
  const double* Mr[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int lr = lr0 + (rr < nr ? rr : nr - 1);
    Mr[rr] = GM ? M2 + (size_t)grow[lr] * n : Ms + (size_t)lr * n;
  }
#pragma unroll 4
  for (int j = lane; j < n; j += 32) {
    const double x0 = x[j], x1 = nc > 1 ? x[n + j] : 0.0;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      if (rr < nr) {
        const double m = Mr[rr][j];
        a0[rr] = fma(m, x0, a0[rr]);
        if (nc > 1) a1[rr] = fma(m, x1, a1[rr]);
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0[rr] += __shfl_xor_sync(0xffffffffu, a0[rr], o);
      a1[rr] += __shfl_xor_sync(0xffffffffu, a1[rr], o);
    }
  }
}
// adjoint slab halves of columns tid and tid + ECL_NT (est_adj_kernel's accumulators a_2h,
// a_2h+1, remainder rows into a_0), pushed to each column's owner CTA
template <bool GM>
__device__ __forceinline__ void ecl_adj_cols(const double* M2, const int* grow, const double* Ms, int n, int NG, int R,
                                             bool two, const double* x, int tid, int rank, int RC, double* recv,
                                             cooperative_groups::cluster_group& cl) {
  const int c0 = tid, c1 = tid + ECL_NT;
  const bool v0 = c0 < n, v1 = c1 < n;
  const int d0 = v0 ? c0 : 0, d1 = v1 ? c1 : 0;
  double lo[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, hi[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [column][vector]
#pragma unroll 2
  for (int i = 0; i < NG; ++i) {
    const int g0 = grow[2 * i], g1 = grow[2 * i + 1];
    const double* r0 = GM ? M2 + (size_t)g0 * n : Ms + (size_t)(2 * i) * n;
    const double* r1 = GM ? M2 + (size_t)g1 * n : Ms + (size_t)(2 * i + 1) * n;
    const double m00 = r0[d0], m10 = r1[d0], m01 = r0[d1], m11 = r1[d1];
    const double xa = x[g0], xb = x[g1];
    lo[0][0] = fma(m00, xa, lo[0][0]);
    hi[0][0] = fma(m10, xb, hi[0][0]);
    lo[1][0] = fma(m01, xa, lo[1][0]);
    hi[1][0] = fma(m11, xb, hi[1][0]);
    if (two) {
      const double ya = x[n + g0], yb = x[n + g1];
      lo[0][1] = fma(m00, ya, lo[0][1]);
      hi[0][1] = fma(m10, yb, hi[0][1]);
      lo[1][1] = fma(m01, ya, lo[1][1]);
      hi[1][1] = fma(m11, yb, hi[1][1]);
    }
  }
  for (int lr = 2 * NG; lr < R; ++lr) {  // remainder rows (h = 0): accumulator a_0
    const int g = grow[lr];
    const double* rr = GM ? M2 + (size_t)g * n : Ms + (size_t)lr * n;
    const double ma = rr[d0], mb = rr[d1];
    lo[0][0] = fma(ma, x[g], lo[0][0]);
    lo[1][0] = fma(mb, x[g], lo[1][0]);
    if (two) {
      lo[0][1] = fma(ma, x[n + g], lo[0][1]);
      lo[1][1] = fma(mb, x[n + g], lo[1][1]);
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int c = k ? c1 : c0;
    if (k ? v1 : v0) {
      const int ow = c / RC, oc = c - ow * RC;
      double* rv = cl.map_shared_rank(recv, ow);
      rv[(rank * 2 + 0) * ECL_MAXC + oc] = lo[k][0] + hi[k][0];
      rv[(rank * 2 + 1) * ECL_MAXC + oc] = lo[k][1] + hi[k][1];
    }
  }
}
#ifdef ECL_PROF  // clock64 phase split of job 0's estimate (rank 0, thread 0), printed per launch
#define ECL_T(v) long long v = clock64()
#define ECL_ADD(i, a, b) ecl_cyc[i] += (b) - (a)
#else
#define ECL_T(v)
#define ECL_ADD(i, a, b)
#endif
template <bool CX>
__global__ void __launch_bounds__(ECL_NT, 1) est_cluster_kernel(EstJob* jobs, int n, double rsum, double rsum_c,
                                                                int itmax) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double ecl[];
  __shared__ EclSmem es;
  const int CL = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  EstJob& G = jobs[blockIdx.x / CL];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Ms = ecl;                             // [ECL_MAXR][n] my rows of M1 (local order)
  double* V0 = Ms + (size_t)ECL_MAXR * n;       // [2][n]
  double* V1 = V0 + 2 * n;                      // [2][n]
  double* recv = V1 + 2 * n;                    // [CL][2][ECL_MAXC] adjoint slab halves
#ifdef ECL_PROF
  long long ecl_cyc[10] = {};
#endif
  ECL_T(t_init);
  const bool dead = !G.live || (G.zchk && !G.nzf);
  if (dead) {  // (uniform over the cluster: every CTA reads the same job)
    if (rank == 0 && tid == 0) {
      G.done = 1;
      G.est = 0.0;
      G.passes = 0;
      G.mm = INFINITY;
    }
    return;
  }
  // my rows: slab s, half h (see above)
  const int s = rank >> 1, h = rank & 1;
  const int L = min(64, n - 64 * s), NG = L >> 2, rem = L & 3;
  const int R = 2 * NG + (h == 0 ? rem : 0);
  const int RC = (n + CL - 1) / CL;             // adjoint columns owned per CTA
  if (tid < ECL_MAXR) {
    const int lr = tid;
    es.grow[lr] = lr < 2 * NG ? 64 * s + 4 * (lr >> 1) + 2 * h + (lr & 1) : 64 * s + 4 * NG + (lr - 2 * NG);
  }
  EstJob& S = es.S;
  if (tid == 0) {
    S = G;
    S.V0 = V0;
    S.V1 = V1;
    S.hist = es.hist;
  }
  __syncthreads();
  {
    const int t = est_x0(S, n, rsum, rsum_c, tid, ECL_NT);
    if (tid == 0) {
      S.est = 0.0; S.best_j = 0; S.ncols = t; S.nhist = 0; S.passes = 0; S.mm = INFINITY;
      S.total = S.p1 + (S.M2 ? 1 : 0);
      S.done = 0;
    }
  }
  for (int lr0 = 0; lr0 < R; lr0 += ECL_NT / 32) {  // warp per row, all of a lane's loads in flight
    const int lr = lr0 + warp;
    if (lr < R) {
      const double* src = G.M1 + (size_t)es.grow[lr] * n;
      double* dst = Ms + (size_t)lr * n;
      if ((n & 1) == 0) {
        double2 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = 2 * lane + 64 * e;
          if (j < n) v[e] = *reinterpret_cast<const double2*>(src + j);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = 2 * lane + 64 * e;
          if (j < n) *reinterpret_cast<double2*>(dst + j) = v[e];
        }
      } else {
        double v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int j = lane + 32 * e;
          if (j < n) v[e] = src[j];
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int j = lane + 32 * e;
          if (j < n) dst[j] = v[e];
        }
      }
    }
  }
  __syncthreads();
  cl.sync();  // every CTA's vectors initialised before the first push
  ECL_T(t_ld);
  ECL_ADD(0, t_init, t_ld);
  const int total = S.total, p1 = S.p1;
  const double* M2 = S.M2;
  for (int sweep = 0; sweep < itmax; ++sweep) {
    if (S.done) break;
    const int nc = S.ncols;
    for (int q = 0; q < total; ++q) {  // forward: y = M x for my rows, pushed to every CTA
      ECL_T(f0);
      const bool use2 = M2 && q == 0;
      const double* x = (q & 1) ? V1 : V0;
      double* y = (q & 1) ? V0 : V1;
      const int lr0 = warp * 4;
      if (lr0 < R) {
        const int nr = min(4, R - lr0);
        double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
        if (use2) ecl_fwd_rows<true>(M2, es.grow, Ms, n, lr0, nr, nc, x, lane, a0, a1);
        else ecl_fwd_rows<false>(M2, es.grow, Ms, n, lr0, nr, nc, x, lane, a0, a1);
        ECL_T(f1);
        ECL_ADD(1, f0, f1);
        if (lane < CL) {  // lane p stores the warp's rows into CTA p's y
          double* ry = cl.map_shared_rank(y, lane);
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            if (rr < nr) {
              const int gi = es.grow[lr0 + rr];
              ry[gi] = a0[rr];
              if (nc > 1) ry[n + gi] = a1[rr];
            }
          }
        }
      }
      ECL_T(f2);
      cl.sync();
      ECL_T(f3);
      ECL_ADD(2, f0, f2);
      ECL_ADD(3, f2, f3);
    }
    ECL_T(af0);
    est_after_fwd_impl<CX>(S, n, sweep, es.sred);
    __syncthreads();
    ECL_T(af1);
    ECL_ADD(4, af0, af1);
    cl.sync();  // no push of the adjoint lands in a vector a slower peer's after-body reads
    if (S.done) break;
    const bool two = S.ncols > 1;
    for (int q = 0; q < total; ++q) {  // adjoint: slab halves -> owner -> every CTA
      ECL_T(a0t);
      const bool use2 = q >= p1;
      const double* x = (q & 1) ? V1 : V0;
      double* y = (q & 1) ? V0 : V1;
      if (use2) ecl_adj_cols<true>(M2, es.grow, Ms, n, NG, R, two, x, tid, rank, RC, recv, cl);
      else ecl_adj_cols<false>(M2, es.grow, Ms, n, NG, R, two, x, tid, rank, RC, recv, cl);
      ECL_T(a1t);
      cl.sync();
      ECL_T(a2t);
      ECL_ADD(5, a0t, a1t);
      ECL_ADD(6, a1t, a2t);
      const int c0 = rank * RC, nown = max(0, min(RC, n - c0));
      if (tid < nown) {  // my columns: slab halves, then slabs in order, from 0.0
        double s0 = 0.0, s1 = 0.0;
        for (int sl = 0; sl < CL / 2; ++sl) {
          s0 += recv[((2 * sl) * 2 + 0) * ECL_MAXC + tid] + recv[((2 * sl + 1) * 2 + 0) * ECL_MAXC + tid];
          s1 += recv[((2 * sl) * 2 + 1) * ECL_MAXC + tid] + recv[((2 * sl + 1) * 2 + 1) * ECL_MAXC + tid];
        }
        es.own[0][tid] = s0;
        es.own[1][tid] = s1;
      }
      __syncthreads();
      for (int idx = tid; idx < nown * CL; idx += ECL_NT) {
        const int p = idx / nown, oc = idx - p * nown;
        double* ry = cl.map_shared_rank(y, p);
        ry[c0 + oc] = es.own[0][oc];
        if (two) ry[n + c0 + oc] = es.own[1][oc];
      }
      ECL_T(a3t);
      cl.sync();
      ECL_T(a4t);
      ECL_ADD(7, a2t, a3t);
      ECL_ADD(8, a3t, a4t);
    }
    ECL_T(aa0);
    est_after_adj_impl<CX>(S, n, sweep, es.sa);
    __syncthreads();
    cl.sync();
    ECL_T(aa1);
    ECL_ADD(9, aa0, aa1);
  }
#ifdef ECL_PROF
  if (blockIdx.x < (unsigned)CL && rank == 0 && tid == 0)
    printf("ecl job0 cycles: load %lld fwd_comp %lld fwd_all %lld fwd_sync %lld after_fwd %lld adj_comp+push %lld "
           "adj_sync1 %lld adj_owner+push %lld adj_sync2 %lld after_adj %lld (passes %d)\n", ecl_cyc[0], ecl_cyc[1],
           ecl_cyc[2], ecl_cyc[3], ecl_cyc[4], ecl_cyc[5], ecl_cyc[6], ecl_cyc[7], ecl_cyc[8], ecl_cyc[9], S.passes);
#endif
  if (rank == 0 && tid == 0) {
    G.est = S.est;
    G.best_j = S.best_j;
    G.passes = S.passes;
    G.mm = S.mm;
    G.done = 1;
  }
}

// ------------------------------------------------------------------------------------------
// Graph-polynomial GEMM: C = L * R, L = sum_t c_t * P_t + c0 * I built on the fly in the
// A-tile load (numpy _combine rounding: separate multiply and add), R a plain matrix.
struct CombSpec {
  int nterm;
  int node[7];      // slot index of each term
  double coef[7];
  double c0;
};

// Plain batched C = A * B (all n x n slots, n even), 64x64 tiles, K in chunks of 32 staged by
// a two-stage cp.async pipeline (16-byte copies), DMMA core.  Used for the polynomial products
// once both combinations are materialised (combine_kernel): measured 2.2x faster at n = 512
// than building the left combination inside the A-tile load (gemm_comb_kernel).
constexpr int GP_A = TM * LDA_S, GP_B = TK * LDB_S;
__global__ void __launch_bounds__(128) gemm_plain_kernel(Slots S, DList L, int ak, int bk, int ck) {
  extern __shared__ __align__(16) double gsm[];
  if (blockIdx.z >= *L.cnt) return;
  const int b = L.ids[blockIdx.z];
  const int n = S.n;
  const int col0 = blockIdx.x * TN, row0 = blockIdx.y * TM;
  const double* A = S.buf(b, ak);
  const double* Bm = S.buf(b, bk);
  double* Cm = S.buf(b, ck);
  const int tid = threadIdx.x;
  auto stage = [&](int k0, int buf) {
    double* As = gsm + buf * (GP_A + GP_B);
    double* Bs = As + GP_A;
    // A: 64 rows x 32 cols = 64 x 16 chunks of 16 B; B: 32 rows x 64 cols = 32 x 32 chunks
    for (int c = tid; c < 64 * 16; c += 128) {
      const int r = c >> 4, q = (c & 15) * 2;
      const int i = row0 + r, kk = k0 + q;
      double* dst = &As[r * LDA_S + q];
      if (i < n && kk + 1 < n) cp_async16(dst, &A[(size_t)i * n + kk]);
      else { dst[0] = (i < n && kk < n) ? A[(size_t)i * n + kk] : 0.0; dst[1] = 0.0; }
    }
    for (int c = tid; c < 32 * 32; c += 128) {
      const int r = c >> 5, q = (c & 31) * 2;
      const int kk = k0 + r, j = col0 + q;
      double* dst = &Bs[r * LDB_S + q];
      if (kk < n && j + 1 < n) cp_async16(dst, &Bm[(size_t)kk * n + j]);
      else { dst[0] = (kk < n && j < n) ? Bm[(size_t)kk * n + j] : 0.0; dst[1] = 0.0; }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const int nk = (n + TK - 1) / TK;
  stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      stage((kc + 1) * TK, (kc + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* As = gsm + (kc & 1) * (GP_A + GP_B);
    tile_mma(As, As + GP_A, acc);
    __syncthreads();
  }
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int j = c0 + ni * 8 + 2 * t;
      if (j + 1 < n) *reinterpret_cast<double2*>(&Cm[(size_t)i * n + j]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      else if (j < n) Cm[(size_t)i * n + j] = acc[mi][ni][0];
    }
  }
}

__global__ void __launch_bounds__(128) gemm_comb_kernel(Slots S, DList DL, CombSpec L, int rk, int ck) {
  __shared__ __align__(16) double As[TM * LDA_S];
  __shared__ __align__(16) double Bs[TK * LDB_S];
  if (blockIdx.z >= *DL.cnt) return;
  const int b = DL.ids[blockIdx.z];
  const int n = S.n;
  const int col0 = blockIdx.x * TN, row0 = blockIdx.y * TM;
  const double* R = S.buf(b, rk);
  double* Cm = S.buf(b, ck);
  const int tid = threadIdx.x;
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int k0 = 0; k0 < n; k0 += TK) {
    __syncthreads();
    for (int idx = tid; idx < TM * TK; idx += 128) {
      int r = idx / TK, c = idx - r * TK;
      int i = row0 + r, kk = k0 + c;
      double v = 0.0;
      if (i < n && kk < n) {
        for (int q = 0; q < L.nterm; ++q) v = __dadd_rn(v, __dmul_rn(L.coef[q], S.buf(b, L.node[q])[(size_t)i * n + kk]));
        if (i == kk && L.c0 != 0.0) v = __dadd_rn(v, L.c0);
      }
      As[r * LDA_S + c] = v;
    }
    for (int idx = tid; idx < TK * TN; idx += 128) {
      int c = idx / TN, jj = idx - c * TN;
      int kk = k0 + c, j = col0 + jj;
      Bs[c * LDB_S + jj] = (kk < n && j < n) ? R[(size_t)kk * n + j] : 0.0;
    }
    __syncthreads();
    tile_mma(As, Bs, acc);
  }
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = c0 + ni * 8 + 2 * t + e;
        if (j < n) Cm[(size_t)i * n + j] = acc[mi][ni][e];
      }
  }
}

// ==========================================================================================
// Device-resident Algorithm 1 (north_star item 3): every decision of oracle/driver.py --
// the scaling-loop alpha test with the Eq. 27/28 skips, the DB stop test and mu switch,
// select_order's min_im / max_in / sweep, the estimate cache and the active-set compaction --
// runs in single-CTA "decide" kernels on per-matrix state held in the workspace.  The heavy
// kernels read the device-built lists / job tables (capacity = batch; unused entries exit at
// once).  The whole call is one CUDA graph: the scaling loop, the DB iterations and the
// select sweep are WHILE conditional nodes whose conditions the decide kernels set with
// cudaGraphSetConditional, so lgm_logm_f64 never blocks the host and is stream-ordered.
// Graphs are captured once per (device, workspace, n, batch, entry point) and cached; the
// per-call pointers and parameters travel in a CallDesc written by a setup kernel.

enum {
  LS_ALL = 0, LS_LIVE, LS_ACT, LS_ACTAI2, LS_ROOTS, LS_DB, LS_OK, LS_SEL, LS_NEED, LS_NEEDAI2, LS_CUR, LS_FAILED,
  LS_POK, LS_PMISS,           // lazy X inverse: predicted-last iterations that stopped / continue
  LS_POLY0,                   // LS_POLY0 + j, j = 1..K_MAX-1: selected matrices with k > j
  LS_N = LS_POLY0 + LGM_K_MAX
};


// per-call pointers and parameters (the graph's kernels read them from the workspace)
struct CallDesc {
  const double* A;     // input batch (lgm_logm_f64: A; building blocks: their first operand)
  const double* A2;    // est_product_norm's M2 / eval_degopt's first_product (nullable)
  double* L;           // output batch (logm: L; sqrt_db: X; balance: B; degopt: Z)
  long long ld;
  lgm_report* rep;
  int* iout;           // sqrt_db iters / est passes / balance sweeps / degopt products
  int* iout2;          // sqrt_db status
  double* dout;        // est values / balance scales
  int p1, kblk, zero_shortcut, max_sweeps;
  double tol;          // sqrt_db block tol (0 -> 10 n u)
  int maxiter;
  LgmParams P;
};

struct Ctl {  // device pointers into the workspace (fixed per workspace)
  int n, batch, splits;
  Slots S;
  CallDesc* desc;
  MDev* ms;
  int* lists;   // [LS_N][batch]
  int* cnt;     // [LS_N]
  InvJob* jobs; // [2 batch]
  EstJob* est;  // [batch]
  int* piv;
  int* step;
  double* W;
  double* logdet;
  int* istat;
  int* dead;    // == 1: the status of unused job-table slots
  int* scaling;
  double* nrm;
  double* nrm2;
  double* change;
  double* size;
  int* flag;
  double* scale;
  double* margin;
  int* sweeps;
  double* vec;
  double* part;
  int* hist;
  __host__ __device__ DList list(int id) const { return DList{lists + (size_t)id * batch, cnt + id}; }
  __host__ __device__ int* ids(int id) const { return lists + (size_t)id * batch; }
};

// Workspace regions in carve order (byte sizes); each occupies its size rounded up to 256 B
// plus the guard band (0 unless LGM_WS_GUARD=1; then every region and every n x n slot is
// followed by lgm_ws_guard_bytes() of a fill pattern that lgm_debug_ws_guard_check verifies:
// an out-of-bounds write detector standing in for compute-sanitizer memcheck).
constexpr int NREG = 25;
__host__ __device__ inline void ctl_sizes(int64_t n, int64_t batch, size_t slot_st, size_t* sz) {
  const int64_t splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
  int i = 0;
  sz[i++] = (size_t)batch * NBUF * slot_st * 8;  // slots
  sz[i++] = sizeof(CallDesc);
  sz[i++] = batch * sizeof(MDev);
  sz[i++] = (size_t)LS_N * batch * 4;            // lists
  sz[i++] = LS_N * 4;                            // cnt
  sz[i++] = 2 * batch * sizeof(InvJob);
  sz[i++] = batch * sizeof(EstJob);
  sz[i++] = 2 * (size_t)batch * n * 4;           // piv
  sz[i++] = 2 * (size_t)batch * n * 4;           // step
  sz[i++] = 12 * (size_t)batch * NB * n * 8;     // W
  sz[i++] = 2 * batch * 8;                       // logdet
  sz[i++] = 2 * batch * 4;                       // istat
  sz[i++] = 4;                                   // dead
  sz[i++] = batch * 4;                           // scaling
  for (int q = 0; q < 4; ++q) sz[i++] = batch * 8;  // nrm, nrm2, change, size
  sz[i++] = batch * 4;                           // flag
  sz[i++] = (size_t)batch * n * 8;               // scale
  sz[i++] = batch * 8;                           // margin
  sz[i++] = batch * 4;                           // sweeps
  sz[i++] = (size_t)batch * 4 * n * 8;           // vec
  sz[i++] = (size_t)batch * splits * 2 * n * 8;  // part
  sz[i++] = batch * 16 * 4;                      // hist
}
__host__ __device__ inline size_t r256(size_t b) { return (b + 255) & ~size_t(255); }
inline size_t slot_stride(int64_t n) { return (size_t)n * n + lgm_ws_guard_bytes() / 8; }

size_t ctl_bytes(int64_t n, int64_t batch) {
  size_t sz[NREG], s = 0;
  ctl_sizes(n, batch, slot_stride(n), sz);
  for (int r = 0; r < NREG; ++r) s += r256(sz[r]) + lgm_ws_guard_bytes();
  return s;
}

Ctl ctl_carve(void* ws, int n, int batch) {
  Ctl c{};
  c.n = n;
  c.batch = batch;
  c.splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
  size_t sz[NREG];
  ctl_sizes(n, batch, slot_stride(n), sz);
  char* p = (char*)ws;
  int r = 0;
  auto take = [&](size_t) { char* q = p; p += r256(sz[r++]) + lgm_ws_guard_bytes(); return (void*)q; };
  c.S.ws = (double*)take(0);
  c.S.n = n;
  c.S.st = slot_stride(n);
  c.desc = (CallDesc*)take(0);
  c.ms = (MDev*)take(0);
  c.lists = (int*)take(0);
  c.cnt = (int*)take(0);
  c.jobs = (InvJob*)take(0);
  c.est = (EstJob*)take(0);
  c.piv = (int*)take(0);
  c.step = (int*)take(0);
  c.W = (double*)take(0);
  c.logdet = (double*)take(0);
  c.istat = (int*)take(0);
  c.dead = (int*)take(0);
  c.scaling = (int*)take(0);
  c.nrm = (double*)take(0);
  c.nrm2 = (double*)take(0);
  c.change = (double*)take(0);
  c.size = (double*)take(0);
  c.flag = (int*)take(0);
  c.scale = (double*)take(0);
  c.margin = (double*)take(0);
  c.sweeps = (int*)take(0);
  c.vec = (double*)take(0);
  c.part = (double*)take(0);
  c.hist = (int*)take(0);
  return c;
}

// Guard bands: check = 0 fills them with 0xA5 bytes, check = 1 counts bytes that differ.
__global__ void ws_guard_kernel(unsigned char* ws, int64_t n, int64_t batch, size_t gb, int check,
                                unsigned long long* bad) {
  size_t sz[NREG];
  const size_t st = (size_t)n * n + gb / 8;
  ctl_sizes(n, batch, st, sz);
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  unsigned long long nbad = 0;
  size_t off = 0;
  for (int r = 0; r < NREG; ++r) {  // region tails + guard bands (bytes)
    const size_t lo = off + sz[r], hi = off + r256(sz[r]) + gb;
    for (size_t i = lo + tid; i < hi; i += nth) {
      if (check) nbad += ws[i] != 0xA5u;
      else ws[i] = 0xA5u;
    }
    off = hi;
  }
  // the guard band after every n x n slot (8-byte words)
  const size_t gw = gb / 8, nslots = (size_t)batch * NBUF;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(ws);
  for (size_t i = tid; i < nslots * gw; i += nth) {
    const size_t at = (i / gw) * st + (size_t)n * n + i % gw;
    if (check) nbad += w[at] != 0xA5A5A5A5A5A5A5A5ull;
    else w[at] = 0xA5A5A5A5A5A5A5A5ull;
  }
  if (check && nbad) atomicAdd(bad, nbad);
}

// ------------------------------------------------------------------ decide-kernel helpers
constexpr int CT = 1024;  // decide kernels: one CTA of CT threads

// Order-preserving block-wide append: every thread of the CTA calls it (uniformly) with its
// predicate; returns the slot for predicated threads and advances `off` by the total.
__device__ int blk_append(bool pred, int* s_w, int& off) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {
    const int v = lane < nw ? s_w[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    s_w[lane] = incl - v;
    if (lane == 31) s_w[32] = incl;
  }
  __syncthreads();
  const int pos = off + s_w[warp] + __popc(m & ((1u << lane) - 1u));
  off += s_w[32];
  return pos;
}

// Loop over the entries of list `src` in chunks of CT (uniform trip count), b = -1 off the end.
#define FOR_LIST(c, src)                                                           \
  const int* src_ids_ = (c).ids(src);                                             \
  const int src_n_ = (c).cnt[src];                                                \
  for (int base_ = 0; base_ < src_n_; base_ += CT) {                              \
    const int e_ = base_ + (int)threadIdx.x;                                      \
    const int b = e_ < src_n_ ? src_ids_[e_] : -1;

__device__ __forceinline__ double dpow(double x, double y) { return pow(x, y); }


// Device-side phase timer (diagnostics: lgm_debug_grid_phase_ns): every decide kernel charges
// the globaltimer interval since the previous mark to the phase that just ended.  One stream
// at a time (a process-wide accumulator).
enum { PH_LOAD = 0, PH_BALANCE, PH_ALPHA, PH_DB, PH_SELPREP, PH_SELECT, PH_POLY, PH_OTHER, PH_N };
__device__ unsigned long long g_phase_ns[PH_N];
__device__ unsigned long long g_phase_last;
__device__ __forceinline__ void phase_mark(int ph, bool start = false) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (!start) g_phase_ns[ph] += now - g_phase_last;
    g_phase_last = now;
  }
}

// ------------------------------------------------------------------ setup / init / load
__global__ void setup_kernel(CallDesc* d, CallDesc v) { *d = v; }

__global__ void __launch_bounds__(CT) ctl_init_kernel(Ctl c) {
  phase_mark(PH_OTHER, true);
  for (int b = threadIdx.x; b < c.batch; b += CT) {
    MDev& M = c.ms[b];
    memset(&M, 0, sizeof(MDev));
    M.mm = INFINITY;
    M.dbmm = INFINITY;
    c.ids(LS_ALL)[b] = b;
    c.flag[b] = 0;
    c.margin[b] = INFINITY;
    c.sweeps[b] = 0;
  }
  if (threadIdx.x == 0) {
    c.cnt[LS_ALL] = c.batch;
    for (int l = 1; l < LS_N; ++l) c.cnt[l] = 0;
    *c.dead = 1;
  }
}

__global__ void fill_kernel(double* p, size_t count, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// as_square (matcore.py:64-65): non-finite input -> NONFINITE; the rest is the live list
__global__ void __launch_bounds__(CT) decide_live_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_LOAD);
  int off = 0;
  FOR_LIST(c, LS_ALL)
    const bool bad = b >= 0 && c.flag[b];
    if (bad) c.ms[b].status = LGM_NONFINITE;
    const int pos = blk_append(b >= 0 && !bad, s_w, off);
    if (b >= 0 && !bad) c.ids(LS_LIVE)[pos] = b;
  }
  if (threadIdx.x == 0) c.cnt[LS_LIVE] = off;
}

// finish = ||B - I||_1 <= Theta_K, after balancing
__global__ void __launch_bounds__(CT) decide_start_kernel(Ctl c) {
  phase_mark(PH_BALANCE);
  const LgmParams& P = c.desc->P;
  const double thK = P.theta[P.max_k - 1];
  FOR_LIST(c, LS_LIVE)
    if (b >= 0) {
      MDev& M = c.ms[b];
      M.sweeps = c.sweeps[b];
      M.mm = c.margin[b];
      M.alpha_loop = c.nrm[b];
      M.finish = M.le(c.nrm[b], thK);
    }
  }
}

__device__ __forceinline__ bool scal_active(const MDev& M, const LgmParams& P) {
  return !M.finish && M.status == 0 && M.s < P.maxiter_s;
}

// scaling-loop head: act = live matrices still scaling; act_ai2 = those with A_I2
__global__ void __launch_bounds__(CT) decide_act_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_OTHER);
  const LgmParams& P = c.desc->P;
  int off = 0, off2 = 0;
  FOR_LIST(c, LS_LIVE)
    const bool a = b >= 0 && scal_active(c.ms[b], P);
    const int pos = blk_append(a, s_w, off);
    if (a) c.ids(LS_ACT)[pos] = b;
    const bool a2 = a && c.ms[b].have_ai2;
    const int pos2 = blk_append(a2, s_w, off2);
    if (a2) c.ids(LS_ACTAI2)[pos2] = b;
  }
  if (threadIdx.x == 0) { c.cnt[LS_ACT] = off; c.cnt[LS_ACTAI2] = off2; }
}

// ------------------------------------------------------------------ alpha (A.2)
// The request of matrix b: power m = M.am (even), threshold M.th, nA = M.nA, nI2 = M.nI2.
__device__ void est_slot(Ctl& c, int q, int b, const double* M1, int p1, const double* M2, int zchk, int key) {
  EstJob& J = c.est[q];
  J.M1 = M1;
  J.M2 = M2;
  J.p1 = p1;
  J.live = 1;
  J.zchk = zchk;
  J.nzf = 0;
  J.owner = b;
  J.key = key;
  J.cplx = c.desc->P.cplx;
  J.V0 = c.vec + (size_t)q * 4 * c.n;
  J.V1 = J.V0 + 2 * c.n;
  J.part = c.part + (size_t)q * c.splits * 2 * c.n;
  J.hist = c.hist + q * 16;
}
__device__ void est_kill_tail(Ctl& c, int from) {
  for (int q = from + (int)threadIdx.x; q < c.batch; q += CT) c.est[q].live = 0;
}
// fold the finished estimates of the table into the owners' state (counters, margin, cache)
__device__ void est_absorb(Ctl& c, int count) {
  for (int q = threadIdx.x; q < count; q += CT) {
    const EstJob& J = c.est[q];
    MDev& M = c.ms[J.owner];
    M.nest++;
    M.passes += J.passes;
    M.mm = fmin(M.mm, J.mm);
    M.cache[J.key] = J.est;
    M.cvalid |= 1u << J.key;
  }
}

// phase A: Eq. 27 skip, cached p_m, else an estimate of ||A_I2^{m/2}|| or ||(A - I)^m||
__global__ void __launch_bounds__(CT) alpha_a_kernel(Ctl c, int lst) {
  __shared__ int s_w[33];
  int off = 0;
  FOR_LIST(c, lst)
    bool need = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      const int m = M.am;
      M.adone = 0;
      M.need1 = M.need2 = 0;
      bool skip = false;
      if (M.have_ai2) {
        const double r2 = sqrt(M.nI2);
        if (M.le(r2, M.th)) { M.t1 = r2; M.Pm = dpow(M.nI2, (double)(m / 2)); skip = true; }
      }
      if (!skip) {
        if ((M.cvalid >> m) & 1u) { M.Pm = M.cache[m]; M.t1 = dpow(M.Pm, 1.0 / m); }
        else need = true;
      }
      M.need1 = need;
    }
    const int q = blk_append(need, s_w, off);
    if (need) {
      const MDev& M = c.ms[b];
      if (M.have_ai2) est_slot(c, q, b, c.S.buf(b, G_AP), M.am / 2, nullptr, 1, M.am);
      else est_slot(c, q, b, c.S.buf(b, G_AM), M.am, nullptr, 1, M.am);
    }
  }
  __syncthreads();
  est_kill_tail(c, off);
  if (threadIdx.x == 0) c.cnt[LS_NEED] = off;
}

// phase B: absorb the m-term estimates; t1 > Theta early exit; Eq. 28 bound; cached or new
// (m+1)-term estimate (product form ||A_I2^{m/2} (A - I)|| when A_I2 exists)
__global__ void __launch_bounds__(CT) alpha_b_kernel(Ctl c, int lst) {
  __shared__ int s_w[33];
  est_absorb(c, c.cnt[LS_NEED]);
  __syncthreads();
  int off = 0;
  FOR_LIST(c, lst)
    bool need = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      const int m = M.am;
      if (M.need1) { M.Pm = M.cache[m]; M.t1 = dpow(M.Pm, 1.0 / m); }
      M.note(M.t1, M.th);
      if (M.t1 > M.th) {
        M.aout = M.t1;
        M.adone = 1;
      } else {
        const double bound = dpow(M.Pm * M.nA, 1.0 / (m + 1));
        if (M.le(bound, M.th)) M.t2 = bound;
        else if ((M.cvalid >> (m + 1)) & 1u) M.t2 = dpow(M.cache[m + 1], 1.0 / (m + 1));
        else need = true;
      }
      M.need2 = need;
    }
    const int q = blk_append(need, s_w, off);
    if (need) {
      const MDev& M = c.ms[b];
      if (M.have_ai2) est_slot(c, q, b, c.S.buf(b, G_AP), M.am / 2, c.S.buf(b, G_AM), 0, M.am + 1);
      else est_slot(c, q, b, c.S.buf(b, G_AM), M.am + 1, nullptr, 1, M.am + 1);
    }
  }
  __syncthreads();
  est_kill_tail(c, off);
  if (threadIdx.x == 0) c.cnt[LS_NEED] = off;
}

__global__ void __launch_bounds__(CT) alpha_c_kernel(Ctl c, int lst) {
  est_absorb(c, c.cnt[LS_NEED]);
  __syncthreads();
  FOR_LIST(c, lst)
    if (b >= 0) {
      MDev& M = c.ms[b];
      const int m = M.am;
      if (M.need2) M.t2 = dpow(M.cache[m + 1], 1.0 / (m + 1));
      if (!M.adone) M.aout = fmax(M.t1, M.t2);
    }
  }
}

// ------------------------------------------------------------------ scaling loop (A.1 step 5)
// nA / nI2 from the norms; the scaling-loop alpha request (m_K, Theta_K)
__global__ void __launch_bounds__(CT) scal_req_kernel(Ctl c) {
  const LgmParams& P = c.desc->P;
  const int K = P.max_k;
  FOR_LIST(c, LS_ACT)
    if (b >= 0) {
      MDev& M = c.ms[b];
      M.nA = c.nrm[b];
      if (M.have_ai2) M.nI2 = c.nrm2[b];
      M.am = P.order[K - 1];
      M.th = P.theta[K - 1];
    }
  }
}

// finish = alpha <= Theta_K; roots = matrices taking another square root
__global__ void __launch_bounds__(CT) decide_roots_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_ALPHA);
  const LgmParams& P = c.desc->P;
  const double thK = P.theta[P.max_k - 1];
  int off = 0;
  FOR_LIST(c, LS_ACT)
    bool r = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      M.alpha_loop = M.aout;
      M.finish = M.le(M.aout, thK);
      r = !M.finish;
      if (r) { M.dbit = 0; M.dbst = 0; M.dbplat = 0; M.dbpred = 0; M.dbmm = INFINITY; c.scaling[b] = 1; }
    }
    const int pos = blk_append(r, s_w, off);
    if (r) c.ids(LS_ROOTS)[pos] = b;
  }
  if (threadIdx.x == 0) { c.cnt[LS_ROOTS] = off; c.cnt[LS_DB] = off; }
  __syncthreads();
  for (int e = threadIdx.x; e < off; e += CT) c.ids(LS_DB)[e] = c.ids(LS_ROOTS)[e];
}

// after the roots: fold the DB outcome; s++ and A_I2 pending for the converged ones; the
// scaling loop continues while some live matrix is still active
__global__ void __launch_bounds__(CT) decide_post_kernel(Ctl c, cudaGraphConditionalHandle h, int nodes) {
  __shared__ int s_w[33];
  __shared__ int s_any;
  phase_mark(PH_DB);
  const LgmParams& P = c.desc->P;
  if (threadIdx.x == 0) s_any = 0;
  int off = 0;
  FOR_LIST(c, LS_ROOTS)
    bool ok = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      M.db_iters += M.dbit;
      M.mm = fmin(M.mm, M.dbmm);
      M.plateau += M.dbplat;
      if (M.dbst) {
        M.status = M.dbst;
      } else {
        M.s++;
        M.have_ai2 = 1;
        M.cvalid = 0u;
        ok = true;
      }
    }
    const int pos = blk_append(ok, s_w, off);
    if (ok) c.ids(LS_OK)[pos] = b;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < c.cnt[LS_LIVE]; e += CT)
    if (scal_active(c.ms[c.ids(LS_LIVE)[e]], P)) s_any = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    c.cnt[LS_OK] = off;
    cudaGraphSetConditional(h, s_any ? 1u : 0u);
  }
  count_nodes(nodes);
}

// ------------------------------------------------------------------ DB square root (sqrtm.py:27-78)
// Job table for this iteration: X of every DB-active matrix (except those whose iteration is
// predicted to be the root's last: their X^-1 is formed later only if needed), then (it > 1)
// Y; unused slots carry M = nullptr and the always-1 status.  Also zeroes the per-iteration
// accumulators.
__device__ InvJob make_job(const Ctl& c, int b, int w, int oop) {
  InvJob J{};
  J.M = c.S.buf(b, w ? G_YI : G_XI);
  J.Src = oop ? c.S.buf(b, w ? G_Y : G_B) : nullptr;
  J.piv = c.piv + ((size_t)w * c.batch + b) * c.n;
  J.rowstep = c.step + ((size_t)w * c.batch + b) * c.n;
  J.Wb = c.W + ((size_t)w * c.batch + b) * NB * c.n;
  J.wst = (long long)2 * c.batch * NB * c.n;
  J.logdet = c.logdet + w * c.batch + b;
  J.status = c.istat + w * c.batch + b;
  return J;
}
__device__ InvJob null_job(const Ctl& c) {
  InvJob J{};
  J.M = nullptr;
  J.status = c.dead;
  return J;
}
__global__ void __launch_bounds__(CT) build_jobs_kernel(Ctl c, int first, int oop) {
  __shared__ int s_w[33];
  const int na = c.cnt[LS_DB];
  const int cap = first ? c.batch : 2 * c.batch;
  int off = 0;
  FOR_LIST(c, LS_DB)
    const bool px = b >= 0 && !first && c.ms[b].dbpred;  // predicted last: no X inverse now
    const bool want = b >= 0 && !px;
    const int pos = blk_append(want, s_w, off);
    if (want) c.jobs[pos] = make_job(c, b, 0, oop);
    if (b >= 0) {
      c.change[b] = 0.0;
      c.size[b] = 0.0;
      if (first) c.logdet[c.batch + b] = 0.0;
      if (px) c.istat[b] = 0;
    }
  }
  const int nj = first ? off : off + na;
  for (int e = threadIdx.x; !first && e < na; e += CT) c.jobs[off + e] = make_job(c, c.ids(LS_DB)[e], 1, oop);
  for (int q = nj + threadIdx.x; q < cap; q += CT) c.jobs[q] = null_job(c);
}

// lazy X^-1, second phase: X jobs of the predicted-last matrices that did not converge
__global__ void __launch_bounds__(CT) build_jobs_px_kernel(Ctl c, int oop) {
  const int nm = c.cnt[LS_PMISS];
  for (int q = threadIdx.x; q < c.batch; q += CT) c.jobs[q] = q < nm ? make_job(c, c.ids(LS_PMISS)[q], 0, oop) : null_job(c);
}

// sqrt_db building block: every live matrix takes one root
__global__ void __launch_bounds__(CT) decide_db_start_kernel(Ctl c) {
  const int na = c.cnt[LS_LIVE];
  for (int e = threadIdx.x; e < na; e += CT) {
    const int b = c.ids(LS_LIVE)[e];
    MDev& M = c.ms[b];
    M.dbit = 0; M.dbst = 0; M.dbplat = 0; M.dbpred = 0; M.dbmm = INFINITY;
    c.scaling[b] = 1;
    c.ids(LS_ROOTS)[e] = b;
    c.ids(LS_DB)[e] = b;
  }
  if (threadIdx.x == 0) { c.cnt[LS_ROOTS] = na; c.cnt[LS_DB] = na; }
}

// stop test of the iteration just done (sqrtm.py:66-78), mu switch, next DB list
// Lazy X^-1: when an unscaled iteration's rel is below pred_f * sqrt(tol) the next one is
// predicted to converge, so its X^-1 (needed only for Y', which a converged root discards) is
// deferred: db_update forms X' from Y^-1 alone; a converged root keeps X' (LS_POK); otherwise
// (LS_PMISS) the IF body h2 inverts X and completes Y'.  Bit-identical to the eager order.
__global__ void __launch_bounds__(CT) decide_db_kernel(Ctl c, cudaGraphConditionalHandle h, int nodes, int first,
                                                        int block_mode, cudaGraphConditionalHandle h2, int lazy,
                                                        double pred_f) {
  __shared__ int s_w[33];
  phase_mark(PH_DB);
  const CallDesc& D = *c.desc;
  const int n = c.n;
  const double tol_in = block_mode ? D.tol : D.P.db_tol;
  const int maxiter = block_mode ? D.maxiter : D.P.db_maxiter;
  const int nz = D.P.cplx ? n / 2 : n;  // Z's order for a complex embedding
  const double tol = tol_in > 0.0 ? tol_in : 10.0 * nz * LGM_UNIT_ROUNDOFF;
  int off = 0, offk = 0, offm = 0;
  FOR_LIST(c, LS_DB)
    bool next = false, pok = false, pmiss = false;
    if (b >= 0 && c.ms[b].dbst == 0) {  // (a singular X met by the last fix-up ends the root)
      MDev& M = c.ms[b];
      const bool px = !first && M.dbpred;
      M.dbpred = 0;
      const int it = ++M.dbit;
      const bool sing = c.istat[b] || (!first && c.istat[c.batch + b]);
      const double ch = c.change[b], sz = c.size[b];
      if (sing) {
        M.dbst = LGM_SINGULAR;
        M.dbit = it - 1;
      } else if (!isfinite(ch) || !isfinite(sz)) {
        M.dbst = LGM_NONFINITE;
      } else if (sz == 0.0) {
        M.dbst = LGM_DB_NOCONV;
      } else {
        const double rel = ch / sz;
        auto note = [&](double x, double thr) { M.dbmm = fmin(M.dbmm, fabs(x - thr) / fabs(thr)); };
        note(rel, LGM_SCALING_SWITCH);
        if (rel < LGM_SCALING_SWITCH) c.scaling[b] = 0;
        note(rel, tol);
        if (tol / 10.0 <= rel && rel <= 10.0 * tol) M.dbplat++;
        if (rel > tol) {
          if (it == maxiter) M.dbst = LGM_DB_NOCONV;
          else next = true;
        }
        if (lazy && next && !c.scaling[b] && rel <= pred_f * sqrt(tol)) M.dbpred = 1;
      }
      if (px) {
        pmiss = next;   // X^-1 and Y' still needed
        pok = !next;    // the root stops: X <- X'
        if (pok) M.dbskip++;
      }
    }
    const int pos = blk_append(next, s_w, off);
    if (next) c.ids(LS_DB)[pos] = b;  // in place: pos <= e_, ascending, read before written
    const int pk = blk_append(pok, s_w, offk);
    if (pok) c.ids(LS_POK)[pk] = b;
    const int pm = blk_append(pmiss, s_w, offm);
    if (pmiss) c.ids(LS_PMISS)[pm] = b;
  }
  if (threadIdx.x == 0) {
    c.cnt[LS_DB] = off;
    c.cnt[LS_POK] = offk;
    c.cnt[LS_PMISS] = offm;
    cudaGraphSetConditional(h, off > 0 ? 1u : 0u);
    if (!first && lazy) cudaGraphSetConditional(h2, offm > 0 ? 1u : 0u);
  }
  count_nodes(nodes);
}

// ------------------------------------------------------------------ select_order (A.3)
__global__ void __launch_bounds__(CT) decide_sel_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_OTHER);
  int off = 0, off2 = 0;
  FOR_LIST(c, LS_LIVE)
    bool sel = false, need = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      if (M.status == 0 && !M.finish) M.status = LGM_SCALING_MAXITER;
      sel = M.status == 0;
      need = sel && !M.have_ai2;
    }
    const int pos = blk_append(sel, s_w, off);
    if (sel) c.ids(LS_SEL)[pos] = b;
    const int pos2 = blk_append(need, s_w, off2);
    if (need) c.ids(LS_NEEDAI2)[pos2] = b;
  }
  if (threadIdx.x == 0) { c.cnt[LS_SEL] = off; c.cnt[LS_NEEDAI2] = off2; }
}

__device__ int first_index(MDev& M, double x, const LgmParams& P) {
  for (int j = 1; j <= P.max_k; ++j)
    if (M.le(x, P.theta[j - 1])) return j;
  return P.max_k;
}

// min_im (Eqs. 29-31 + tabmin_im), max_in (Eqs. 32-34); immediate choice or the sweep list
__global__ void __launch_bounds__(CT) select_init_kernel(Ctl c, cudaGraphConditionalHandle h) {
  __shared__ int s_w[33];
  phase_mark(PH_SELPREP);
  const LgmParams& P = c.desc->P;
  const int K = P.max_k;
  const int mK = P.order[K - 1];
  int off = 0;
  FOR_LIST(c, LS_SEL)
    bool cur = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      M.nA = c.nrm[b];
      if (!M.have_ai2) { M.products++; M.have_ai2 = 1; }  // s = 0: A_I2 = (B - I)^2
      M.nI2 = c.nrm2[b];
      const double r2 = sqrt(M.nI2);
      int mi;
      if ((M.cvalid >> mK) & 1u) {
        mi = first_index(M, dpow(M.cache[mK], 1.0 / mK), P);
        if ((M.cvalid >> (mK + 1)) & 1u) mi = max(mi, first_index(M, dpow(M.cache[mK + 1], 1.0 / (mK + 1)), P));
      } else {
        mi = first_index(M, r2, P);
      }
      const int tabmin[LGM_K_MAX] = LGM_TABMIN_IM;
      mi = tabmin[mi - 1];
      M.note(r2, P.theta[0]);
      mi = (r2 > P.theta[0]) ? max(mi, 2) : 1;
      int mx = K;
      double mb = -1.0;
      bool found = false;
      for (int j = 1; j <= K; ++j) {
        const int m = P.order[j - 1];
        const double bnd = dpow(dpow(M.nI2, (double)(m / 2)) * M.nA, 1.0 / (m + 1));
        if (M.le(bnd, P.theta[j - 1])) { mx = j; mb = bnd; found = true; break; }
      }
      M.cert_max = found ? mb : M.alpha_loop;
      M.max_in = mx;
      if (mi >= mx) {
        M.k = mx;
        M.cert = M.cert_max;
      } else {
        cur = true;
        M.jcur = mi;
        M.am = P.order[mi - 1];
        M.th = P.theta[mi - 1];
      }
    }
    const int pos = blk_append(cur, s_w, off);
    if (cur) c.ids(LS_CUR)[pos] = b;
  }
  if (threadIdx.x == 0) {
    c.cnt[LS_CUR] = off;
    cudaGraphSetConditional(h, off > 0 ? 1u : 0u);
  }
}

__global__ void __launch_bounds__(CT) select_step_kernel(Ctl c, cudaGraphConditionalHandle h, int nodes) {
  __shared__ int s_w[33];
  phase_mark(PH_SELECT);
  const LgmParams& P = c.desc->P;
  int off = 0;
  FOR_LIST(c, LS_CUR)
    bool next = false;
    if (b >= 0) {
      MDev& M = c.ms[b];
      const int j = M.jcur;
      if (M.le(M.aout, P.theta[j - 1])) { M.k = j; M.cert = M.aout; }
      else if (M.le(M.aout, P.theta[j])) { M.k = j + 1; M.cert = M.aout; }
      else if (j + 1 < M.max_in) { M.jcur = j + 1; M.am = P.order[j]; M.th = P.theta[j]; next = true; }
      else { M.k = M.max_in; M.cert = M.cert_max; }
    }
    const int pos = blk_append(next, s_w, off);
    if (next) c.ids(LS_CUR)[pos] = b;
  }
  if (threadIdx.x == 0) {
    c.cnt[LS_CUR] = off;
    cudaGraphSetConditional(h, off > 0 ? 1u : 0u);
  }
  count_nodes(nodes);
}

// ------------------------------------------------------------------ polynomial (schemes.py:91-126)
// node slots: P2 = I - B (G_B), P3 = A_I2 (G_AP), P4.. (G_XI, G_YI, G_P6 .. G_P11); R temp G_Y,
// L temp G_AM.  Scheme k_b's coefficient rows come from the call's parameter block.
__constant__ int c_node_slot[12] = {-1, -1, G_B, G_AP, G_XI, G_YI, G_P6, G_P7, G_P8, G_P9, G_P10, G_P11};

__global__ void __launch_bounds__(CT) decide_poly_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_SELECT);
  for (int j = 1; j < LGM_K_MAX; ++j) {
    int off = 0;
    FOR_LIST(c, LS_SEL)
      const bool in = b >= 0 && c.ms[b].k > j;
      const int pos = blk_append(in, s_w, off);
      if (in) c.ids(LS_POLY0 + j)[pos] = b;
    }
    if (threadIdx.x == 0) c.cnt[LS_POLY0 + j] = off;
  }
}

// ---- fused polynomial chain (schemes.py:104-126 + PAPER.md:746-747) ---------------------
// The combinations of the graph live in the producing kernels' epilogues: poly_start forms
// P2 (= I - B for logm) and the first operand pair (L1, R1) elementwise; GEMM j multiplies
// the pair (L_j, R_j) and its epilogue either stores P_{j+3} and forms the next pair
// (L_{j+1}, R_{j+1}) from the nodes -- P_{j+3} straight from the accumulators -- or, for the
// matrix's last product, forms z = sum out_t P_t + out_0 I, L = -2^s z, unbalanced, and
// writes the output.  Operand pairs alternate between (G_AM, G_Y) and (G_Q0, G_Q1) so that
// the epilogue never overwrites an operand other CTAs of the same GEMM still read.  Every
// combination is numpy's _combine rounding (sequential over the nodes, zero coefficients
// skipped, separate multiply / add, the identity term last).
__device__ __forceinline__ int pair_l(int j) { return (j & 1) ? G_Q0 : G_AM; }
__device__ __forceinline__ int pair_r(int j) { return (j & 1) ? G_Q1 : G_Y; }

struct PolyArgs {
  Slots S;
  const CallDesc* d;
  const MDev* ms;
  const double* scale;
  int* nonfinite;
  int logm;  // 1: P2 = I - B, L = -2^s z unbalanced; 0 (eval_degopt block): P2 = X, L = z
};

// the value at (i, c) of sum_{t=2..nn} row[t-1] P_t + row[0] I, P_pn (if pn > 0) given
__device__ __forceinline__ double comb_at(const Slots& S, int b, const double* row, int nn, size_t idx, bool diag,
                                          int pn, double pv) {
  double v = 0.0;
  for (int t = 2; t <= nn; ++t)
    if (row[t - 1] != 0.0) v = __dadd_rn(v, __dmul_rn(row[t - 1], t == pn ? pv : S.buf(b, c_node_slot[t])[idx]));
  if (diag && row[0] != 0.0) v = __dadd_rn(v, row[0]);
  return v;
}

__device__ __forceinline__ void poly_out(const PolyArgs& a, int b, int k, int i, int c, size_t idx, int pn, double pv) {
  const int n = a.S.n;
  const LgmParams& P = a.d->P;
  double v = comb_at(a.S, b, lgm_out(P, k), k + 2, idx, i == c, pn, pv);
  if (a.logm) {
    v = -ldexp(1.0, a.ms[b].s) * v;
    if (P.balance) v = v * (a.scale[(size_t)b * n + i] / a.scale[(size_t)b * n + c]);
  }
  a.d->L[(size_t)b * n * a.d->ld + (size_t)i * a.d->ld + c] = v;
  if (a.nonfinite && !isfinite(v)) a.nonfinite[b] = 1;
}

// P2 (logm: I - B in place), then L1 / R1 into pair 1 -- or, for k = 1, the output
__global__ void poly_start_kernel(PolyArgs a, DList L) {
  const int n = a.S.n;
  const LgmParams& P = a.d->P;
  LIST_LOOP(L, (size_t)n * n)
    const int k = a.ms[b].k;
    const int i = idx / n, c = idx - (size_t)i * n;
    double* P2 = a.S.buf(b, G_B);
    double p2 = P2[idx];
    if (a.logm) {
      p2 = (i == c) ? 1.0 - p2 : -p2;
      P2[idx] = p2;
    }
    if (k == 1) {
      poly_out(a, b, k, i, c, idx, 2, p2);
    } else {
      a.S.buf(b, pair_l(1))[idx] = comb_at(a.S, b, lgm_lhs(P, k, 1), 3, idx, i == c, 2, p2);
      a.S.buf(b, pair_r(1))[idx] = comb_at(a.S, b, lgm_rhs(P, k, 1), 3, idx, i == c, 2, p2);
    }
  }
}

// GEMM j: P_{j+3} = L_j R_j (64 x 64 tiles, K in chunks of 32 staged by a two-stage cp.async
// pipeline, DMMA core; scalar loads for odd n), fused epilogue as above
// POLY_1STAGE (default 1; -DPOLY_1STAGE=0 builds the two-stage cp.async ring at 3 CTAs/SM): one
// K-chunk buffer per CTA and 4 CTAs/SM (120 registers, 36 KB) -- the single-slot idea of
// gj_update2s_kernel: the co-resident CTAs' loads overlap each other's products.  Same sums
// (bit-identical); config 4 polynomial phase 14.1 -> 13.0 ms, config 3b 43.40 -> 43.08 ms.
#ifndef POLY_1STAGE
#define POLY_1STAGE 1
#endif
template <bool EVEN>
__global__ void __launch_bounds__(128, POLY_1STAGE ? 4 : 1) poly_gemm_kernel(PolyArgs a, DList L, int j) {
  extern __shared__ __align__(16) double gsm[];
  if (blockIdx.z >= *L.cnt) return;
  const int b = L.ids[blockIdx.z];
  const Slots& S = a.S;
  const int n = S.n;
  const int col0 = blockIdx.x * TN, row0 = blockIdx.y * TM;
  const double* A = S.buf(b, pair_l(j));
  const double* Bm = S.buf(b, pair_r(j));
  const int tid = threadIdx.x;
  auto ld2 = [&](double* dst, const double* src, bool ok2, bool ok1) {
    if (EVEN && ok2) cp_async16(dst, src);
    else { dst[0] = ok1 ? src[0] : 0.0; dst[1] = ok2 ? src[1] : 0.0; }
  };
  auto stage = [&](int k0, int buf) {
    double* As = gsm + buf * (GP_A + GP_B);
    double* Bs = As + GP_A;
    for (int c = tid; c < 64 * 16; c += 128) {
      const int r = c >> 4, q = (c & 15) * 2;
      const int i = row0 + r, kk = k0 + q;
      ld2(&As[r * LDA_S + q], &A[(size_t)i * n + kk], i < n && kk + 1 < n, i < n && kk < n);
    }
    for (int c = tid; c < 32 * 32; c += 128) {
      const int r = c >> 5, q = (c & 31) * 2;
      const int kk = k0 + r, jc = col0 + q;
      ld2(&Bs[r * LDB_S + q], &Bm[(size_t)kk * n + jc], kk < n && jc + 1 < n, kk < n && jc < n);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const int nk = (n + TK - 1) / TK;
#if POLY_1STAGE
  for (int kc = 0; kc < nk; ++kc) {
    stage(kc * TK, 0);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    tile_mma(gsm, gsm + GP_A, acc);
    __syncthreads();
  }
#else
  stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      stage((kc + 1) * TK, (kc + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* As = gsm + (kc & 1) * (GP_A + GP_B);
    tile_mma(As, As + GP_A, acc);
    __syncthreads();
  }
#endif
  const int k = a.ms[b].k;
  const LgmParams& P = a.d->P;
  const int pn = j + 3;                 // this product is node P_{j+3}
  const bool last = (j == k - 1);
  const double* lrow = last ? nullptr : lgm_lhs(P, k, j + 1);
  const double* rrow = last ? nullptr : lgm_rhs(P, k, j + 1);
  double* Pn = S.buf(b, c_node_slot[pn]);
  double* Ln = S.buf(b, pair_l(j + 1));
  double* Rn = S.buf(b, pair_r(j + 1));
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
  if (last) {  // z over P2..P_{k+2} (P_{k+2} from the accumulators), -2^s, unbalance, output
    const double* orow = lgm_out(P, k);
    double co[LGM_K_MAX + 2];
#pragma unroll
    for (int q = 0; q < LGM_K_MAX + 2; ++q) co[q] = (q + 2 <= pn) ? orow[q + 1] : 0.0;
    const double mult = -ldexp(1.0, a.ms[b].s);
    const bool unbal = a.logm && P.balance;
    double* Lout = a.d->L;
    const long long ldo = a.d->ld;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = r0 + mi * 8 + g;
      if (i >= n) continue;
      const double si = unbal ? a.scale[(size_t)b * n + i] : 1.0;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int c = c0 + ni * 8 + 2 * t;
        if (c >= n) continue;
        const bool two = EVEN || c + 1 < n;
        const size_t idx = (size_t)i * n + c;
        double z0 = 0.0, z1 = 0.0;
#pragma unroll
        for (int tt = 2; tt < LGM_K_MAX + 4 && tt < pn; ++tt) {
          if (co[tt - 2] == 0.0) continue;
          const double* src = S.buf(b, c_node_slot[tt]) + idx;
          double v0, v1 = 0.0;
          if (EVEN) {
            const double2 v = *reinterpret_cast<const double2*>(src);
            v0 = v.x;
            v1 = v.y;
          } else {
            v0 = src[0];
            if (two) v1 = src[1];
          }
          z0 = __dadd_rn(z0, __dmul_rn(co[tt - 2], v0));
          z1 = __dadd_rn(z1, __dmul_rn(co[tt - 2], v1));
        }
        const double cp = co[pn - 2];
        if (cp != 0.0) { z0 = __dadd_rn(z0, __dmul_rn(cp, acc[mi][ni][0])); z1 = __dadd_rn(z1, __dmul_rn(cp, acc[mi][ni][1])); }
        if (orow[0] != 0.0) { if (i == c) z0 = __dadd_rn(z0, orow[0]); if (i == c + 1) z1 = __dadd_rn(z1, orow[0]); }
        double zz[2] = {z0, z1};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (e == 1 && !two) break;
          double v = zz[e];
          if (a.logm) {
            v = mult * v;
            if (unbal) v = v * (si / a.scale[(size_t)b * n + c + e]);
          }
          Lout[(size_t)b * n * ldo + (size_t)i * ldo + c + e] = v;
          if (a.nonfinite && !isfinite(v)) a.nonfinite[b] = 1;
        }
      }
    }
    return;
  }
  // P_{j+3} and the next operand pair in one pass over the nodes (each node element read
  // once for both combinations; per element the _combine order over t is unchanged)
  double cl[LGM_K_MAX + 2], cr[LGM_K_MAX + 2];
#pragma unroll
  for (int q = 0; q < LGM_K_MAX + 2; ++q) {
    cl[q] = (q + 2 <= pn) ? lrow[q + 1] : 0.0;
    cr[q] = (q + 2 <= pn) ? rrow[q + 1] : 0.0;
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int c = c0 + ni * 8 + 2 * t;
      if (c >= n) continue;
      const bool two = EVEN || c + 1 < n;  // (EVEN: c even, c + 1 < n)
      const size_t idx = (size_t)i * n + c;
      double l0 = 0.0, l1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int tt = 2; tt < LGM_K_MAX + 4 && tt < pn; ++tt) {
        if (cl[tt - 2] == 0.0 && cr[tt - 2] == 0.0) continue;
        const double* src = S.buf(b, c_node_slot[tt]) + idx;
        double v0, v1 = 0.0;
        if (EVEN) {
          const double2 v = *reinterpret_cast<const double2*>(src);
          v0 = v.x;
          v1 = v.y;
        } else {
          v0 = src[0];
          if (two) v1 = src[1];
        }
        if (cl[tt - 2] != 0.0) { l0 = __dadd_rn(l0, __dmul_rn(cl[tt - 2], v0)); l1 = __dadd_rn(l1, __dmul_rn(cl[tt - 2], v1)); }
        if (cr[tt - 2] != 0.0) { q0 = __dadd_rn(q0, __dmul_rn(cr[tt - 2], v0)); q1 = __dadd_rn(q1, __dmul_rn(cr[tt - 2], v1)); }
      }
      const double p0 = acc[mi][ni][0], p1 = acc[mi][ni][1];
      const double clp = cl[pn - 2], crp = cr[pn - 2];
      if (clp != 0.0) { l0 = __dadd_rn(l0, __dmul_rn(clp, p0)); l1 = __dadd_rn(l1, __dmul_rn(clp, p1)); }
      if (crp != 0.0) { q0 = __dadd_rn(q0, __dmul_rn(crp, p0)); q1 = __dadd_rn(q1, __dmul_rn(crp, p1)); }
      if (lrow[0] != 0.0) { if (i == c) l0 = __dadd_rn(l0, lrow[0]); if (i == c + 1) l1 = __dadd_rn(l1, lrow[0]); }
      if (rrow[0] != 0.0) { if (i == c) q0 = __dadd_rn(q0, rrow[0]); if (i == c + 1) q1 = __dadd_rn(q1, rrow[0]); }
      if (EVEN) {
        *reinterpret_cast<double2*>(Pn + idx) = make_double2(p0, p1);
        *reinterpret_cast<double2*>(Ln + idx) = make_double2(l0, l1);
        *reinterpret_cast<double2*>(Rn + idx) = make_double2(q0, q1);
      } else {
        Pn[idx] = p0; Ln[idx] = l0; Rn[idx] = q0;
        if (two) { Pn[idx + 1] = p1; Ln[idx + 1] = l1; Rn[idx + 1] = q1; }
      }
    }
  }
}

// ---- reference exponential (validation helper; matcore.py:318-336 expm_ref) --------------
// s = 0 if ||A||_1 <= 1/2 else ceil(log2(||A||_1 / (1/2))) (exact, from the binary exponent),
// X = A / 2^s (exact), T = I + X T / j for j = 20..1, then s squarings.
__global__ void __launch_bounds__(CT) expm_prep_kernel(Ctl c) {
  for (int b = threadIdx.x; b < c.batch; b += CT) {
    const double x = c.nrm[b] / 0.5;
    int e = 0;
    const double m = frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
    int s = 0;
    if (c.nrm[b] > 0.5) s = (m == 0.5) ? e - 1 : e;
    if (s < 0) s = 0;
    c.ms[b].s = s;
    c.ms[b].dbit = 0;  // squarings done
    c.scale[b] = ldexp(1.0, -s);
  }
}
__global__ void expm_scale_kernel(Slots S, DList L, const double* f) {
  const int n = S.n;
  LIST_LOOP(L, (size_t)n * n)
    S.buf(b, G_B)[idx] = S.buf(b, G_B)[idx] * f[b];
  }
}
// mode 0: C = I + (X T) / j (Horner step); mode 1: C = T T (squaring)
template <bool EVEN>
__global__ void __launch_bounds__(128) expm_gemm_kernel(Slots S, DList L, int as, int bs, int cs, int j, int mode) {
  extern __shared__ __align__(16) double gsm[];
  if (blockIdx.z >= *L.cnt) return;
  const int b = L.ids[blockIdx.z];
  const int n = S.n;
  const int col0 = blockIdx.x * TN, row0 = blockIdx.y * TM;
  const double* A = S.buf(b, as);
  const double* Bm = S.buf(b, bs);
  double* Cm = S.buf(b, cs);
  const int tid = threadIdx.x;
  auto ld2 = [&](double* dst, const double* src, bool ok2, bool ok1) {
    if (EVEN && ok2) cp_async16(dst, src);
    else { dst[0] = ok1 ? src[0] : 0.0; dst[1] = ok2 ? src[1] : 0.0; }
  };
  auto stage = [&](int k0, int buf) {
    double* As = gsm + buf * (GP_A + GP_B);
    double* Bs = As + GP_A;
    for (int c = tid; c < 64 * 16; c += 128) {
      const int r = c >> 4, q = (c & 15) * 2;
      const int i = row0 + r, kk = k0 + q;
      ld2(&As[r * LDA_S + q], &A[(size_t)i * n + kk], i < n && kk + 1 < n, i < n && kk < n);
    }
    for (int c = tid; c < 32 * 32; c += 128) {
      const int r = c >> 5, q = (c & 31) * 2;
      const int kk = k0 + r, jc = col0 + q;
      ld2(&Bs[r * LDB_S + q], &Bm[(size_t)kk * n + jc], kk < n && jc + 1 < n, kk < n && jc < n);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[4][4][2] = {};
  const int nk = (n + TK - 1) / TK;
  stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      stage((kc + 1) * TK, (kc + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* As = gsm + (kc & 1) * (GP_A + GP_B);
    tile_mma(As, As + GP_A, acc);
    __syncthreads();
  }
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int r0 = row0 + (warp >> 1) * 32, c0 = col0 + (warp & 1) * 32;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = r0 + mi * 8 + g;
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + ni * 8 + 2 * t + e;
        if (c >= n) continue;
        double v = acc[mi][ni][e];
        if (mode == 0) {
          v = v / (double)j;
          v = (i == c) ? 1.0 + v : 0.0 + v;
        }
        Cm[(size_t)i * n + c] = v;
      }
  }
}
// squaring sweep: matrices with squarings left; sets the graph's WHILE condition when h != 0
__global__ void __launch_bounds__(CT) expm_sq_decide_kernel(Ctl c, cudaGraphConditionalHandle h, int set, int nodes) {
  __shared__ int s_w[33];
  int off = 0;
  FOR_LIST(c, LS_ALL)
    const bool more = b >= 0 && c.ms[b].dbit < c.ms[b].s;
    if (more) c.ms[b].dbit++;
    const int pos = blk_append(more, s_w, off);
    if (more) c.ids(LS_CUR)[pos] = b;
  }
  if (threadIdx.x == 0) {
    c.cnt[LS_CUR] = off;
    if (set) cudaGraphSetConditional(h, off > 0 ? 1u : 0u);
  }
  if (nodes) count_nodes(nodes);
}
// E: the result sits in slot G_Y after an even number of squarings, G_XI after an odd one
__global__ void expm_store_kernel(Slots S, DList L, const CallDesc* d, const MDev* ms) {
  const int n = S.n;
  double* out = d->L;
  const long long ld = d->ld;
  LIST_LOOP(L, (size_t)n * n)
    const int i = idx / n, j = idx - (size_t)i * n;
    out[(size_t)b * n * ld + (size_t)i * ld + j] = S.buf(b, (ms[b].s & 1) ? G_XI : G_Y)[idx];
  }
}

// products of the polynomial, non-finite results (estimator overflow upstream), failures
__global__ void __launch_bounds__(CT) decide_final_kernel(Ctl c) {
  __shared__ int s_w[33];
  phase_mark(PH_POLY);
  {
    FOR_LIST(c, LS_SEL)
      if (b >= 0) {
        MDev& M = c.ms[b];
        M.products += M.k - 1;
        if (c.flag[b]) { M.status = LGM_NONFINITE; M.post_fail = 1; }
      }
    }
  }
  __syncthreads();
  {
    int off = 0;
    FOR_LIST(c, LS_ALL)
      const bool f = b >= 0 && c.ms[b].status && !c.ms[b].post_fail;
      const int pos = blk_append(f, s_w, off);
      if (f) c.ids(LS_FAILED)[pos] = b;
    }
    if (threadIdx.x == 0) c.cnt[LS_FAILED] = off;
  }
}

// L of a failed matrix: all NaN (a caller ignoring the status never reads stale data)
__global__ void nan_fill_kernel(Slots S, DList L, const CallDesc* d) {
  const int n = S.n;
  double* out = d->L;
  const long long ld = d->ld;
  LIST_LOOP(L, (size_t)n * n)
    const int i = idx / n, j = idx - (size_t)i * n;
    out[(size_t)b * n * ld + (size_t)i * ld + j] = __longlong_as_double(0x7ff8000000000000LL);
  }
}

__global__ void report_kernel(Ctl c, int nodes) {
  const CallDesc& D = *c.desc;
  phase_mark(PH_OTHER);
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < c.batch; b += gridDim.x * blockDim.x) {
    const MDev& M = c.ms[b];
    lgm_report r;
    memset(&r, 0, sizeof(r));
    const bool keep = !M.status || M.post_fail;
    r.status = M.status;
    r.s = M.s;
    r.k = keep ? M.k : 0;
    r.db_iters = M.db_iters;
    r.products = keep ? M.products : 0;
    r.divisions = 2 * M.db_iters;
    r.estimation_passes = M.passes;
    r.norm_estimations = M.nest;
    r.balanced = D.P.balance;
    r.balance_sweeps = M.sweeps;
    r.db_plateau = M.plateau;
    r.inv_skipped = M.dbskip;
    r.alpha_used = keep ? M.cert : 0.0;
    r.min_margin = M.mm;
    D.rep[b] = r;
  }
  if (blockIdx.x == 0) count_nodes(nodes);
}

// ------------------------------------------------------------------ building-block epilogues
__global__ void store_kernel(Slots S, DList L, const CallDesc* d, int k) {
  const int n = S.n;
  double* out = d->L;
  const long long ld = d->ld;
  LIST_LOOP(L, (size_t)n * n)
    const int i = idx / n, j = idx - (size_t)i * n;
    out[(size_t)b * n * ld + (size_t)i * ld + j] = S.buf(b, k)[idx];
  }
}

__global__ void block_out_kernel(Ctl c, int kind, int nodes) {
  const CallDesc& D = *c.desc;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < c.batch; b += gridDim.x * blockDim.x) {
    const MDev& M = c.ms[b];
    if (kind == 0) {         // sqrt_db: iterations, status
      D.iout[b] = M.status ? 0 : M.dbit;
      D.iout2[b] = M.status ? M.status : M.dbst;
    } else if (kind == 1) {  // estimate: value, passes (one job per matrix, table order = b)
      D.dout[b] = c.est[b].est;
      D.iout[b] = c.est[b].passes;
    } else if (kind == 2) {  // balance: sweeps, scales
      D.iout[b] = c.sweeps[b];
      for (int i = 0; i < c.n; ++i) D.dout[(size_t)b * c.n + i] = c.scale[(size_t)b * c.n + i];
    } else if (kind == 3) {  // degopt: products
      D.iout[b] = M.products;
    }
  }
  if (blockIdx.x == 0) count_nodes(nodes);
}

// est building block: one job per matrix, M1 in G_B, M2 (optional) in G_AM
__global__ void __launch_bounds__(CT) est_block_jobs_kernel(Ctl c, int has_m2) {
  const CallDesc& D = *c.desc;
  for (int b = threadIdx.x; b < c.batch; b += CT)
    est_slot(c, b, b, c.S.buf(b, G_B), D.p1, has_m2 ? c.S.buf(b, G_AM) : nullptr, D.zero_shortcut, 0);
}

// degopt building block: every matrix uses scheme kblk; first_product given or one product
__global__ void __launch_bounds__(CT) degopt_block_init_kernel(Ctl c, int have_fp) {
  const int k = c.desc->kblk;
  for (int b = threadIdx.x; b < c.batch; b += CT) {
    MDev& M = c.ms[b];
    M.k = k;
    M.s = 0;
    M.products = have_fp ? 0 : 1;
    c.ids(LS_SEL)[b] = b;
  }
  if (threadIdx.x == 0) c.cnt[LS_SEL] = c.batch;
}

}  // namespace

// ==========================================================================================
// Graph construction (stream capture) and the per-workspace graph cache
#include <mutex>

namespace {

thread_local int t_cap_nodes = 0;  // kernel launches recorded by the current capture
// LGM_GRAPH_DEBUG=1: trace the capture steps on stderr (diagnostics only)
bool graph_debug() {
  static const bool on = std::getenv("LGM_GRAPH_DEBUG") != nullptr;
  return on;
}
double gdbg_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
#define GDBG(...) do { if (graph_debug()) { std::fprintf(stderr, "[lgm graph %9.3f ms] ", gdbg_ms()); std::fprintf(stderr, __VA_ARGS__); std::fputc('\n', stderr); std::fflush(stderr); } } while (0)
inline int cap_launch() { ++t_cap_nodes; return 0; }
#define GL cap_launch(),

double host_pairwise_abs_ramp(int n) {
  // numpy pairwise sum of |(-1)^i (1 + i/max(1, n-1))| (matcore.py:270-271)
  auto get = [n](int i) { return std::fabs(((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))); };
  return lgm_pairwise_sum(get, n);
}

struct Cap {
  Ctl c;
  int n, batch;
  cudaStream_t s[4];  // capture streams by nesting depth (s[0] top level)
  cudaStream_t sB[4]; // G2 look-ahead stream of each capture sequence (a side stream joins one
                      // sequence until it ends, so every sequence forks its own)
  cudaStream_t side(cudaStream_t st) const {
    for (int i = 0; i < 4; ++i)
      if (s[i] == st) return sB[i];
    return sB[0];
  }
  cudaEvent_t evN, evP;
  int itmax;
  int mk = 14;          // m_K: estimator thin products <= m_K + 1 (s = 0) / m_K / 2 + 1
  bool cplx = false;    // complex embeddings (lgm_opts.embedded_complex): estimator variants
  bool tma = false;     // rank-64 passes by gj_update2_tma_kernel (W stored transposed)
  CUtensorMap wmap;     // the W region as (12 batch n) rows x NB doubles, 64 x 16 boxes
};

// LGM_G2_TMA=1: rank-64 passes by gj_update2_tma_kernel (TMA ring; measured 9.04 vs 8.48 ms
// per 512-job n = 512 inversion step against the one-tile-per-CTA cp.async kernel, so off
// by default -- DESIGN.md section 4)
bool g2_tma_on() {
  static const bool on = [] {
    const char* e = std::getenv("LGM_G2_TMA");
    return e && e[0] == '1';
  }();
  return on;
}

// TMA descriptor of the W region (driver entry point; no libcuda link dependency)
int make_wmap(Cap& C) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode) return LGM_ERR_CUDA;
  const cuuint64_t rows = (cuuint64_t)12 * C.batch * C.n;
  cuuint64_t gdim[2] = {(cuuint64_t)NB, rows};
  cuuint64_t gstride[1] = {(cuuint64_t)NB * 8};
  cuuint32_t box[2] = {16, 64};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&C.wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)C.c.W, gdim, gstride, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::fprintf(stderr, "logmpoly_b200 grid: cuTensorMapEncodeTiled failed (%d)\n", (int)r);
    return LGM_ERR_CUDA;
  }
  return 0;
}

dim3 ew_blocks() { return dim3(EW_BLOCKS); }

// WHILE node whose handle is set by a kernel upstream of it (captured before this call)
int cap_while_after(cudaStream_t st, cudaGraphConditionalHandle h, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaGraph_t g;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  *body = p.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  return 0;
}



int new_handle(cudaStream_t st, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus cs;
  unsigned long long id = 0;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaGraph_t g = nullptr;
  CK(cudaStreamGetCaptureInfo(st, &cs, &id, &g, &deps, &nd));
  if (cs != cudaStreamCaptureStatusActive || !g) {
    std::fprintf(stderr, "logmpoly_b200 grid: stream not capturing (%d)\n", (int)cs);
    return LGM_ERR_CUDA;
  }
  CK(cudaGraphConditionalHandleCreate(h, g, 0, 0));
  return 0;
}

int cap_ew(Cap& C, cudaStream_t st, int lst, int op, int dk, int sk, int s2k) {
  GL ew_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(lst), op, dk, sk, s2k);
  return 0;
}

int cap_norm(Cap& C, cudaStream_t st, int lst, int slot, double* out) {
  CK(cudaMemsetAsync(out, 0, C.batch * 8, st));
  GL onenorm_kernel<<<ew_blocks(), 128, 0, st>>>(C.c.S, C.c.list(lst), slot, out, &C.c.desc->P);
  return 0;
}

// one estimate per live entry of the EstJob table (batched; maxq >= every job's p1 + [M2])
int cap_estimate(Cap& C, cudaStream_t st, int maxq) {
  const int n = C.n, nj = C.batch;
  const double rsum = host_pairwise_abs_ramp(n);
  const double rsum_c = host_pairwise_abs_ramp(n > 1 ? n / 2 : 1);  // complex embeddings (order n / 2)
  GL est_nz_kernel<<<dim3(std::max(1, std::min(32, n * n / 4096)), nj), 256, 0, st>>>(C.c.est, n);
  if (n <= EST_FUSED_MAXN && est_fused_on()) {
    const int sm = n * n * 8;
#if EST_FUSED_V2
    if (n <= ESTF_SMALL_N) {  // fewer, busier warps for the small matrices (same bits)
      if (C.cplx) GL est_fused_kernel<true, 256><<<nj, 256, sm, st>>>(C.c.est, n, rsum, rsum_c, C.itmax);
      else GL est_fused_kernel<false, 256><<<nj, 256, sm, st>>>(C.c.est, n, rsum, rsum_c, C.itmax);
      return 0;
    }
#endif
    if (C.cplx) GL est_fused_kernel<true><<<nj, ESTF_THREADS, sm, st>>>(C.c.est, n, rsum, rsum_c, C.itmax);
    else GL est_fused_kernel<false><<<nj, ESTF_THREADS, sm, st>>>(C.c.est, n, rsum, rsum_c, C.itmax);
    return 0;
  }
  if (n > EST_FUSED_MAXN && n <= 512 && est_cluster_on()) {  // M1 resident in a cluster's smem
    const int cl = ecl_cl(n);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nj * cl);
    cfg.blockDim = dim3(ECL_NT);
    cfg.dynamicSmemBytes = ecl_smem(n);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (C.cplx) CK((cap_launch(), cudaLaunchKernelEx(&cfg, est_cluster_kernel<true>, C.c.est, n, rsum, rsum_c, C.itmax)));
    else CK((cap_launch(), cudaLaunchKernelEx(&cfg, est_cluster_kernel<false>, C.c.est, n, rsum, rsum_c, C.itmax)));
    return 0;
  }
  GL est_init_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(C.c.est, n, rsum, rsum_c);
  for (int sweep = 0; sweep < C.itmax; ++sweep) {
    for (int q = 0; q < maxq; ++q)
      GL est_fwd_kernel<<<dim3((n + 8 * EST_FWD_R - 1) / (8 * EST_FWD_R), nj), 256, 0, st>>>(C.c.est, n, q);
    if (C.cplx) GL est_after_fwd_kernel<true><<<nj, 256, 0, st>>>(C.c.est, n, sweep);
    else GL est_after_fwd_kernel<false><<<nj, 256, 0, st>>>(C.c.est, n, sweep);
    for (int q = 0; q < maxq; ++q) {
      // (flip: the first adjoint product runs opposite to the last forward one)
      if ((n & 1) == 0) GL est_adj2_kernel<<<dim3((n + 255) / 256, C.c.splits, nj), 128, 0, st>>>(C.c.est, n, q, maxq & 1);
      else GL est_adj_kernel<<<dim3((n + 127) / 128, C.c.splits, nj), 128, 0, st>>>(C.c.est, n, q, maxq & 1);
      GL est_adj_reduce_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(C.c.est, n, q, C.c.splits);
    }
    if (C.cplx) GL est_after_adj_kernel<true><<<nj, 256, 0, st>>>(C.c.est, n, sweep);
    else GL est_after_adj_kernel<false><<<nj, 256, 0, st>>>(C.c.est, n, sweep);
  }
  return 0;
}

// alpha (A.2) for the matrices of list `lst` (request m / th already in the state)
int cap_alpha(Cap& C, cudaStream_t st, int lst, int maxq) {
  GL alpha_a_kernel<<<1, CT, 0, st>>>(C.c, lst);
  if (cap_estimate(C, st, maxq)) return LGM_ERR_CUDA;
  GL alpha_b_kernel<<<1, CT, 0, st>>>(C.c, lst);
  if (cap_estimate(C, st, maxq)) return LGM_ERR_CUDA;
  GL alpha_c_kernel<<<1, CT, 0, st>>>(C.c, lst);
  return 0;
}

// ---- batched Gauss-Jordan inversion of the job table (capacity nj jobs)
template <int NT>
int launch_g1(Cap& C, cudaStream_t st, int nj) {
  const size_t sm = G1Smem<NT>::bytes;
  if constexpr (NT == 128) {
    if (g1_warp_panel_on() && C.n % 32 == 0) {  // warp-level panels (opt-in LGM_G1_WP=1; bit-identical, slower)
      GL gj_inv_cta_kernel<128, true><<<nj, NT, sm, st>>>(C.c.jobs, C.n);
      return 0;
    }
  }
  GL gj_inv_cta_kernel<NT><<<nj, NT, sm, st>>>(C.c.jobs, C.n);
  return 0;
}

int cap_invert(Cap& C, cudaStream_t st, int nj) {
  const int n = C.n;
  const InvJob* d_jobs = C.c.jobs;
  if (use_g1(n)) {  // G1: one CTA per inversion, no per-panel launches
    if (n <= 128) return launch_g1<128>(C, st, nj);
    if (n <= 256) return launch_g1<256>(C, st, nj);
    return launch_g1<512>(C, st, nj);
  }
  if (g3_on() && n > 256 && n <= 512 && n % (2 * NB) == 0) {  // one warp-specialised CTA per job
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GL gj_inv_ws_kernel<<<std::min(nj, sms), G3_THREADS, g3_smem(), st>>>(d_jobs, nj, n);
    return 0;
  }
  cudaStream_t sB = C.side(st);
  cudaEvent_t evN = C.evN, evP = C.evP;
  GL gj_init_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(d_jobs, n);
  const int tiles = (n + TM - 1) / TM;
  const bool cta_panel = n <= 512;  // one CTA per panel (writes A1 itself: no gj_copy_a1_kernel)
  auto panel = [&](int k0, cudaStream_t s, int a1_kind = -1, int s1_a1kind = -1) {
    const int nb = std::min(NB, n - k0);
    if (n <= 128) {
      GL gj_panel_cta_kernel<128><<<nj, 128, 4 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
    } else if (n <= 256) {
      GL gj_panel_cta_kernel<256><<<nj, 256, 8 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
    } else if (n <= 512) {
      GL gj_panel_cta_kernel<512><<<nj, 512, 16 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
    } else if (n <= CL * 512) {  // G2 panel: one 8-CTA cluster per inversion
      GL gj_panel_cluster_kernel<<<nj * CL, 512, 0, s>>>(d_jobs, n, k0, nb);
    } else {
      GL gj_panel_kernel<<<nj, 512, 0, s>>>(d_jobs, n, k0, nb, 0);
    }
  };
  auto snapshot = [&](int k0, int kind, int jlo = 0, int jhi = -1, cudaStream_t s = nullptr) {
    const int nb = std::min(NB, n - k0);
    if (jhi < 0) jhi = n;
    GL gj_snapshot_kernel<<<dim3((nb * (jhi - jlo) + 255) / 256, nj), 256, 0, s ? s : st>>>(d_jobs, n, k0, nb, kind, jlo,
                                                                                            jhi);
  };
  static const bool rank64 = [] {  // LGM_G2_RANK64=0 falls back to rank-32 passes (A/B switch)
    const char* e = std::getenv("LGM_G2_RANK64");
    return !(e && e[0] == '0');
  }();
  // rank-64 vs rank-32 passes round differently: the choice depends on n only, so a
  // matrix's arithmetic never depends on its batch-mates or on how many have converged
  const bool use64 = rank64 && n % (2 * NB) == 0;
  const bool pair0 = use64 && cta_panel && [] {
    const char* e = std::getenv("LGM_G2_PAIR");
    return !(e && e[0] == '0');
  }();
  if (!pair0) panel(0, st, use64 && cta_panel ? 2 : -1);
  if (use64) {
    // rank-64 delayed update with both panels of the next pair factored on sB during the
    // current combined pass.  Per pair (P1, P2) in buffer set q: W1 (snapshot of P1's pivot
    // rows), A1 (copy of P1's multipliers), stage-1 update of P2's columns, factor P2, W2.
    auto prepare_pair = [&](int k0, int q, cudaStream_t s, bool full_snapshot) {
      // P1 = [k0, k0+NB) already factored; everything except the full-width W1 / W2
      if (cta_panel) {  // stage-1 update fused into P2's panel kernel
        panel(k0 + NB, s, -1, 3 * q + 2);
        return;
      }
      if (full_snapshot) snapshot(k0, 3 * q, 0, n, s);
      else snapshot(k0, 3 * q, k0 + NB, k0 + 2 * NB, s);  // P2's columns only (for stage 1)
      GL gj_copy_a1_kernel<<<dim3((n * NB + 255) / 256, nj), 256, 0, s>>>(d_jobs, n, k0, 3 * q + 2);
      GL gj_update_kernel<<<dim3(1, tiles, nj), 128, 0, s>>>(d_jobs, n, k0, NB, k0 + NB, k0 + NB, k0 + 2 * NB, 0, 0,
                                                             3 * q);
      panel(k0 + NB, s);
    };
    const bool tma = cta_panel && C.tma;
    static const bool pair_on = [] {  // LGM_G2_PAIR=0: the two panels as separate launches (A/B)
      const char* e = std::getenv("LGM_G2_PAIR");
      return !(e && e[0] == '0');
    }();
    const bool pairk = cta_panel && pair_on;
    auto panel_pair = [&](int k0p, cudaStream_t s, int a1k) {  // both panels of a pair, one launch
      if (n <= 128) GL gj_panel_pair_kernel<128><<<nj, 128, 4 * 32 * 33 * 8, s>>>(d_jobs, n, k0p, a1k);
      else if (n <= 256) GL gj_panel_pair_kernel<256><<<nj, 256, 8 * 32 * 33 * 8, s>>>(d_jobs, n, k0p, a1k);
      else if (panel2_on() && n % 32 == 0) GL gj_panel_pair2_kernel<<<nj, 256, 8 * 32 * 33 * 8, s>>>(d_jobs, n, k0p, a1k);
      else GL gj_panel_pair_kernel<512><<<nj, 512, 16 * 32 * 33 * 8, s>>>(d_jobs, n, k0p, a1k);
    };
    auto pass = [&](int k0p, int cb, int clo, int chi, int exlo, int exhi, int qq, bool narrow) {
      if (tma) {
        GL gj_update2_tma_kernel<<<dim3((n + UT_ROWS - 1) / UT_ROWS, nj), UT_THREADS, ut_smem(), st>>>(d_jobs, n, k0p, cb, clo, chi, exlo,
                                                                                      exhi, qq, C.c.W, C.wmap);
      } else if (up2s_on()) {  // one K-half slot per CTA (4 CTAs/SM)
        if (narrow)
          GL gj_update2s_kernel<64><<<dim3(1, tiles, nj), 128, up2s_smem<64>(), st>>>(d_jobs, n, k0p, cb, clo, chi, exlo,
                                                                                     exhi, qq);
        else
          GL gj_update2s_kernel<64><<<dim3(tiles, n / 64, nj), 128, up2s_smem<64>(), st>>>(d_jobs, n, k0p, cb, clo, chi,
                                                                                          exlo, exhi, qq);
      } else if (narrow) {
        GL gj_update2_kernel<64><<<dim3(1, tiles, nj), 128, up2_smem<64>(), st>>>(d_jobs, n, k0p, cb, clo, chi, exlo,
                                                                                 exhi, qq);
      } else {
        GL gj_update2_kernel<G2_RT><<<dim3(tiles, n / G2_RT, nj), 2 * G2_RT, up2_smem<G2_RT>(), st>>>(
            d_jobs, n, k0p, cb, clo, chi, exlo, exhi, qq);
      }
    };
    if (pairk) panel_pair(0, st, 2);
    else prepare_pair(0, 0, st, !cta_panel);
    if (cta_panel) GL gj_w2_mma_kernel<<<dim3(n / 64, nj), 128, 0, st>>>(d_jobs, n, 0, 0, tma ? 1 : 0);
    else GL gj_w2_kernel<<<dim3((n + 127) / 128, nj), 128, 0, st>>>(d_jobs, n, 0, 0, 0);
    for (int k0 = 0, q = 0; k0 < n; k0 += 2 * NB, q ^= 1) {
      const int kn = k0 + 2 * NB;
      const bool next = kn < n;
      if (next) {  // finish the next pair's columns, then factor both of its panels on sB
        pass(k0, kn, kn, kn + 2 * NB, 0, 0, q, true);
        CK(cudaEventRecord(evN, st));
        CK(cudaStreamWaitEvent(sB, evN, 0));
        if (pairk) {
          panel_pair(kn, sB, 3 * (q ^ 1) + 2);
        } else {
          panel(kn, sB, cta_panel ? 3 * (q ^ 1) + 2 : -1);
          prepare_pair(kn, q ^ 1, sB, false);
        }
        CK(cudaEventRecord(evP, sB));
      }
      pass(k0, 0, 0, n, next ? kn : 0, next ? kn + 2 * NB : 0, q, false);
      if (next) {  // full-width W1 / W2 of the next pair need this pass's rows
        CK(cudaStreamWaitEvent(st, evP, 0));
        if (cta_panel) {
          GL gj_w2_mma_kernel<<<dim3(n / 64, nj), 128, 0, st>>>(d_jobs, n, kn, q ^ 1, tma ? 1 : 0);
        } else {
          snapshot(kn, 3 * (q ^ 1));
          GL gj_w2_kernel<<<dim3((n + 127) / 128, nj), 128, 0, st>>>(d_jobs, n, kn, q ^ 1, 0);
        }
      }
    }
    return 0;
  }
  snapshot(0, 0);
  for (int k0 = 0, par = 0; k0 < n; k0 += NB, par ^= 1) {
    const int nb = std::min(NB, n - k0);
    const int kn = k0 + NB, nbn = kn < n ? std::min(NB, n - kn) : 0;
    if (kn < n) {
      GL gj_update_kernel<<<dim3(1, tiles, nj), 128, 0, st>>>(d_jobs, n, k0, nb, kn, kn, kn + nbn, 0, 0, par);
      CK(cudaEventRecord(evN, st));
      CK(cudaStreamWaitEvent(sB, evN, 0));
      panel(kn, sB);
      CK(cudaEventRecord(evP, sB));
    }
    GL gj_update_kernel<<<dim3(tiles, tiles, nj), 128, 0, st>>>(d_jobs, n, k0, nb, 0, 0, n, kn, kn + nbn, par);
    if (kn < n) {
      CK(cudaStreamWaitEvent(st, evP, 0));
      snapshot(kn, par ^ 1);
    }
  }
  return 0;
}

int cap_if_after(cudaStream_t st, cudaGraphConditionalHandle h, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaGraph_t g;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  *body = p.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  return 0;
}

DbArgs db_args(Cap& C, bool first, int list) {
  const int n = C.n;
  DbArgs a;
  a.S = C.c.S;
  a.L = C.c.list(list);
  a.xpiv = C.c.piv;
  a.xstep = C.c.step;
  a.ypiv = C.c.piv + (size_t)C.batch * n;
  a.ystep = C.c.step + (size_t)C.batch * n;
  a.xlog = C.c.logdet;
  a.ylog = C.c.logdet + C.batch;
  a.scaling = C.c.scaling;
  a.first = first ? 1 : 0;
  a.change = C.c.change;
  a.size = C.c.size;
  a.istat = C.c.istat;
  a.batch = C.batch;
  a.ms = C.c.ms;
  a.xn_slot = G_Q0;
  a.P = &C.c.desc->P;
  return a;
}

// one DB iteration over LS_DB (first: X only, Y = I), ending in decide_db_kernel(h); later
// iterations add the lazy-X^-1 tail (IF body captured on st_if)
int cap_db_iter(Cap& C, cudaStream_t st, bool first, cudaGraphConditionalHandle h, int block_mode,
                cudaStream_t st_if = nullptr) {
  const int n = C.n;
  const int n0 = t_cap_nodes;
  const bool oop = inv_oop(n);
  const bool lazy = !first && st_if && lazyx_on();
  cudaGraphConditionalHandle h2 = 0;
  if (lazy && new_handle(st, &h2)) return LGM_ERR_CUDA;
  GL build_jobs_kernel<<<1, CT, 0, st>>>(C.c, first ? 1 : 0, oop ? 1 : 0);
  if (!oop) {  // G2 inverts in place: copies first
    if (cap_ew(C, st, LS_DB, 1, G_XI, G_B, G_B)) return LGM_ERR_CUDA;
    if (!first && cap_ew(C, st, LS_DB, 1, G_YI, G_Y, G_Y)) return LGM_ERR_CUDA;
  }
  if (cap_invert(C, st, first ? C.batch : 2 * C.batch)) return LGM_ERR_CUDA;
  GL db_update_kernel<<<dim3((n + 127) / 128, C.batch), 128, 0, st>>>(db_args(C, first, LS_DB));
  const int nodes = t_cap_nodes - n0 + 1 + (lazy ? 1 : 0);
  GL decide_db_kernel<<<1, CT, 0, st>>>(C.c, h, first ? 0 : nodes, first ? 1 : 0, block_mode, h2, lazy ? 1 : 0,
                                         lazyx_f());
  if (lazy) {
    if (cap_ew(C, st, LS_POK, 1, G_B, G_Q0, G_Q0)) return LGM_ERR_CUDA;  // converged: X <- X'
    cudaGraph_t body;
    if (cap_if_after(st, h2, &body)) return LGM_ERR_CUDA;
    const int saved = t_cap_nodes;
    CK(cudaStreamBeginCaptureToGraph(st_if, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int m0 = t_cap_nodes;
    GL build_jobs_px_kernel<<<1, CT, 0, st_if>>>(C.c, oop ? 1 : 0);
    if (!oop && cap_ew(C, st_if, LS_PMISS, 1, G_XI, G_B, G_B)) return LGM_ERR_CUDA;
    if (cap_invert(C, st_if, C.batch)) return LGM_ERR_CUDA;
    const int mnodes = t_cap_nodes - m0 + 1;
    GL db_fix_kernel<<<dim3((n + 127) / 128, C.batch), 128, 0, st_if>>>(db_args(C, false, LS_PMISS), mnodes);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(st_if, &tmp));
    t_cap_nodes = saved;  // the IF body's kernels are counted by db_fix_kernel when it runs
  }
  return 0;
}

// the square roots of LS_DB (already = roots): Y = I, iteration 1, WHILE(more iterations)
int cap_sqrt_db(Cap& C, int depth, int block_mode) {
  cudaStream_t st = C.s[depth];
  if (cap_ew(C, st, LS_DB, 2, G_Y, G_Y, G_Y)) return LGM_ERR_CUDA;  // Y = I
  cudaGraphConditionalHandle h;
  cudaGraph_t body;
  // handle created first so that iteration 1's decide kernel can set it
  if (new_handle(st, &h)) return LGM_ERR_CUDA;
  GDBG("sqrt_db: handle created (depth %d)", depth);
  if (cap_db_iter(C, st, true, h, block_mode)) return LGM_ERR_CUDA;
  GDBG("sqrt_db: first iteration captured");
  if (cap_while_after(st, h, &body)) return LGM_ERR_CUDA;
  GDBG("sqrt_db: while node added");
  cudaStream_t sb = C.s[depth + 1];
  const int saved = t_cap_nodes;  // the body's kernels are counted by its decide kernel
  CK(cudaStreamBeginCaptureToGraph(sb, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  if (cap_db_iter(C, sb, false, h, block_mode, depth + 2 < 4 ? C.s[depth + 2] : nullptr)) return LGM_ERR_CUDA;
  cudaGraph_t tmp;
  CK(cudaStreamEndCapture(sb, &tmp));
  t_cap_nodes = saved;
  GDBG("sqrt_db: body captured");
  return 0;
}

// one scaling-loop iteration (A.1 step 5) at depth d, ending in decide_post_kernel(h)
int cap_scal_iter(Cap& C, int depth, int maxq, cudaGraphConditionalHandle h, bool in_loop) {
  cudaStream_t st = C.s[depth];
  const int n0 = t_cap_nodes;
  GL decide_act_kernel<<<1, CT, 0, st>>>(C.c);
  if (cap_ew(C, st, LS_ACT, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;  // A - I
  if (cap_norm(C, st, LS_ACT, G_AM, C.c.nrm)) return LGM_ERR_CUDA;
  if (cap_norm(C, st, LS_ACTAI2, G_AP, C.c.nrm2)) return LGM_ERR_CUDA;
  GL scal_req_kernel<<<1, CT, 0, st>>>(C.c);
  if (cap_alpha(C, st, LS_ACT, maxq)) return LGM_ERR_CUDA;
  GL decide_roots_kernel<<<1, CT, 0, st>>>(C.c);
  if (cap_ew(C, st, LS_ROOTS, 1, G_AP, G_B, G_B)) return LGM_ERR_CUDA;  // A_prev = B
  if (cap_sqrt_db(C, depth, 0)) return LGM_ERR_CUDA;
  const int nodes = t_cap_nodes - n0 + 2;
  GL decide_post_kernel<<<1, CT, 0, st>>>(C.c, h, in_loop ? nodes : 0);
  if (cap_ew(C, st, LS_OK, 3, G_AP, G_AP, G_B)) return LGM_ERR_CUDA;  // A_I2 = A_prev - 2B + I
  return 0;
}

// ------------------------------------------------------------------ whole programs
enum { PROG_LOGM = 0, PROG_SQRTDB, PROG_EST, PROG_BALANCE, PROG_DEGOPT, PROG_EXPM };

int cap_load(Cap& C, cudaStream_t st, const double* const* src, int slot) {
  // load_kernel writes slot G_B; other slots by a copy
  GL load_kernel<<<ew_blocks(), 256, 0, st>>>(src, &C.c.desc->ld, C.c.S, C.c.list(LS_ALL), C.c.flag);
  if (slot != G_B && cap_ew(C, st, LS_ALL, 1, slot, G_B, G_B)) return LGM_ERR_CUDA;
  return 0;
}

// the fused polynomial chain over LS_SEL (lists LS_POLY0 + j built by decide_poly_kernel)
int cap_poly(Cap& C, cudaStream_t st, bool logm) {
  const int n = C.n;
  PolyArgs a;
  a.S = C.c.S;
  a.d = C.c.desc;
  a.ms = C.c.ms;
  a.scale = C.c.scale;
  a.nonfinite = logm ? C.c.flag : nullptr;
  a.logm = logm ? 1 : 0;
  GL poly_start_kernel<<<ew_blocks(), 256, 0, st>>>(a, C.c.list(LS_SEL));
  const int tiles = (n + TM - 1) / TM;
  const size_t gsm = (POLY_1STAGE ? 1 : 2) * (size_t)(GP_A + GP_B) * 8;
  for (int j = 1; j < LGM_K_MAX; ++j) {
    if ((n & 1) == 0) GL poly_gemm_kernel<true><<<dim3(tiles, tiles, C.batch), 128, gsm, st>>>(a, C.c.list(LS_POLY0 + j), j);
    else GL poly_gemm_kernel<false><<<dim3(tiles, tiles, C.batch), 128, gsm, st>>>(a, C.c.list(LS_POLY0 + j), j);
  }
  return 0;
}

int cap_logm(Cap& C) {
  cudaStream_t st = C.s[0];
  const int n = C.n;
  GL ctl_init_kernel<<<1, CT, 0, st>>>(C.c);
  GL fill_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.scale, (size_t)C.batch * n, 1.0);
  if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
  GL decide_live_kernel<<<1, CT, 0, st>>>(C.c);
  // balance (matcore.py:180-215); the kernel returns at once when the call disables it
  GL balance_kernel_g<<<C.batch, bal_threads(n), bal_smem(n), st>>>(C.c.S, C.c.list(LS_LIVE), C.c.scale, C.c.sweeps,
                                                                    100, C.c.margin, &C.c.desc->P.balance, nullptr,
                                                                    &C.c.desc->P);
  if (cap_ew(C, st, LS_LIVE, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;
  if (cap_norm(C, st, LS_LIVE, G_AM, C.c.nrm)) return LGM_ERR_CUDA;
  GL decide_start_kernel<<<1, CT, 0, st>>>(C.c);
  // scaling loop: iteration 1 peeled (s = 0: estimates of (A - I)^{m_K}, (A - I)^{m_K + 1}),
  // then WHILE(some matrix still scaling) with s >= 1 (A_I2-based estimates: <= m_K/2 + 1)
  cudaGraphConditionalHandle hs;
  if (new_handle(st, &hs)) return LGM_ERR_CUDA;
  const int mk = C.mk;
  if (cap_scal_iter(C, 0, mk + 1, hs, false)) return LGM_ERR_CUDA;
  cudaGraph_t body;
  if (cap_while_after(st, hs, &body)) return LGM_ERR_CUDA;
  int saved = t_cap_nodes;
  CK(cudaStreamBeginCaptureToGraph(C.s[1], body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  if (cap_scal_iter(C, 1, mk / 2 + 1, hs, true)) return LGM_ERR_CUDA;
  {
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(C.s[1], &tmp));
  }
  t_cap_nodes = saved;
  // select_order
  GL decide_sel_kernel<<<1, CT, 0, st>>>(C.c);
  if (cap_ew(C, st, LS_SEL, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;
  if (cap_norm(C, st, LS_SEL, G_AM, C.c.nrm)) return LGM_ERR_CUDA;
  {  // s = 0: A_I2 = (B - I)(B - I), one product
    const int tiles = (n + TM - 1) / TM;
    if ((n & 1) == 0) {
      const size_t sm = 2 * (size_t)(GP_A + GP_B) * 8;
      GL gemm_plain_kernel<<<dim3(tiles, tiles, C.batch), 128, sm, st>>>(C.c.S, C.c.list(LS_NEEDAI2), G_AM, G_AM, G_AP);
    } else {
      CombSpec cs{};
      cs.nterm = 1;
      cs.node[0] = G_AM;
      cs.coef[0] = 1.0;
      GL gemm_comb_kernel<<<dim3(tiles, tiles, C.batch), 128, 0, st>>>(C.c.S, C.c.list(LS_NEEDAI2), cs, G_AM, G_AP);
    }
  }
  if (cap_norm(C, st, LS_SEL, G_AP, C.c.nrm2)) return LGM_ERR_CUDA;
  cudaGraphConditionalHandle hsel;
  if (new_handle(st, &hsel)) return LGM_ERR_CUDA;
  GL select_init_kernel<<<1, CT, 0, st>>>(C.c, hsel);
  if (cap_while_after(st, hsel, &body)) return LGM_ERR_CUDA;
  saved = t_cap_nodes;
  CK(cudaStreamBeginCaptureToGraph(C.s[1], body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  {
    const int n0 = t_cap_nodes;
    if (cap_alpha(C, C.s[1], LS_CUR, mk / 2 + 1)) return LGM_ERR_CUDA;
    GL select_step_kernel<<<1, CT, 0, C.s[1]>>>(C.c, hsel, t_cap_nodes - n0 + 1);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(C.s[1], &tmp));
  }
  t_cap_nodes = saved;
  // polynomial: one fused kernel per product (cap_poly)
  GL decide_poly_kernel<<<1, CT, 0, st>>>(C.c);
  CK(cudaMemsetAsync(C.c.flag, 0, C.batch * 4, st));
  if (cap_poly(C, st, true)) return LGM_ERR_CUDA;
  GL decide_final_kernel<<<1, CT, 0, st>>>(C.c);
  GL nan_fill_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_FAILED), C.c.desc);
  GL report_kernel<<<(C.batch + 255) / 256, 256, 0, st>>>(C.c, t_cap_nodes + 1);
  return 0;
}

int cap_block(Cap& C, int prog, int has2, int p1) {
  cudaStream_t st = C.s[0];
  const int n = C.n;
  GL ctl_init_kernel<<<1, CT, 0, st>>>(C.c);
  GL fill_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.scale, (size_t)C.batch * n, 1.0);
  if (prog == PROG_SQRTDB) {
    if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
    GL decide_live_kernel<<<1, CT, 0, st>>>(C.c);
    GL decide_db_start_kernel<<<1, CT, 0, st>>>(C.c);
    if (cap_sqrt_db(C, 0, 1)) return LGM_ERR_CUDA;
    GL store_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_ALL), C.c.desc, G_B);
    GL block_out_kernel<<<(C.batch + 255) / 256, 256, 0, st>>>(C.c, 0, t_cap_nodes + 1);
  } else if (prog == PROG_EST) {
    if (has2) {  // M2 -> G_AM (via G_B), then M1 -> G_B
      if (cap_load(C, st, &C.c.desc->A2, G_AM)) return LGM_ERR_CUDA;
    }
    if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
    GL est_block_jobs_kernel<<<1, CT, 0, st>>>(C.c, has2);
    if (cap_estimate(C, st, p1 + (has2 ? 1 : 0))) return LGM_ERR_CUDA;
    GL block_out_kernel<<<(C.batch + 255) / 256, 256, 0, st>>>(C.c, 1, t_cap_nodes + 1);
  } else if (prog == PROG_BALANCE) {
    if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
    GL balance_kernel_g<<<C.batch, bal_threads(n), bal_smem(n), st>>>(C.c.S, C.c.list(LS_ALL), C.c.scale, C.c.sweeps,
                                                                      0, C.c.margin, nullptr, &C.c.desc->max_sweeps, nullptr);
    GL store_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_ALL), C.c.desc, G_B);
    GL block_out_kernel<<<(C.batch + 255) / 256, 256, 0, st>>>(C.c, 2, t_cap_nodes + 1);
  } else if (prog == PROG_EXPM) {
    if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
    if (cap_norm(C, st, LS_ALL, G_B, C.c.nrm)) return LGM_ERR_CUDA;
    GL expm_prep_kernel<<<1, CT, 0, st>>>(C.c);
    GL expm_scale_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_ALL), C.c.scale);
    if (cap_ew(C, st, LS_ALL, 2, G_Y, G_Y, G_Y)) return LGM_ERR_CUDA;  // T = I
    const int tiles = (n + TM - 1) / TM;
    const size_t gsm = 2 * (size_t)(GP_A + GP_B) * 8;
    auto gemm = [&](cudaStream_t s, DList L, int as, int bs, int cs, int j, int mode) {
      if ((n & 1) == 0) GL expm_gemm_kernel<true><<<dim3(tiles, tiles, C.batch), 128, gsm, s>>>(C.c.S, L, as, bs, cs, j, mode);
      else GL expm_gemm_kernel<false><<<dim3(tiles, tiles, C.batch), 128, gsm, s>>>(C.c.S, L, as, bs, cs, j, mode);
    };
    for (int j = 20; j >= 1; --j) {  // Horner: 20 steps, T ends in G_Y (even count)
      const bool fromY = (j % 2 == 0);
      gemm(st, C.c.list(LS_ALL), G_B, fromY ? G_Y : G_XI, fromY ? G_XI : G_Y, j, 0);
    }
    // squarings: WHILE(some matrix has squarings left), two per body (slot parity)
    cudaGraphConditionalHandle h;
    if (new_handle(st, &h)) return LGM_ERR_CUDA;
    GL expm_sq_decide_kernel<<<1, CT, 0, st>>>(C.c, h, 1, 0);
    cudaGraph_t body;
    if (cap_while_after(st, h, &body)) return LGM_ERR_CUDA;
    const int saved = t_cap_nodes;
    CK(cudaStreamBeginCaptureToGraph(C.s[1], body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    {
      const int n0 = t_cap_nodes;
      gemm(C.s[1], C.c.list(LS_CUR), G_Y, G_Y, G_XI, 0, 1);
      GL expm_sq_decide_kernel<<<1, CT, 0, C.s[1]>>>(C.c, h, 0, 0);
      gemm(C.s[1], C.c.list(LS_CUR), G_XI, G_XI, G_Y, 0, 1);
      GL expm_sq_decide_kernel<<<1, CT, 0, C.s[1]>>>(C.c, h, 1, t_cap_nodes - n0 + 1);
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(C.s[1], &tmp));
    }
    t_cap_nodes = saved;
    GL expm_store_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_ALL), C.c.desc, C.c.ms);
    GL block_out_kernel<<<1, 32, 0, st>>>(C.c, 4, t_cap_nodes + 1);
  } else {  // PROG_DEGOPT: X -> P2 slot G_B, first product -> G_AP (given, or one GEMM)
    if (has2 && cap_load(C, st, &C.c.desc->A2, G_AP)) return LGM_ERR_CUDA;
    if (cap_load(C, st, &C.c.desc->A, G_B)) return LGM_ERR_CUDA;
    GL degopt_block_init_kernel<<<1, CT, 0, st>>>(C.c, has2);
    const int tiles = (n + TM - 1) / TM;
    if (!has2) {
      CombSpec cs{};
      cs.nterm = 1;
      cs.node[0] = G_B;
      cs.coef[0] = 1.0;
      GL gemm_comb_kernel<<<dim3(tiles, tiles, C.batch), 128, 0, st>>>(C.c.S, C.c.list(LS_ALL), cs, G_B, G_AP);
    }
    GL decide_poly_kernel<<<1, CT, 0, st>>>(C.c);
    if (cap_poly(C, st, false)) return LGM_ERR_CUDA;
    GL decide_final_kernel<<<1, CT, 0, st>>>(C.c);
    GL block_out_kernel<<<(C.batch + 255) / 256, 256, 0, st>>>(C.c, 3, t_cap_nodes + 1);
  }
  return 0;
}

// ------------------------------------------------------------------ cache
struct GraphKey {
  int dev, prog, n, batch, itmax, has2, p1;
  const void* ws;
  int mk;  // m_K of the call's max_k (bounds the estimator's thin-product count)
  int cplx = 0;  // complex embeddings (estimator kernel variants)
  bool operator==(const GraphKey& o) const {
    return dev == o.dev && prog == o.prog && n == o.n && batch == o.batch && itmax == o.itmax && has2 == o.has2 &&
           p1 == o.p1 && ws == o.ws && mk == o.mk && cplx == o.cplx;
  }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  unsigned long long used = 0;
};
std::mutex g_cache_mu;
std::vector<GraphEntry> g_cache;  // small LRU of instantiated programs
unsigned long long g_cache_tick = 0;
constexpr size_t CACHE_MAX = 24;

struct CapStreams {
  cudaStream_t s[8] = {};
  cudaEvent_t evN = nullptr, evP = nullptr;
  ~CapStreams() {
    for (auto x : s)
      if (x) cudaStreamDestroy(x);
    if (evN) cudaEventDestroy(evN);
    if (evP) cudaEventDestroy(evP);
  }
};

// dynamic shared-memory limits are per device: set before every capture (no process-wide flag)
int set_attrs(int n) {
  const cudaFuncAttribute mx = cudaFuncAttributeMaxDynamicSharedMemorySize;
  CK(cudaFuncSetAttribute(est_fused_kernel<false>, mx, EST_FUSED_MAXN * EST_FUSED_MAXN * 8));
  CK(cudaFuncSetAttribute(est_fused_kernel<true>, mx, EST_FUSED_MAXN * EST_FUSED_MAXN * 8));
#if EST_FUSED_V2
  CK(cudaFuncSetAttribute(est_fused_kernel<false, 256>, mx, ESTF_SMALL_N * ESTF_SMALL_N * 8));
  CK(cudaFuncSetAttribute(est_fused_kernel<true, 256>, mx, ESTF_SMALL_N * ESTF_SMALL_N * 8));
#endif
  CK(cudaFuncSetAttribute(gj_inv_cta_kernel<128>, mx, (int)G1Smem<128>::bytes));
  CK(cudaFuncSetAttribute(gj_inv_cta_kernel<128, true>, mx, (int)G1Smem<128>::bytes));
  CK(cudaFuncSetAttribute(gj_inv_cta_kernel<256>, mx, (int)G1Smem<256>::bytes));
  CK(cudaFuncSetAttribute(gj_inv_cta_kernel<512>, mx, (int)G1Smem<512>::bytes));
  CK(cudaFuncSetAttribute(gj_panel_cta_kernel<128>, mx, 4 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_cta_kernel<256>, mx, 8 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_cta_kernel<512>, mx, 16 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_pair_kernel<128>, mx, 4 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_pair_kernel<256>, mx, 8 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_pair_kernel<512>, mx, 16 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_panel_pair2_kernel, mx, 8 * 32 * 33 * 8));
  CK(cudaFuncSetAttribute(gj_update2_kernel<64>, mx, (int)up2_smem<64>()));
  CK(cudaFuncSetAttribute(gj_update2_kernel<128>, mx, (int)up2_smem<128>()));
  CK(cudaFuncSetAttribute(gj_update2s_kernel<64>, mx, (int)up2s_smem<64>()));
  CK(cudaFuncSetAttribute(gj_inv_ws_kernel, mx, (int)g3_smem()));
  CK(cudaFuncSetAttribute(gemm_plain_kernel, mx, (int)(2 * (size_t)(GP_A + GP_B) * 8)));
  CK(cudaFuncSetAttribute(poly_gemm_kernel<true>, mx, (int)(2 * (size_t)(GP_A + GP_B) * 8)));
  CK(cudaFuncSetAttribute(expm_gemm_kernel<true>, mx, (int)(2 * (size_t)(GP_A + GP_B) * 8)));
  CK(cudaFuncSetAttribute(expm_gemm_kernel<false>, mx, (int)(2 * (size_t)(GP_A + GP_B) * 8)));
  CK(cudaFuncSetAttribute(poly_gemm_kernel<false>, mx, (int)(2 * (size_t)(GP_A + GP_B) * 8)));
  CK(cudaFuncSetAttribute(gj_update2_tma_kernel, mx, (int)ut_smem()));
  CK(cudaFuncSetAttribute(est_cluster_kernel<false>, mx, (int)ecl_smem(512)));
  CK(cudaFuncSetAttribute(est_cluster_kernel<true>, mx, (int)ecl_smem(512)));
  CK(cudaFuncSetAttribute(est_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(est_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(balance_kernel_g, mx, (int)bal_smem(n)));
  return 0;
}

int build_exec(const GraphKey& k, void* ws, cudaGraphExec_t* out) {
  GDBG("build_exec start");
  if (set_attrs(k.n)) return LGM_ERR_CUDA;
  GDBG("attrs set");
  CapStreams cs;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (int i = 0; i < 4; ++i) CK(cudaStreamCreateWithFlags(&cs.s[i], cudaStreamNonBlocking));
  for (int i = 4; i < 8; ++i) CK(cudaStreamCreateWithPriority(&cs.s[i], cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&cs.evN, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&cs.evP, cudaEventDisableTiming));
  GDBG("streams created");
  Cap C;
  C.n = k.n;
  C.batch = k.batch;
  C.c = ctl_carve(ws, k.n, k.batch);
  for (int i = 0; i < 4; ++i) {
    C.s[i] = cs.s[i];
    C.sB[i] = cs.s[4 + i];
  }
  C.evN = cs.evN;
  C.evP = cs.evP;
  C.itmax = k.itmax;
  C.mk = k.mk > 0 ? k.mk : LGM_ORDER_DEFAULT[LGM_K_DEFAULT - 1];
  C.cplx = k.cplx != 0;
  C.tma = g2_tma_on() && k.n <= 512 && k.n % (2 * NB) == 0 && !use_g1(k.n);
  if (C.tma && make_wmap(C)) return LGM_ERR_CUDA;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  GDBG("capture prog %d n %d batch %d", k.prog, k.n, k.batch);
  CK(cudaStreamBeginCaptureToGraph(C.s[0], g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  t_cap_nodes = 0;
  int rc = k.prog == PROG_LOGM ? cap_logm(C) : cap_block(C, k.prog, k.has2, k.p1);
  GDBG("capture body done rc %d nodes %d", rc, t_cap_nodes);
  for (int i = 3; i >= 1; --i) {  // a failed capture may leave a body sequence open
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(C.s[i], &st);
    if (st != cudaStreamCaptureStatusNone) {
      cudaGraph_t t2 = nullptr;
      cudaStreamEndCapture(C.s[i], &t2);
    }
  }
  cudaGraph_t tmp;
  cudaError_t e = cudaStreamEndCapture(C.s[0], &tmp);
  GDBG("end capture: %s", cudaGetErrorString(e));
  if (rc || e != cudaSuccess) {
    cudaGetLastError();  // clear the sticky capture error
    cudaGraphDestroy(g);
    std::fprintf(stderr, "logmpoly_b200 grid: graph capture failed (%s)\n", cudaGetErrorString(e));
    return LGM_ERR_CUDA;
  }
  e = cudaGraphInstantiate(out, g, 0);
  GDBG("instantiate: %s", cudaGetErrorString(e));
  cudaGraphDestroy(g);
  GDBG("graph destroyed");
  if (e != cudaSuccess) {
    std::fprintf(stderr, "logmpoly_b200 grid: graph instantiate failed (%s)\n", cudaGetErrorString(e));
    return LGM_ERR_CUDA;
  }
  return 0;
}

// launch the program for key k on stream st with this call's descriptor
int run_prog(const GraphKey& k0, void* ws, const CallDesc& d, cudaStream_t st) {
  GraphKey k = k0;
  CK(cudaGetDevice(&k.dev));
  k.ws = ws;
  const Ctl c = ctl_carve(ws, k.n, k.batch);
  if (lgm_ws_guard_bytes())
    ws_guard_kernel<<<256, 256, 0, st>>>((unsigned char*)ws, k.n, k.batch, lgm_ws_guard_bytes(), 0, nullptr);
  lgm_count_launch(), setup_kernel<<<1, 1, 0, st>>>(c.desc, d);
  CK(cudaGetLastError());
  std::lock_guard<std::mutex> lock(g_cache_mu);
  GraphEntry* ent = nullptr;
  for (auto& e : g_cache)
    if (e.key == k) ent = &e;
  if (!ent) {
    cudaGraphExec_t ex = nullptr;
    if (build_exec(k, ws, &ex)) return LGM_ERR_CUDA;
    GDBG("build_exec done (streams destroyed)");
    if (g_cache.size() >= CACHE_MAX) {
      auto old = std::min_element(g_cache.begin(), g_cache.end(),
                                  [](const GraphEntry& a, const GraphEntry& b) { return a.used < b.used; });
      cudaGraphExecDestroy(old->exec);  // freed asynchronously if still in flight
      g_cache.erase(old);
    }
    g_cache.push_back(GraphEntry{k, ex, 0});
    ent = &g_cache.back();
  }
  ent->used = ++g_cache_tick;
  GDBG("launch");
  CK(cudaGraphLaunch(ent->exec, st));
  GDBG("launched");
  return 0;
}

CallDesc desc_base(const LgmParams& P) {
  CallDesc d;
  std::memset(&d, 0, sizeof(d));
  d.P = P;
  return d;
}

}  // namespace

// ============================================================================ entry points (n > 64)

size_t lgm_grid_workspace_bytes(int64_t n, int64_t batch) { return ctl_bytes(n, batch); }

int lgm_grid_logm(const double* A, double* L, int64_t n, int64_t batch, int64_t ld, const LgmParams& P,
                  lgm_report* rep, void* ws, cudaStream_t st) {
  CallDesc d = desc_base(P);
  d.A = A;
  d.L = L;
  d.ld = ld;
  d.rep = rep;
  GraphKey k{0, PROG_LOGM, (int)n, (int)batch, P.est_itmax, 0, 0, nullptr, P.order[P.max_k - 1], P.cplx};
  return run_prog(k, ws, d, st);
}

int lgm_grid_sqrt_db(const double* A, double* X, int64_t n, int64_t batch, int64_t ld, double tol, int maxiter,
                     int* iters, int* status, void* ws, cudaStream_t st) {
  LgmParams P{};
  CallDesc d = desc_base(P);
  d.A = A;
  d.L = X;
  d.ld = ld;
  d.iout = iters;
  d.iout2 = status;
  d.tol = tol;
  d.maxiter = maxiter;
  GraphKey k{0, PROG_SQRTDB, (int)n, (int)batch, 0, 0, 0, nullptr, 0};
  return run_prog(k, ws, d, st);
}

int lgm_grid_est(const double* M1, int p1, const double* M2, int64_t n, int64_t batch, int64_t ld, int itmax,
                 int zero_shortcut, double* est, int* passes, void* ws, cudaStream_t st) {
  LgmParams P{};
  CallDesc d = desc_base(P);
  d.A = M1;
  d.A2 = M2;
  d.ld = ld;
  d.p1 = p1;
  d.zero_shortcut = zero_shortcut;
  d.dout = est;
  d.iout = passes;
  GraphKey k{0, PROG_EST, (int)n, (int)batch, itmax, M2 ? 1 : 0, p1, nullptr, 0};
  return run_prog(k, ws, d, st);
}

int lgm_grid_balance(const double* A, double* B, double* scale, int64_t n, int64_t batch, int64_t ld,
                     int max_sweeps, int* sweeps, void* ws, cudaStream_t st) {
  LgmParams P{};
  CallDesc d = desc_base(P);
  d.A = A;
  d.L = B;
  d.ld = ld;
  d.dout = scale;
  d.iout = sweeps;
  d.max_sweeps = max_sweeps;
  GraphKey k{0, PROG_BALANCE, (int)n, (int)batch, 0, 0, 0, nullptr, 0};
  return run_prog(k, ws, d, st);
}

int lgm_grid_degopt(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld, int k,
                    int* products, const LgmParams& P, void* ws, cudaStream_t st) {
  CallDesc d = desc_base(P);
  d.A = X;
  d.A2 = FP;
  d.L = Z;
  d.ld = ld;
  d.kblk = k;
  d.iout = products;
  GraphKey key{0, PROG_DEGOPT, (int)n, (int)batch, 0, FP ? 1 : 0, 0, nullptr, 0};
  return run_prog(key, ws, d, st);
}

int lgm_grid_expm(const double* A, double* E, int64_t n, int64_t batch, int64_t ld, void* ws, cudaStream_t st) {
  LgmParams P{};
  CallDesc d = desc_base(P);
  d.A = A;
  d.L = E;
  d.ld = ld;
  GraphKey k{0, PROG_EXPM, (int)n, (int)batch, 0, 0, 0, nullptr, 0};
  return run_prog(k, ws, d, st);
}

size_t lgm_ws_guard_bytes() {
  static const size_t v = [] {  // thread-safe once-init
    const char* e = std::getenv("LGM_WS_GUARD");
    return (e && e[0] == '1') ? (size_t)4096 : (size_t)0;
  }();
  return v;
}

int lgm_grid_ws_guard(int64_t n, int64_t batch, void* ws, int check, unsigned long long* bad, cudaStream_t st) {
  if (!lgm_ws_guard_bytes()) return 0;
  ws_guard_kernel<<<256, 256, 0, st>>>((unsigned char*)ws, n, batch, lgm_ws_guard_bytes(), check, bad);
  CK(cudaGetLastError());
  return 1;
}

// kernels executed inside graphs on the current device (read back synchronously: stats only)
unsigned long long lgm_grid_exec_nodes() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_exec_nodes, sizeof(v)) != cudaSuccess) return 0;
  return v;
}

extern "C" int lgm_debug_g3_cycles(unsigned long long* out, int reset) {
#ifdef LGM_G3_PROF
  cudaMemcpyFromSymbol(out, g_g3_cyc, sizeof(g_g3_cyc));
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_g3_cyc, z, sizeof(z));
  }
  return 8;
#else
  (void)out; (void)reset;
  return 0;
#endif
}

extern "C" int lgm_debug_panel_cycles(unsigned long long* out) {
#ifdef LGM_PANEL_PROF
  cudaMemcpyFromSymbol(out, g_panel_cyc, sizeof(g_panel_cyc));  // 12 entries
  return 12;
#else
  (void)out;
  return 0;
#endif
}

// Engine G phase times (ns, accumulated on the current device; diagnostics): load, balance,
// alpha (scaling-loop estimates), DB (inversions + updates), select prep, select, poly, other.
extern "C" int lgm_debug_grid_phase_ns(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_phase_ns, sizeof(unsigned long long) * PH_N) != cudaSuccess) return -2;
  if (reset) {
    unsigned long long z[PH_N] = {};
    cudaMemcpyToSymbol(g_phase_ns, z, sizeof(z));
  }
  return PH_N;
}

// Inversion micro-benchmark (diagnostics; tools/inv_bench.py): the batched Gauss-Jordan of
// Engine G on 2*batch jobs (X and Y slots loaded from A), launched directly on `stream`
// (no graph, so ncu sees every kernel).  Each rep re-copies the inputs into the job slots.
extern "C" int lgm_debug_invert_f64(const double* A, int64_t n64, int64_t batch64, int reps, void* ws,
                                    cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  if (n <= 64 || !ws) return LGM_ERR_ARG;
  if (set_attrs(n)) return LGM_ERR_CUDA;
  CapStreams cs;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&cs.s[4], cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&cs.evN, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&cs.evP, cudaEventDisableTiming));
  Cap C;
  C.n = n;
  C.batch = batch;
  C.c = ctl_carve(ws, n, batch);
  for (int i = 0; i < 4; ++i) { C.s[i] = st; C.sB[i] = cs.s[4]; }
  C.evN = cs.evN;
  C.evP = cs.evP;
  C.itmax = 5;
  C.tma = g2_tma_on() && n <= 512 && n % (2 * NB) == 0 && !use_g1(n);
  if (C.tma && make_wmap(C)) return LGM_ERR_CUDA;
  CallDesc d = desc_base(LgmParams{});
  d.A = A;
  d.ld = n;
  setup_kernel<<<1, 1, 0, st>>>(C.c.desc, d);
  ctl_init_kernel<<<1, CT, 0, st>>>(C.c);
  load_kernel<<<ew_blocks(), 256, 0, st>>>(&C.c.desc->A, &C.c.desc->ld, C.c.S, C.c.list(LS_ALL), C.c.flag);
  ew_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_ALL), 1, G_Y, G_B, G_B);
  decide_live_kernel<<<1, CT, 0, st>>>(C.c);
  decide_db_start_kernel<<<1, CT, 0, st>>>(C.c);
  const bool oop = inv_oop(n);
  for (int r = 0; r < reps; ++r) {
    build_jobs_kernel<<<1, CT, 0, st>>>(C.c, 0, oop ? 1 : 0);
    if (!oop) {
      ew_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_DB), 1, G_XI, G_B, G_B);
      ew_kernel<<<ew_blocks(), 256, 0, st>>>(C.c.S, C.c.list(LS_DB), 1, G_YI, G_Y, G_Y);
    }
    if (cap_invert(C, st, 2 * batch)) return LGM_ERR_CUDA;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return 0;
}
