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

#include "lgm_grid.cuh"

namespace {

// Optional host-side phase timing (LGM_GRID_PROFILE=1): stream-synchronised wall time per
// phase, read back with lgm_debug_grid_phase_ms (tools/grid_prof.py).  Off by default.
enum { PH_BALANCE = 0, PH_ALPHA, PH_INVERT, PH_DBUPD, PH_SELECT, PH_POLY, PH_OTHER, PH_N };
double g_phase_ms[PH_N];
bool prof_on() {
  static const bool on = std::getenv("LGM_GRID_PROFILE") != nullptr;  // thread-safe once-init
  return on;
}
struct PhaseTimer {
  int ph;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  PhaseTimer(int p, cudaStream_t s) : ph(p), st(s) {
    if (prof_on()) { cudaStreamSynchronize(st); t0 = std::chrono::steady_clock::now(); }
  }
  ~PhaseTimer() {
    if (prof_on()) {
      cudaStreamSynchronize(st);
      g_phase_ms[ph] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  }
};

constexpr int NB = 32;      // Gauss-Jordan panel width
#ifndef G2_RT
#define G2_RT 64            // rows per tile of the rank-64 combined pass (64: 4 warps; 128 measured equal)
#endif
constexpr int NBUF = 8;     // n x n slots per matrix
enum { G_B = 0, G_Y, G_XI, G_YI, G_AP, G_AM, G_P6, G_P7 };

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

template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) gj_inv_cta_kernel(const InvJob* jobs, int n) {
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
        const double rp = lgm_rcp(wval[par * 16 + (p >> 5)]);
        double* pw = prow + par * 40;
        const bool own = (tid == p);
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
  double r[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) r[c] = (valid && c < nb) ? J.M[(size_t)row * n + k0 + c] : 0.0;
  bool used = valid ? (J.rowstep[row] >= 0) : true;
  bool piv_here = false;
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
      const unsigned long long wk = warp_max(pack(r0, valid && !used));
      if (lane == 0) s_wkey[par][warp] = wk;
      __syncthreads();
      const unsigned long long bk = warp_max(lane < 16 ? s_wkey[par][lane] : 0ull);
      const int brow = 4095 - (int)(bk & 0xfffu);
      if (tid == 0) s_key[par] = bk;
      if (bk != 0ull && valid && row == brow) {  // publish this CTA's candidate row
#pragma unroll
        for (int c = 0; c < 32; ++c) s_cand[par][c] = r[c];
      }
      cl.sync();
      // cluster winner: lanes q < CL of every warp read CTA q's key over DSMEM
      const unsigned long long ck = warp_max(lane < CL ? *cl.map_shared_rank(&s_key[par], lane) : 0ull);
      if (ck == 0ull) { status = 1; break; }  // exact zero pivot (matcore.py:124-125)
      const int p = 4095 - (int)(ck & 0xfffu);
      if (tid < 32) s_prow[par][tid] = cl.map_shared_rank(&s_cand[par][0], p / rpc)[tid];
      __syncthreads();
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
}

#ifdef LGM_PANEL_PROF
__device__ unsigned long long g_panel_cyc[6];  // load, stage-1, factor, store, CTAs
#define PP_T(v) long long v = clock64()
#define PP_ADD(i, val) if (threadIdx.x == 0) atomicAdd(&g_panel_cyc[i], (unsigned long long)(val))
#else
#define PP_T(v)
#define PP_ADD(i, val)
#endif
// G2 panel for n <= 512 (many jobs): one CTA of NT >= n threads per inversion, row `tid`
// of the 32-column panel in registers, the pivot rule and shift-in-FMA frame of G1
// (gj_inv_cta_kernel).  No cluster: with hundreds of jobs the 8-CTA cluster panel's
// per-step cluster barriers serialise into many waves.
template <int NT>
// s1_a1kind >= 0 (P2 of a rank-64 pair): the stage-1 update of P2's columns by P1 is applied
// to the loaded rows first (r <- z1 r + A1 W1[:, P2], FMA chain in c' order), replacing the
// narrow gj_update_kernel launch and its snapshot.
__global__ void __launch_bounds__(NT, 512 / NT) gj_panel_cta_kernel(const InvJob* jobs, int n, int k0, int nb, int a1_kind,
                                                                   int s1_a1kind) {
  constexpr int NW = NT / 32;
  __shared__ __align__(16) double prow[2][40];
  __shared__ unsigned wkey32[2][16];
  __shared__ double wval[2][16];
  __shared__ double red[16];
  __shared__ int piv_s[32];
  const InvJob J = jobs[blockIdx.x];
  if (*J.status) return;  // uniform per CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 80) (&prow[0][0])[tid] = 0.0;  // pure-rotation steps read it with g = 0
  PP_T(t0);
  bool used = tid < n ? (J.rowstep[tid] >= 0) : true;
  double r[32];
  double* M = J.M;
  // full panels move through a per-warp 32 x 33 shared tile: the warp reads / writes its 32
  // rows' 256-byte segments coalesced (one row per instruction) instead of one strided
  // 256-byte segment per lane
  extern __shared__ __align__(16) double ptile[];
  double* T = ptile + warp * 32 * 33;
  const bool tiled = nb == 32 && (n & 31) == 0;
  if (tiled) {
    if (warp * 32 < n) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) r[rr] = M[(size_t)(warp * 32 + rr) * n + k0 + lane];  // all in flight
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) T[rr * 33 + lane] = r[rr];
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = T[lane * 33 + c];
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = 0.0;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      if (tid < n && c + 1 < nb && (n & 1) == 0) {
        const double2 v = *reinterpret_cast<const double2*>(&M[(size_t)tid * n + k0 + c]);
        r[c] = v.x;
        r[c + 1] = v.y;
      } else {
        r[c] = (tid < n && c < nb) ? M[(size_t)tid * n + k0 + c] : 0.0;
        r[c + 1] = (tid < n && c + 1 < nb) ? M[(size_t)tid * n + k0 + c + 1] : 0.0;
      }
    }
  }
  __syncthreads();
  PP_T(t1);
  PP_ADD(0, t1 - t0);
  if (s1_a1kind >= 0) {
    __shared__ __align__(16) double w1s[32][34];
    const int p1 = k0 - NB;
    for (int idx = tid; idx < 32 * 32; idx += NT) {
      const int c1 = idx >> 5, c = idx & 31;
      w1s[c1][c] = M[(size_t)J.piv[p1 + c1] * n + k0 + c];
    }
    __syncthreads();
    if (tid < n) {
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
      __syncthreads();
      const unsigned bk = __reduce_max_sync(0xffffffffu, lane < NW ? wkey32[par][lane] : 0u);
      if (bk == 0u) {  // exact zero pivot (matcore.py:124-125)
        if (tid == 0) *J.status = 1;
        return;
      }
      const int p = 1023 - (int)(bk & 0x3ffu);
      const double rp = lgm_rcp(wval[par][p >> 5]);
      const bool own = (tid == p);
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
__global__ void __launch_bounds__(128) gj_w2_mma_kernel(const InvJob* jobs, int n, int k0, int q) {
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
  for (int idx = tid; idx < NB * NB; idx += 128) {
    const int c = idx >> 5, cc = idx & 31;
    a1s[c][cc] = A1[(size_t)p2s[c] * NB + cc];
  }
  for (int idx = tid; idx < NB * 32; idx += 128) {  // W1 rows, 16-byte chunks
    const int cc = idx >> 5, jj = (idx & 31) * 2;
    const int j = j0 + jj;
    double2 v = *reinterpret_cast<const double2*>(&J.M[(size_t)p1s[cc] * n + j]);
    if (j >= k0 && j < k0 + NB) v = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(&w1s[cc][jj]) = v;
    *reinterpret_cast<double2*>(&W1[(size_t)cc * n + j]) = v;
  }
  __syncthreads();
  const int g8 = lane >> 2, t4 = lane & 3, wc = warp * 16;
  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(&J.M[(size_t)p2s[mi * 8 + g8] * n + j0 + wc + ni * 8 + 2 * t4]);
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
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
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int c = mi * 8 + g8;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int j = j0 + wc + ni * 8 + 2 * t4;  // j, j + 1 on the same side of 32-aligned bounds
      double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      if (j >= k0 && j < k0 + NB) v = make_double2(a1s[c][j - k0], a1s[c][j + 1 - k0]);
      else if (j >= k0 + NB && j < k0 + 2 * NB) v = make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(&W2[(size_t)c * n + j]) = v;
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
  const InvJob J = jobs[blockIdx.z];
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
      const double2 v = *reinterpret_cast<const double2*>(&J.M[(size_t)i * n + j]);
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

// ------------------------------------------------------------------------------------------
// Elementwise / reduction kernels over a list of matrices (index list `ids`).
struct Slots {
  double* ws;       // base of the n x n slots
  int n;
  __device__ __host__ double* buf(int b, int k) const { return ws + ((size_t)b * NBUF + k) * (size_t)n * n; }
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
__global__ void onenorm_kernel(Slots S, DList L, int k, double* out) {
  const int n = S.n;
  LIST_LOOP(L, (size_t)n)
    const double* M = S.buf(b, k);
    const int j = (int)idx;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = (i == 0) ? fabs(M[(size_t)i * n + j]) : acc + fabs(M[(size_t)i * n + j]);
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

__global__ void __launch_bounds__(1024) balance_kernel_g(Slots S, DList L, double* scale, int* sweeps_out,
                                                        int max_sweeps, double* margin) {
  if (blockIdx.x >= *L.cnt) return;
  const int b = L.ids[blockIdx.x];
  const int n = S.n;
  double* B = S.buf(b, G_B);
  double* sc = scale + (size_t)b * n;
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
  for (int i = threadIdx.x; i < n; i += blockDim.x) sc[i] = 1.0;
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
        const double* p = which == 0 ? B + (size_t)loff[q] * n + i : B + (size_t)i * n + loff[q];
        const size_t stride = which == 0 ? (size_t)n : 1;
        const int m8 = len - len % 8;
        double r;
        if (m8 == 128) {  // full leaf: all 16 loads in flight, then the in-order sum
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = fabs(p[(a + 8 * u) * stride]);
          r = v[0];
#pragma unroll
          for (int u = 1; u < 16; ++u) r += v[u];
        } else {
          r = fabs(p[a * stride]);
          for (int k = 8 + a; k < m8; k += 8) r += fabs(p[k * stride]);
        }
        lacc_dyn[which * nleaf * 8 + rem] = r;
      }
      __syncthreads();
      for (int l = threadIdx.x; l < 2 * nleaf; l += blockDim.x) {
        const int which = l / nleaf, q = l - which * nleaf;
        const int len = llen[q];
        const double* p = which == 0 ? B + (size_t)loff[q] * n + i : B + (size_t)i * n + loff[q];
        const size_t stride = which == 0 ? (size_t)n : 1;
        double res;
        if (len < 8) {
          res = 0.0;
          for (int k = 0; k < len; ++k) res += fabs(p[k * stride]);
        } else {
          const double* r = &lacc_dyn[which * nleaf * 8 + q * 8];
          res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
          for (int k = len - len % 8; k < len; ++k) res += fabs(p[k * stride]);
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
        double dg = fabs(B[(size_t)i * n + i]);
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
        for (int q = threadIdx.x; q < n; q += blockDim.x) B[(size_t)q * n + i] *= f;
        __syncthreads();
        for (int q = threadIdx.x; q < n; q += blockDim.x) B[(size_t)i * n + q] *= inv;
        if (threadIdx.x == 0) sc[i] *= f;
        moved = true;
      }
      __syncthreads();
    }
    if (!moved) break;
  }
  if (threadIdx.x == 0) { sweeps_out[b] = sweeps; margin[b] = s_mm; }
}

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
};

__global__ void __launch_bounds__(128) db_update_kernel(DbArgs a) {
  if (blockIdx.y >= *a.L.cnt) return;
  const int b = a.L.ids[blockIdx.y];
  const int n = a.S.n;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (a.istat[b] || (!a.first && a.istat[a.batch + b])) return;  // singular iterate: X, Y kept
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
  double* V0;         // ping
  double* V1;         // pong
  double* part;       // adjoint partial sums [splits][2][n]
  int* hist;          // [16]
  // state
  double est;
  int best_j, ncols, done, nhist, passes, total;
  double mm;
};

__global__ void est_init_kernel(EstJob* jobs, int n, double rsum) {
  EstJob& J = jobs[blockIdx.y];
  const int t = n < 2 ? n : 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    J.V0[i] = 1.0 / n;
    if (t > 1) J.V0[n + i] = (((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))) / rsum;
  }
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
__global__ void __launch_bounds__(256) est_fwd_kernel(EstJob* jobs, int n, int q) {
  EstJob& J = jobs[blockIdx.y];
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
__global__ void __launch_bounds__(128) est_adj_kernel(EstJob* jobs, int n, int q) {
  EstJob& J = jobs[blockIdx.z];
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
__global__ void __launch_bounds__(128) est_adj2_kernel(EstJob* jobs, int n, int q) {
  EstJob& J = jobs[blockIdx.z];
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
__device__ void est_after_fwd_body(EstJob& J, int n, int sweep, double* sred) {
  if (J.done) return;
  double* Yv = (J.total & 1) ? J.V1 : J.V0;
  const int nc = J.ncols;
  double cn[2] = {0.0, 0.0};
  for (int c = 0; c < nc; ++c) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += fabs(Yv[c * n + i]);
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
  if (!stop) {  // S = sign(Y) in place (matcore.py:231); the adjoint reads it as step 0 input
    for (int c = 0; c < nc; ++c)
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double v = Yv[c * n + i];
        double s = (v >= 0.0) ? 1.0 : -1.0;
        // adjoint starts from V0: move if the forward result landed in V1
        if (J.total & 1) J.V0[c * n + i] = s;
        else Yv[c * n + i] = s;
      }
  }
}
__global__ void __launch_bounds__(256) est_after_fwd_kernel(EstJob* jobs, int n, int sweep) {
  __shared__ double sred[8];
  est_after_fwd_body(jobs[blockIdx.x], n, sweep, sred);
}

// After the adjoint: h = row max |Z|, top-(4t+1) order, picks, stopping test, next X.
struct EstAdjSmem {
  uint64_t skey[8];
  int sidx[8];
  int order[9];
  double hval[9];
};
__device__ void est_after_adj_body(EstJob& J, int n, int sweep, EstAdjSmem& sa) {
  uint64_t* skey = sa.skey;
  int* sidx = sa.sidx;
  int* order = sa.order;
  double* hval = sa.hval;
  if (J.done) return;
  const double* Z = (J.total & 1) ? J.V1 : J.V0;
  const int nc = J.ncols;
  const int t = n < 2 ? n : 2;
  const int ntop = n < 4 * t + 1 ? n : 4 * t + 1;
  // repeated block argmax over h with exclusion of already taken rows
  for (int qq = 0; qq < ntop; ++qq) {
    uint64_t key = 0ull;
    int idx = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      bool taken = false;
      for (int u = 0; u < qq; ++u) taken |= (order[u] == i);
      if (taken) continue;
      double h = fabs(Z[i]);
      if (nc > 1) h = fmax(h, fabs(Z[n + i]));
      uint64_t kq = dkey(h);
      if (kq > key) { key = kq; idx = i; }
    }
    uint64_t kmax;
    int p;
    block_argmax(key, idx, skey, sidx, kmax, p);
    if (threadIdx.x == 0) { order[qq] = p; hval[qq] = __longlong_as_double((long long)(kmax - 1ull)); }
    __syncthreads();
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
    auto hrow = [&](int i) { double h = fabs(Z[i]); if (nc > 1) h = fmax(h, fabs(Z[n + i])); return h; };
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
__global__ void __launch_bounds__(256) est_after_adj_kernel(EstJob* jobs, int n, int sweep) {
  __shared__ EstAdjSmem sa;
  est_after_adj_body(jobs[blockIdx.x], n, sweep, sa);
}

// The whole estimate for one job per CTA (256 threads), M1 resident in shared memory
// (n <= EST_FUSED_MAXN): one launch instead of 1 + itmax (2 total + 2) per-step launches.
// Every reduction reproduces the per-step kernels' order exactly (forward: warp per row,
// lane-strided FMAs + butterfly; adjoint: thread per column, 64-row slabs with 4 accumulators,
// slab partials summed in order; the after-bodies are shared), so the two paths agree bit for bit.
constexpr int EST_FUSED_MAXN = 160;
__global__ void __launch_bounds__(256) est_fused_kernel(EstJob* jobs, int n, double rsum, int itmax) {
  extern __shared__ __align__(16) double Ms[];
  __shared__ double sred[8];
  __shared__ EstAdjSmem sa;
  EstJob& J = jobs[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {  // est_init_kernel
    const int t = n < 2 ? n : 2;
    for (int i = tid; i < n; i += 256) {
      J.V0[i] = 1.0 / n;
      if (t > 1) J.V0[n + i] = (((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))) / rsum;
    }
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
    est_after_fwd_body(J, n, sweep, sred);
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
    est_after_adj_body(J, n, sweep, sa);
    __syncthreads();
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

// ------------------------------------------------------------------------------------------
// Host side
double host_pairwise_abs_ramp(int n) {
  // numpy pairwise sum of |(-1)^i (1 + i/max(1, n-1))| (matcore.py:270-271)
  auto get = [n](int i) { return std::fabs(((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))); };
  return lgm_pairwise_sum(get, n);
}

struct Grid {
  int n = 0, batch = 0;
  cudaStream_t st = nullptr;
  Slots S{};
  // device arrays
  int* d_ids = nullptr;       // [batch] scratch id list
  int* d_piv = nullptr;       // [2][batch][n]
  int* d_step = nullptr;      // [2][batch][n]
  double* d_W = nullptr;      // [6 kinds][2][batch][NB*n]
  cudaStream_t sB = nullptr;  // G2 look-ahead: panel stream (higher priority)
  cudaEvent_t evN = nullptr, evP = nullptr;
  ~Grid() {
    if (sB) cudaStreamDestroy(sB);
    if (evN) cudaEventDestroy(evN);
    if (evP) cudaEventDestroy(evP);
  }
  double* d_logdet = nullptr; // [2][batch]
  int* d_istat = nullptr;     // [2][batch]
  std::vector<InvJob> jobs_up;  // host copy of the job table last uploaded to d_jobs
  InvJob* d_jobs = nullptr;   // [2*batch]
  double* d_scal = nullptr;   // [batch] scratch doubles
  double* d_scal2 = nullptr;
  int* d_iflag = nullptr;     // [batch]
  int* d_scaling = nullptr;   // [batch]
  double* d_scale = nullptr;  // [batch][n] balancing scales
  double* d_margin = nullptr; // [batch]
  int* d_sweeps = nullptr;    // [batch]
  EstJob* d_est = nullptr;    // [batch]
  double* d_vec = nullptr;    // [batch][2 vectors][2n]
  double* d_part = nullptr;   // [batch][splits][2][n]
  int* d_hist = nullptr;      // [batch][16]
  int splits = 1;

  static size_t bytes(int64_t n, int64_t batch) {
    int64_t splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
    size_t s = 0;
    auto add = [&](size_t b) { s += (b + 255) & ~size_t(255); };
    add((size_t)batch * NBUF * n * n * 8);
    add(batch * 4);
    add(2 * batch * n * 4);
    add(2 * batch * n * 4);
    add(12 * batch * NB * n * 8);
    add(2 * batch * 8);
    add(2 * batch * 4);
    add(2 * batch * sizeof(InvJob));
    add(batch * 8);
    add(batch * 8);
    add(batch * 4);
    add(batch * 4);
    add(batch * n * 8);
    add(batch * 8);
    add(batch * 4);
    add(batch * sizeof(EstJob));
    add(batch * 4 * n * 8);
    add(batch * splits * 2 * n * 8);
    add(batch * 16 * 4);
    return s;
  }

  void carve(void* ws, int n_, int batch_) {
    n = n_;
    batch = batch_;
    splits = (n + ADJ_ROWS - 1) / ADJ_ROWS;
    char* p = (char*)ws;
    auto take = [&](size_t b) { char* r = p; p += (b + 255) & ~size_t(255); return (void*)r; };
    S.ws = (double*)take((size_t)batch * NBUF * n * n * 8);
    S.n = n;
    d_ids = (int*)take(batch * 4);
    d_piv = (int*)take(2 * (size_t)batch * n * 4);
    d_step = (int*)take(2 * (size_t)batch * n * 4);
    d_W = (double*)take(12 * (size_t)batch * NB * n * 8);
    d_logdet = (double*)take(2 * batch * 8);
    // d_scal, d_scal2, d_istat adjacent: the DB step reads all three back in one copy
    d_scal = (double*)take(batch * 8);
    d_scal2 = (double*)take(batch * 8);
    d_istat = (int*)take(2 * batch * 4);
    d_jobs = (InvJob*)take(2 * batch * sizeof(InvJob));
    d_iflag = (int*)take(batch * 4);
    d_scaling = (int*)take(batch * 4);
    d_scale = (double*)take((size_t)batch * n * 8);
    d_margin = (double*)take(batch * 8);
    d_sweeps = (int*)take(batch * 4);
    d_est = (EstJob*)take(batch * sizeof(EstJob));
    d_vec = (double*)take((size_t)batch * 4 * n * 8);
    d_part = (double*)take((size_t)batch * splits * 2 * n * 8);
    d_hist = (int*)take(batch * 16 * 4);
  }

  dim3 ew_grid(int count) const {
    size_t nn = (size_t)n * n;
    int bx = (int)std::min<size_t>((nn + 255) / 256, 1024);
    return dim3(bx, count);
  }

  int upload_ids(const std::vector<int>& ids) {
    CK(cudaMemcpyAsync(d_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st));
    return 0;
  }

  // ---- batched inversion of slot `k` of the listed matrices (jobs: which = 0 for X, 1 for Y)
  template <int NT>
  int launch_g1(int nj) {
    const size_t sm = G1Smem<NT>::bytes;
    CK(cudaFuncSetAttribute(gj_inv_cta_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    lgm_count_launch(), gj_inv_cta_kernel<NT><<<nj, NT, sm, st>>>(d_jobs, n);
    CK(cudaGetLastError());
    return 0;
  }

  int invert(const std::vector<int>& mats, const std::vector<int>& which, const std::vector<int>& slot,
             const std::vector<int>* src_slot = nullptr) {
    const int nj = (int)mats.size();
    if (!nj) return 0;
    std::vector<InvJob> jobs(nj);
    for (int q = 0; q < nj; ++q) {
      int b = mats[q], w = which[q];
      InvJob& J = jobs[q];
      J.M = S.buf(b, slot[q]);
      J.Src = (src_slot && use_g1(n)) ? S.buf(b, (*src_slot)[q]) : nullptr;
      J.piv = d_piv + ((size_t)w * batch + b) * n;
      J.rowstep = d_step + ((size_t)w * batch + b) * n;
      J.Wb = d_W + ((size_t)w * batch + b) * NB * n;
      J.wst = (long long)2 * batch * NB * n;
      J.logdet = d_logdet + w * batch + b;
      J.status = d_istat + w * batch + b;
    }
    // the job table only changes with the active set: skip the (pageable, host-blocking)
    // re-upload between DB steps when it is byte-identical to the last one
    if (jobs_up.size() != jobs.size() || std::memcmp(jobs_up.data(), jobs.data(), nj * sizeof(InvJob)) != 0) {
      CK(cudaMemcpyAsync(d_jobs, jobs.data(), nj * sizeof(InvJob), cudaMemcpyHostToDevice, st));
      jobs_up = jobs;
    }
    if (use_g1(n)) {  // G1: one CTA per inversion, no per-panel launches
      if (n <= 128) return launch_g1<128>(nj);
      if (n <= 256) return launch_g1<256>(nj);
      return launch_g1<512>(nj);
    }
    lgm_count_launch(), gj_init_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(d_jobs, n);
    const int tiles = (n + TM - 1) / TM;
    const bool cta_panel = n <= 512;  // one CTA per panel (writes A1 itself: no gj_copy_a1_kernel)
    // dynamic shared memory limits are per device: set them on every call (no process-wide flag)
    if (n <= 128) CK(cudaFuncSetAttribute(gj_panel_cta_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 33 * 8));
    else if (n <= 256) CK(cudaFuncSetAttribute(gj_panel_cta_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 33 * 8));
    else if (n <= 512) CK(cudaFuncSetAttribute(gj_panel_cta_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 32 * 33 * 8));
    auto panel = [&](int k0, cudaStream_t s, int a1_kind = -1, int s1_a1kind = -1) {
      const int nb = std::min(NB, n - k0);
      if (n <= 128) {  // many small jobs: one CTA per inversion, no cluster
        lgm_count_launch(), gj_panel_cta_kernel<128><<<nj, 128, 4 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
      } else if (n <= 256) {
        lgm_count_launch(), gj_panel_cta_kernel<256><<<nj, 256, 8 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
      } else if (n <= 512) {
        lgm_count_launch(), gj_panel_cta_kernel<512><<<nj, 512, 16 * 32 * 33 * 8, s>>>(d_jobs, n, k0, nb, a1_kind, s1_a1kind);
      } else if (n <= CL * 512) {  // G2 panel: one 8-CTA cluster per inversion
        lgm_count_launch(), gj_panel_cluster_kernel<<<nj * CL, 512, 0, s>>>(d_jobs, n, k0, nb);
      } else {
        lgm_count_launch(), gj_panel_kernel<<<nj, 512, 0, s>>>(d_jobs, n, k0, nb, 0);
      }
    };
    auto snapshot = [&](int k0, int kind, int jlo = 0, int jhi = -1, cudaStream_t s = nullptr) {
      const int nb = std::min(NB, n - k0);
      if (jhi < 0) jhi = n;
      lgm_count_launch(), gj_snapshot_kernel<<<dim3((nb * (jhi - jlo) + 255) / 256, nj), 256, 0, s ? s : st>>>(
                              d_jobs, n, k0, nb, kind, jlo, jhi);
    };
    // Look-ahead: panel k+1 is factored on a second (higher-priority) stream while the
    // trailing update of panel k runs on `st`.  Per panel k: the next panel's columns are
    // updated first (narrow launch), then its factorisation is released to sB, then the
    // full update skips both panels; the snapshot of panel k+1's pivot rows waits for both.
    if (!sB) {
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&sB, cudaStreamNonBlocking, hi));
      CK(cudaEventCreateWithFlags(&evN, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&evP, cudaEventDisableTiming));
    }
    static const bool rank64 = [] {  // LGM_G2_RANK64=0 falls back to rank-32 passes (A/B switch)
      const char* e = std::getenv("LGM_G2_RANK64");
      return !(e && e[0] == '0');
    }();
    // rank-64 vs rank-32 passes round differently: the choice depends on n only, so a
    // matrix's arithmetic never depends on its batch-mates or on how many have converged
    const bool use64 = rank64 && n % (2 * NB) == 0;
    panel(0, st, use64 && cta_panel ? 2 : -1);
    if (use64) {
      // rank-64 delayed update with both panels of the next pair factored on sB during the
      // current combined pass.  Per pair (P1, P2) in buffer set q: W1 (snapshot of P1's pivot
      // rows), A1 (copy of P1's multipliers), stage-1 update of P2's columns, factor P2, W2.
      CK(cudaFuncSetAttribute(gj_update2_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)up2_smem<64>()));
      CK(cudaFuncSetAttribute(gj_update2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)up2_smem<128>()));
      auto prepare_pair = [&](int k0, int q, cudaStream_t s, bool full_snapshot) {
        // P1 = [k0, k0+NB) already factored; everything except the full-width W1 / W2
        if (cta_panel) {  // stage-1 update fused into P2's panel kernel
          panel(k0 + NB, s, -1, 3 * q + 2);
          return;
        }
        if (full_snapshot) snapshot(k0, 3 * q, 0, n, s);
        else snapshot(k0, 3 * q, k0 + NB, k0 + 2 * NB, s);  // P2's columns only (for stage 1)
        if (!cta_panel)
          lgm_count_launch(), gj_copy_a1_kernel<<<dim3((n * NB + 255) / 256, nj), 256, 0, s>>>(d_jobs, n, k0, 3 * q + 2);
        lgm_count_launch(), gj_update_kernel<<<dim3(1, tiles, nj), 128, 0, s>>>(d_jobs, n, k0, NB, k0 + NB, k0 + NB,
                                                                               k0 + 2 * NB, 0, 0, 3 * q);
        panel(k0 + NB, s);
      };
      prepare_pair(0, 0, st, !cta_panel);
      if (cta_panel) lgm_count_launch(), gj_w2_mma_kernel<<<dim3(n / 64, nj), 128, 0, st>>>(d_jobs, n, 0, 0);
      else lgm_count_launch(), gj_w2_kernel<<<dim3((n + 127) / 128, nj), 128, 0, st>>>(d_jobs, n, 0, 0, 0);
      for (int k0 = 0, q = 0; k0 < n; k0 += 2 * NB, q ^= 1) {
        const int kn = k0 + 2 * NB;
        const bool next = kn < n;
        if (next) {  // finish the next pair's columns, then factor both of its panels on sB
          lgm_count_launch(), gj_update2_kernel<64><<<dim3(1, tiles, nj), 128, up2_smem<64>(), st>>>(d_jobs, n, k0, kn, kn,
                                                                                           kn + 2 * NB, 0, 0, q);
          CK(cudaEventRecord(evN, st));
          CK(cudaStreamWaitEvent(sB, evN, 0));
          panel(kn, sB, cta_panel ? 3 * (q ^ 1) + 2 : -1);
          prepare_pair(kn, q ^ 1, sB, false);
          CK(cudaEventRecord(evP, sB));
        }
        lgm_count_launch(), gj_update2_kernel<G2_RT><<<dim3(tiles, n / G2_RT, nj), 2 * G2_RT, up2_smem<G2_RT>(), st>>>(
                                d_jobs, n, k0, 0, 0, n, next ? kn : 0, next ? kn + 2 * NB : 0, q);
        if (next) {  // full-width W1 / W2 of the next pair need this pass's rows
          CK(cudaStreamWaitEvent(st, evP, 0));
          if (cta_panel) {
            lgm_count_launch(), gj_w2_mma_kernel<<<dim3(n / 64, nj), 128, 0, st>>>(d_jobs, n, kn, q ^ 1);
          } else {
            snapshot(kn, 3 * (q ^ 1));
            lgm_count_launch(), gj_w2_kernel<<<dim3((n + 127) / 128, nj), 128, 0, st>>>(d_jobs, n, kn, q ^ 1, 0);
          }
        }
      }
      CK(cudaGetLastError());
      return 0;
    }
    snapshot(0, 0);
    for (int k0 = 0, par = 0; k0 < n; k0 += NB, par ^= 1) {
      const int nb = std::min(NB, n - k0);
      const int kn = k0 + NB, nbn = kn < n ? std::min(NB, n - kn) : 0;
      if (kn < n) {
        lgm_count_launch(), gj_update_kernel<<<dim3(1, tiles, nj), 128, 0, st>>>(d_jobs, n, k0, nb, kn, kn, kn + nbn, 0, 0,
                                                                                par);
        CK(cudaEventRecord(evN, st));
        CK(cudaStreamWaitEvent(sB, evN, 0));
        panel(kn, sB);
        CK(cudaEventRecord(evP, sB));
      }
      lgm_count_launch(), gj_update_kernel<<<dim3(tiles, tiles, nj), 128, 0, st>>>(d_jobs, n, k0, nb, 0, 0, n, kn,
                                                                                   kn + nbn, par);
      if (kn < n) {
        CK(cudaStreamWaitEvent(st, evP, 0));
        snapshot(kn, par ^ 1);
      }
    }
    CK(cudaGetLastError());
    return 0;
  }

  // ---- batched estimator: est[q] for the listed jobs (operator M1^p1 * M2)
  int estimate(const std::vector<const double*>& M1, const std::vector<int>& p1, const std::vector<const double*>& M2,
               const std::vector<int>& zero, int itmax, std::vector<double>& est, std::vector<int>& passes,
               std::vector<double>& mm) {
    const int nj = (int)M1.size();
    est.assign(nj, 0.0);
    passes.assign(nj, 0);
    mm.assign(nj, INFINITY);
    if (!nj) return 0;
    std::vector<EstJob> jobs(nj);
    int maxtot = 0;
    for (int q = 0; q < nj; ++q) {
      EstJob& J = jobs[q];
      std::memset(&J, 0, sizeof(J));
      J.M1 = M1[q];
      J.M2 = M2[q];
      J.p1 = p1[q];
      J.zero = zero[q];
      J.V0 = d_vec + (size_t)q * 4 * n;
      J.V1 = J.V0 + 2 * n;
      J.part = d_part + (size_t)q * splits * 2 * n;
      J.hist = d_hist + q * 16;
      maxtot = std::max(maxtot, p1[q] + (M2[q] ? 1 : 0));
    }
    CK(cudaMemcpyAsync(d_est, jobs.data(), nj * sizeof(EstJob), cudaMemcpyHostToDevice, st));
    const double rsum = host_pairwise_abs_ramp(n);
    if (n <= EST_FUSED_MAXN && est_fused_on()) {
      const int sm = n * n * 8;
      CK(cudaFuncSetAttribute(est_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      lgm_count_launch(), est_fused_kernel<<<nj, 256, sm, st>>>(d_est, n, rsum, itmax);
    } else {
    lgm_count_launch(), est_init_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(d_est, n, rsum);
    for (int sweep = 0; sweep < itmax; ++sweep) {
      for (int q = 0; q < maxtot; ++q)
        lgm_count_launch(), est_fwd_kernel<<<dim3((n + 8 * EST_FWD_R - 1) / (8 * EST_FWD_R), nj), 256, 0, st>>>(d_est, n, q);
      lgm_count_launch(), est_after_fwd_kernel<<<nj, 256, 0, st>>>(d_est, n, sweep);
      for (int q = 0; q < maxtot; ++q) {
        if ((n & 1) == 0) lgm_count_launch(), est_adj2_kernel<<<dim3((n + 255) / 256, splits, nj), 128, 0, st>>>(d_est, n, q);
        else lgm_count_launch(), est_adj_kernel<<<dim3((n + 127) / 128, splits, nj), 128, 0, st>>>(d_est, n, q);
        lgm_count_launch(), est_adj_reduce_kernel<<<dim3((n + 255) / 256, nj), 256, 0, st>>>(d_est, n, q, splits);
      }
      lgm_count_launch(), est_after_adj_kernel<<<nj, 256, 0, st>>>(d_est, n, sweep);
    }
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(jobs.data(), d_est, nj * sizeof(EstJob), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int q = 0; q < nj; ++q) {
      est[q] = jobs[q].est;
      passes[q] = jobs[q].passes;
      mm[q] = jobs[q].mm;
    }
    return 0;
  }

  int onenorms(const std::vector<int>& mats, int k, std::vector<double>& out) {
    const int c = (int)mats.size();
    out.assign(batch, 0.0);
    if (!c) return 0;
    if (upload_ids(mats)) return LGM_ERR_CUDA;
    CK(cudaMemsetAsync(d_scal, 0, batch * 8, st));
    lgm_count_launch(), onenorm_kernel<<<dim3((n + 127) / 128, c), 128, 0, st>>>(S, d_ids, k, d_scal);
    CK(cudaMemcpyAsync(out.data(), d_scal, batch * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
  }

  int any_nonzero(const std::vector<int>& mats, int k, std::vector<int>& out) {
    out.assign(batch, 0);
    if (mats.empty()) return 0;
    if (upload_ids(mats)) return LGM_ERR_CUDA;
    CK(cudaMemsetAsync(d_iflag, 0, batch * 4, st));
    lgm_count_launch(), any_nonzero_kernel<<<ew_grid((int)mats.size()), 256, 0, st>>>(S, d_ids, k, d_iflag);
    CK(cudaMemcpyAsync(out.data(), d_iflag, batch * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
  }

  // plain C = A * B over the matrices in d_ids (first `count`), n even
  int gemm_plain(int count, int ak, int bk, int ck) {
    const size_t sm = 2 * (size_t)(GP_A + GP_B) * 8;
    CK(cudaFuncSetAttribute(gemm_plain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int tiles = (n + TM - 1) / TM;
    lgm_count_launch(), gemm_plain_kernel<<<dim3(tiles, tiles, count), 128, sm, st>>>(S, d_ids, ak, bk, ck);
    CK(cudaGetLastError());
    return 0;
  }

  int ew(const std::vector<int>& mats, int op, int dk, int sk, int s2k) {
    if (mats.empty()) return 0;
    if (upload_ids(mats)) return LGM_ERR_CUDA;
    lgm_count_launch(), ew_kernel<<<ew_grid((int)mats.size()), 256, 0, st>>>(S, d_ids, op, dk, sk, s2k);
    CK(cudaGetLastError());
    return 0;
  }

  // ---- scaled DB square root of slot G_B for the listed matrices (sqrtm.py:27-78)
  // Returns per-matrix status (0 / LGM_SINGULAR / LGM_DB_NOCONV) and iterations.
  int sqrt_db(const std::vector<int>& mats, double tol_in, int maxiter, std::vector<int>& status,
              std::vector<int>& iters, std::vector<double>& mm, std::vector<int>& plateau) {
    std::vector<int> act = mats;
    std::vector<int> scaling(batch, 1);
    if (ew(act, 2, G_Y, G_Y, G_Y)) return LGM_ERR_CUDA;  // Y = I
    for (int it = 1; it <= maxiter && !act.empty(); ++it) {
      // inversions of X -> XI (all) and Y -> YI (it > 1): out of place inside G1 (n <= 512),
      // else copy then invert in place
      const bool oop = use_g1(n);
      if (!oop) {
        if (ew(act, 1, G_XI, G_B, G_B)) return LGM_ERR_CUDA;
        if (it > 1 && ew(act, 1, G_YI, G_Y, G_Y)) return LGM_ERR_CUDA;
      }
      std::vector<int> mats2, which, slot, src;
      for (int b : act) { mats2.push_back(b); which.push_back(0); slot.push_back(G_XI); src.push_back(G_B); }
      if (it > 1)
        for (int b : act) { mats2.push_back(b); which.push_back(1); slot.push_back(G_YI); src.push_back(G_Y); }
      {
        PhaseTimer pt(PH_INVERT, st);
        if (invert(mats2, which, slot, oop ? &src : nullptr)) return LGM_ERR_CUDA;
      }
      // (the singular flags are read back together with the norms below: one sync per iteration)
      // update + norms
      std::vector<int> hs(batch);
      for (int b = 0; b < batch; ++b) hs[b] = scaling[b];
      CK(cudaMemcpyAsync(d_scaling, hs.data(), batch * 4, cudaMemcpyHostToDevice, st));
      if (upload_ids(act)) return LGM_ERR_CUDA;
      if (it == 1) CK(cudaMemsetAsync(d_logdet + batch, 0, batch * 8, st));
      CK(cudaMemsetAsync(d_scal, 0, batch * 8, st));
      CK(cudaMemsetAsync(d_scal2, 0, batch * 8, st));
      DbArgs a;
      a.S = S;
      a.ids = d_ids;
      a.xpiv = d_piv;
      a.xstep = d_step;
      a.ypiv = d_piv + (size_t)batch * n;
      a.ystep = d_step + (size_t)batch * n;
      a.xlog = d_logdet;
      a.ylog = d_logdet + batch;
      a.scaling = d_scaling;
      a.first = it == 1;
      a.change = d_scal;
      a.size = d_scal2;
      a.istat = d_istat;
      a.batch = batch;
      PhaseTimer pt(PH_DBUPD, st);
      lgm_count_launch(), db_update_kernel<<<dim3((n + 127) / 128, (int)act.size()), 128, 0, st>>>(a);
      CK(cudaGetLastError());
      // change, size and the singular flags in one device-to-host copy (adjacent in the carve)
      const char* span0 = (const char*)d_scal;
      const size_t span = (size_t)((const char*)(d_istat + 2 * batch) - span0);
      std::vector<char> rb(span);
      CK(cudaMemcpyAsync(rb.data(), span0, span, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<double> ch(batch), sz(batch);
      std::vector<int> ist(2 * batch);
      std::memcpy(ch.data(), rb.data(), batch * 8);
      std::memcpy(sz.data(), rb.data() + ((const char*)d_scal2 - span0), batch * 8);
      std::memcpy(ist.data(), rb.data() + ((const char*)d_istat - span0), 2 * batch * 4);
      std::vector<int> next;
      for (int b : act) {
        iters[b] = it;
        if (ist[b] || (it > 1 && ist[batch + b])) { status[b] = LGM_SINGULAR; iters[b] = it - 1; continue; }
        const double tol = tol_in > 0.0 ? tol_in : 10.0 * n * LGM_UNIT_ROUNDOFF;
        if (!std::isfinite(ch[b]) || !std::isfinite(sz[b])) { status[b] = LGM_NONFINITE; continue; }
        if (sz[b] == 0.0) { status[b] = LGM_DB_NOCONV; continue; }
        const double rel = ch[b] / sz[b];
        auto note = [&](double x, double thr) { mm[b] = std::fmin(mm[b], std::fabs(x - thr) / std::fabs(thr)); };
        note(rel, LGM_SCALING_SWITCH);
        if (rel < LGM_SCALING_SWITCH) scaling[b] = 0;
        note(rel, tol);
        if (tol / 10.0 <= rel && rel <= 10.0 * tol) plateau[b]++;
        if (rel <= tol) continue;  // converged
        if (it == maxiter) { status[b] = LGM_DB_NOCONV; continue; }
        next.push_back(b);
      }
      act = next;
    }
    return 0;
  }
};

}  // namespace

// ============================================================================ Algorithm 1 host

namespace {

struct MState {
  int status = 0, s = 0, db_iters = 0, nest = 0, passes = 0, products = 0, k = 0, plateau = 0, sweeps = 0;
  bool finish = false, have_ai2 = false, post_fail = false;  // post_fail: non-finite L after the polynomial
  double alpha_loop = 0.0, mm = INFINITY, nA = 0.0, cert = 0.0;
  double cache[20];
  unsigned cvalid = 0u;
  void note(double x, double thr) {
    double d = std::fabs(thr);
    mm = std::fmin(mm, d > 0 ? std::fabs(x - thr) / d : std::fabs(x - thr));
  }
  bool le(double x, double thr) { note(x, thr); return x <= thr; }
};

// Batched alpha (oracle/driver.py _alpha) for requests (matrix, m, theta).  AmI is in slot
// G_AM, A_I2 in slot G_AP.  Returns alpha per request.
int alpha_batched(Grid& G, std::vector<MState>& ms, const std::vector<int>& mats, const std::vector<int>& mv,
                  const std::vector<double>& th, int itmax, std::vector<double>& out) {
  const int R = (int)mats.size();
  out.assign(R, 0.0);
  std::vector<double> t1(R), Pm(R);
  std::vector<int> need1;  // request indices needing the m-term estimate
  // phase A
  std::vector<int> ai2mats;
  for (int r = 0; r < R; ++r) if (ms[mats[r]].have_ai2) ai2mats.push_back(mats[r]);
  std::vector<double> nI2;
  if (G.onenorms(ai2mats, G_AP, nI2)) return LGM_ERR_CUDA;
  for (int r = 0; r < R; ++r) {
    MState& M = ms[mats[r]];
    const int m = mv[r];
    if (M.have_ai2) {
      const double r2 = std::sqrt(nI2[mats[r]]);
      if (M.le(r2, th[r])) { t1[r] = r2; Pm[r] = std::pow(nI2[mats[r]], (double)(m / 2)); continue; }
    }
    if ((M.cvalid >> m) & 1u) { Pm[r] = M.cache[m]; t1[r] = std::pow(Pm[r], 1.0 / m); }
    else need1.push_back(r);
  }
  auto run = [&](const std::vector<int>& reqs, bool second) -> int {
    if (reqs.empty()) return 0;
    // zero-matrix shortcut applies to est_power_norm only (matcore.py:309-310)
    std::vector<int> zm_ai2, zm_ami;
    for (int r : reqs) {
      MState& M = ms[mats[r]];
      bool product = second && M.have_ai2;
      if (!product) (M.have_ai2 ? zm_ai2 : zm_ami).push_back(mats[r]);
    }
    std::vector<int> nz_ai2, nz_ami;
    if (G.any_nonzero(zm_ai2, G_AP, nz_ai2)) return LGM_ERR_CUDA;
    if (G.any_nonzero(zm_ami, G_AM, nz_ami)) return LGM_ERR_CUDA;
    std::vector<const double*> M1, M2;
    std::vector<int> p1, zero;
    for (int r : reqs) {
      const int b = mats[r], m = mv[r];
      MState& M = ms[b];
      if (M.have_ai2) {
        M1.push_back(G.S.buf(b, G_AP));
        p1.push_back(m / 2);
        M2.push_back(second ? G.S.buf(b, G_AM) : nullptr);
        zero.push_back(second ? 0 : (nz_ai2[b] ? 0 : 1));
      } else {
        M1.push_back(G.S.buf(b, G_AM));
        p1.push_back(second ? m + 1 : m);
        M2.push_back(nullptr);
        zero.push_back(nz_ami[b] ? 0 : 1);
      }
    }
    std::vector<double> est, mm;
    std::vector<int> passes;
    if (G.estimate(M1, p1, M2, zero, itmax, est, passes, mm)) return LGM_ERR_CUDA;
    for (size_t q = 0; q < reqs.size(); ++q) {
      const int r = reqs[q], b = mats[r], m = mv[r];
      MState& M = ms[b];
      M.nest++;
      M.passes += passes[q];
      M.mm = std::fmin(M.mm, mm[q]);
      const int key = second ? m + 1 : m;
      M.cache[key] = est[q];
      M.cvalid |= 1u << key;
    }
    return 0;
  };
  if (run(need1, false)) return LGM_ERR_CUDA;
  for (int r : need1) {
    MState& M = ms[mats[r]];
    Pm[r] = M.cache[mv[r]];
    t1[r] = std::pow(Pm[r], 1.0 / mv[r]);
  }
  // phase B
  std::vector<int> need2;
  std::vector<double> t2(R, -1.0);
  std::vector<char> doneq(R, 0);
  for (int r = 0; r < R; ++r) {
    MState& M = ms[mats[r]];
    const int m = mv[r];
    M.note(t1[r], th[r]);
    if (t1[r] > th[r]) { out[r] = t1[r]; doneq[r] = 1; continue; }
    const double bound = std::pow(Pm[r] * M.nA, 1.0 / (m + 1));
    if (M.le(bound, th[r])) { t2[r] = bound; continue; }
    if ((M.cvalid >> (m + 1)) & 1u) t2[r] = std::pow(M.cache[m + 1], 1.0 / (m + 1));
    else need2.push_back(r);
  }
  if (run(need2, true)) return LGM_ERR_CUDA;
  for (int r : need2) t2[r] = std::pow(ms[mats[r]].cache[mv[r] + 1], 1.0 / (mv[r] + 1));
  for (int r = 0; r < R; ++r)
    if (!doneq[r]) out[r] = std::fmax(t1[r], t2[r]);
  return 0;
}

int first_index(MState& M, double x, const LgmParams& P) {
  for (int j = 1; j <= P.max_k; ++j)
    if (M.le(x, P.theta[j - 1])) return j;
  return P.max_k;
}

}  // namespace

size_t lgm_grid_workspace_bytes(int64_t n, int64_t batch) { return Grid::bytes(n, batch); }

int lgm_grid_logm(const double* A, double* L, int64_t n64, int64_t batch64, int64_t ld, const LgmParams& P,
                  lgm_report* rep, void* ws, cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  Grid G;
  G.st = st;
  G.carve(ws, n, batch);
  std::vector<MState> ms(batch);
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  // load + finiteness (as_square, matcore.py:64-65)
  CK(cudaMemsetAsync(G.d_iflag, 0, batch * 4, st));
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(A, ld, G.S, G.d_ids, G.d_iflag);
  std::vector<int> bad(batch);
  CK(cudaMemcpyAsync(bad.data(), G.d_iflag, batch * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int> live;
  for (int b = 0; b < batch; ++b) {
    if (bad[b]) ms[b].status = LGM_NONFINITE;
    else live.push_back(b);
  }
  // balance (matcore.py:180-215)
  {
    std::vector<double> mm0(batch, INFINITY);
    CK(cudaMemcpyAsync(G.d_margin, mm0.data(), batch * 8, cudaMemcpyHostToDevice, st));
    std::vector<double> ones((size_t)batch * n, 1.0);
    CK(cudaMemcpyAsync(G.d_scale, ones.data(), ones.size() * 8, cudaMemcpyHostToDevice, st));
    if (P.balance && !live.empty()) {
      if (G.upload_ids(live)) return LGM_ERR_CUDA;
      PhaseTimer pt(PH_BALANCE, st);
      lgm_count_launch(), balance_kernel_g<<<(int)live.size(), bal_threads(n), bal_smem(n), st>>>(G.S, G.d_ids, G.d_scale, G.d_sweeps, 100, G.d_margin);
      CK(cudaGetLastError());
      std::vector<int> sw(batch);
      CK(cudaMemcpyAsync(sw.data(), G.d_sweeps, batch * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(mm0.data(), G.d_margin, batch * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int b : live) { ms[b].sweeps = sw[b]; ms[b].mm = mm0[b]; }
    }
  }
  const int K = P.max_k;
  const double thK = P.theta[K - 1];
  const int mK = P.order[K - 1];
  // finish = ||B - I||_1 <= Theta_K
  if (G.ew(live, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;
  std::vector<double> nrm;
  if (G.onenorms(live, G_AM, nrm)) return LGM_ERR_CUDA;
  for (int b : live) {
    ms[b].alpha_loop = nrm[b];
    ms[b].finish = ms[b].le(nrm[b], thK);
  }
  // scaling loop
  while (true) {
    std::vector<int> act;
    for (int b : live)
      if (!ms[b].finish && ms[b].status == 0 && ms[b].s < P.maxiter_s) act.push_back(b);
    if (act.empty()) break;
    if (G.ew(act, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;
    if (G.onenorms(act, G_AM, nrm)) return LGM_ERR_CUDA;
    for (int b : act) ms[b].nA = nrm[b];
    std::vector<int> mv(act.size(), mK);
    std::vector<double> th(act.size(), thK), al;
    {
      PhaseTimer pt(PH_ALPHA, st);
      if (alpha_batched(G, ms, act, mv, th, P.est_itmax, al)) return LGM_ERR_CUDA;
    }
    std::vector<int> roots;
    for (size_t q = 0; q < act.size(); ++q) {
      MState& M = ms[act[q]];
      M.alpha_loop = al[q];
      M.finish = M.le(al[q], thK);
      if (!M.finish) roots.push_back(act[q]);
    }
    if (roots.empty()) continue;
    if (G.ew(roots, 1, G_AP, G_B, G_B)) return LGM_ERR_CUDA;  // A_prev = B
    std::vector<int> dst(batch, 0), dit(batch, 0), plat(batch, 0);
    std::vector<double> dmm(batch, INFINITY);
    if (G.sqrt_db(roots, P.db_tol, P.db_maxiter, dst, dit, dmm, plat)) return LGM_ERR_CUDA;
    std::vector<int> ok;
    for (int b : roots) {
      MState& M = ms[b];
      M.db_iters += dit[b];
      M.mm = std::fmin(M.mm, dmm[b]);
      M.plateau += plat[b];
      if (dst[b]) { M.status = dst[b]; continue; }
      M.s++;
      M.have_ai2 = true;
      M.cvalid = 0u;
      ok.push_back(b);
    }
    if (G.ew(ok, 3, G_AP, G_AP, G_B)) return LGM_ERR_CUDA;  // A_I2 = A_prev - 2B + I
  }
  // select (oracle/driver.py _select) for the finished matrices
  std::vector<int> sel;
  for (int b : live) {
    MState& M = ms[b];
    if (M.status == 0 && !M.finish) M.status = LGM_SCALING_MAXITER;
    if (M.status == 0) sel.push_back(b);
  }
  if (G.ew(sel, 0, G_AM, G_B, G_B)) return LGM_ERR_CUDA;
  if (G.onenorms(sel, G_AM, nrm)) return LGM_ERR_CUDA;
  std::vector<int> need_ai2;
  for (int b : sel) {
    ms[b].nA = nrm[b];
    if (!ms[b].have_ai2) need_ai2.push_back(b);
  }
  if (!need_ai2.empty()) {  // s = 0: A_I2 = (B - I)^2, one product
    if (G.upload_ids(need_ai2)) return LGM_ERR_CUDA;
    CombSpec cs{};
    cs.nterm = 1;
    cs.node[0] = G_AM;
    cs.coef[0] = 1.0;
    const int tiles = (n + TM - 1) / TM;
    if ((n & 1) == 0) {
      if (G.gemm_plain((int)need_ai2.size(), G_AM, G_AM, G_AP)) return LGM_ERR_CUDA;
    } else {
      lgm_count_launch(), gemm_comb_kernel<<<dim3(tiles, tiles, (int)need_ai2.size()), 128, 0, st>>>(G.S, G.d_ids, cs, G_AM, G_AP);
    }
    CK(cudaGetLastError());
    for (int b : need_ai2) { ms[b].products++; ms[b].have_ai2 = true; }
  }
  {
    std::vector<double> nI2;
    if (G.onenorms(sel, G_AP, nI2)) return LGM_ERR_CUDA;
    std::vector<int> min_im(batch), max_in(batch);
    std::vector<double> cert_max(batch);
    std::vector<int> cur;  // matrices still sweeping
    for (int b : sel) {
      MState& M = ms[b];
      const double r2 = std::sqrt(nI2[b]);
      int mi;
      if ((M.cvalid >> mK) & 1u) {
        mi = first_index(M, std::pow(M.cache[mK], 1.0 / mK), P);
        if ((M.cvalid >> (mK + 1)) & 1u) mi = std::max(mi, first_index(M, std::pow(M.cache[mK + 1], 1.0 / (mK + 1)), P));
      } else {
        mi = first_index(M, r2, P);
      }
      static const int tabmin[5] = {1, 2, 3, 4, 4};
      mi = tabmin[mi - 1];
      M.note(r2, P.theta[0]);
      mi = (r2 > P.theta[0]) ? std::max(mi, 2) : 1;
      int mx = K;
      double mb = -1.0;
      bool found = false;
      for (int j = 1; j <= K; ++j) {
        const int m = P.order[j - 1];
        const double bnd = std::pow(std::pow(nI2[b], (double)(m / 2)) * M.nA, 1.0 / (m + 1));
        if (M.le(bnd, P.theta[j - 1])) { mx = j; mb = bnd; found = true; break; }
      }
      cert_max[b] = found ? mb : M.alpha_loop;
      min_im[b] = mi;
      max_in[b] = mx;
      if (mi >= mx) { M.k = mx; M.cert = cert_max[b]; }
      else cur.push_back(b);
    }
    std::vector<int> jcur(batch);
    for (int b : cur) jcur[b] = min_im[b];
    while (!cur.empty()) {
      std::vector<int> mv;
      std::vector<double> th, al;
      for (int b : cur) { mv.push_back(P.order[jcur[b] - 1]); th.push_back(P.theta[jcur[b] - 1]); }
      PhaseTimer pt(PH_SELECT, st);
      if (alpha_batched(G, ms, cur, mv, th, P.est_itmax, al)) return LGM_ERR_CUDA;
      std::vector<int> next;
      for (size_t q = 0; q < cur.size(); ++q) {
        const int b = cur[q], j = jcur[b];
        MState& M = ms[b];
        if (M.le(al[q], P.theta[j - 1])) { M.k = j; M.cert = al[q]; continue; }
        if (M.le(al[q], P.theta[j])) { M.k = j + 1; M.cert = al[q]; continue; }
        if (j + 1 < max_in[b]) { jcur[b] = j + 1; next.push_back(b); }
        else { M.k = max_in[b]; M.cert = cert_max[b]; }
      }
      cur = next;
    }
  }
  // polynomial: P2 = I - B (slot G_B), P3 = A_I2 (G_AP), R temp (G_Y), P4.. in G_XI, G_YI, G_P6, G_P7
  PhaseTimer pt_poly(PH_POLY, st);
  if (G.ew(sel, 4, G_B, G_B, G_B)) return LGM_ERR_CUDA;
  const int node_slot[8] = {-1, -1, G_B, G_AP, G_XI, G_YI, G_P6, G_P7};
  for (int kk = 1; kk <= K; ++kk) {
    std::vector<int> grp;
    for (int b : sel)
      if (ms[b].k == kk) grp.push_back(b);
    if (grp.empty()) continue;
    const double* base = P.coef + P.coef_off[kk - 1];
    auto spec = [&](const double* row, int nn) {
      CombSpec cs{};
      cs.c0 = row[0];
      for (int t = 2; t <= nn; ++t)
        if (row[t - 1] != 0.0) { cs.node[cs.nterm] = node_slot[t]; cs.coef[cs.nterm] = row[t - 1]; cs.nterm++; }
      return cs;
    };
    const int tiles = (n + TM - 1) / TM;
    int nn = 3;
    for (int j = 1; j < kk; ++j) {
      const double* lrow = base + j * (j + 3) / 2;
      const double* rrow = base + kk * (kk + 3) / 2 + j * (j + 3) / 2;
      if (G.upload_ids(grp)) return LGM_ERR_CUDA;
      CombSpec rs = spec(rrow, nn);
      lgm_count_launch(), combine_kernel<<<G.ew_grid((int)grp.size()), 256, 0, st>>>(G.S, G.d_ids, rs, G_Y);
      CombSpec ls = spec(lrow, nn);
      if ((n & 1) == 0) {  // materialise L too (slot G_AM is free after select), then a plain GEMM
        lgm_count_launch(), combine_kernel<<<G.ew_grid((int)grp.size()), 256, 0, st>>>(G.S, G.d_ids, ls, G_AM);
        if (G.gemm_plain((int)grp.size(), G_AM, G_Y, node_slot[nn + 1])) return LGM_ERR_CUDA;
      } else {
        lgm_count_launch(), gemm_comb_kernel<<<dim3(tiles, tiles, (int)grp.size()), 128, 0, st>>>(G.S, G.d_ids, ls, G_Y, node_slot[nn + 1]);
      }
      CK(cudaGetLastError());
      nn++;
      for (int b : grp) ms[b].products++;
    }
    const double* orow = base + kk * (kk + 3);
    CombSpec os = spec(orow, nn);
    std::vector<double> mult(batch, 0.0);
    for (int b : grp) mult[b] = -std::ldexp(1.0, ms[b].s);
    CK(cudaMemcpyAsync(G.d_scal, mult.data(), batch * 8, cudaMemcpyHostToDevice, st));
    if (G.upload_ids(grp)) return LGM_ERR_CUDA;
    CK(cudaMemsetAsync(G.d_iflag, 0, batch * 4, st));
    lgm_count_launch(), final_kernel<<<G.ew_grid((int)grp.size()), 256, 0, st>>>(G.S, G.d_ids, os, G.d_scal, G.d_scale,
                                                                                P.balance, L, ld, G.d_iflag);
    CK(cudaGetLastError());
    std::vector<int> nf(batch);
    CK(cudaMemcpyAsync(nf.data(), G.d_iflag, batch * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // a non-finite logarithm (estimator overflow upstream, norms ~1e300) is reported, with
    // the k / products / alpha of the run that produced it
    for (int b : grp)
      if (nf[b]) { ms[b].status = LGM_NONFINITE; ms[b].post_fail = true; }
  }
  {
    std::vector<int> failed;
    for (int b = 0; b < batch; ++b)
      if (ms[b].status && !ms[b].post_fail) failed.push_back(b);
    if (!failed.empty()) {
      if (G.upload_ids(failed)) return LGM_ERR_CUDA;
      lgm_count_launch(), nan_fill_kernel<<<G.ew_grid((int)failed.size()), 256, 0, st>>>(G.d_ids, n, L, ld);
      CK(cudaGetLastError());
    }
  }
  // reports
  std::vector<lgm_report> R(batch);
  for (int b = 0; b < batch; ++b) {
    MState& M = ms[b];
    lgm_report& r = R[b];
    std::memset(&r, 0, sizeof(r));
    r.status = M.status;
    r.s = M.s;
    const bool keep = !M.status || M.post_fail;
    r.k = keep ? M.k : 0;
    r.db_iters = M.db_iters;
    r.products = keep ? M.products : 0;
    r.divisions = 2 * M.db_iters;
    r.estimation_passes = M.passes;
    r.norm_estimations = M.nest;
    r.balanced = P.balance;
    r.balance_sweeps = M.sweeps;
    r.db_plateau = M.plateau;
    r.alpha_used = keep ? M.cert : 0.0;
    r.min_margin = M.mm;
  }
  CK(cudaMemcpyAsync(rep, R.data(), batch * sizeof(lgm_report), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

// ============================================================================ building blocks (n > 64)
// These entry points take no workspace argument; for n > 64 they use stream-ordered scratch
// (cudaMallocAsync) released before returning.

namespace {
struct Scratch {
  void* p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() { if (p) cudaFreeAsync(p, st); }
};
}  // namespace

int lgm_grid_sqrt_db(const double* A, double* X, int64_t n64, int64_t batch64, int64_t ld, double tol, int maxiter,
                     int* iters, int* status, cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  Scratch sc(st);
  CK(cudaMallocAsync(&sc.p, Grid::bytes(n, batch), st));
  Grid G;
  G.st = st;
  G.carve(sc.p, n, batch);
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  CK(cudaMemsetAsync(G.d_iflag, 0, batch * 4, st));
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(A, ld, G.S, G.d_ids, G.d_iflag);
  std::vector<int> bad(batch);
  CK(cudaMemcpyAsync(bad.data(), G.d_iflag, batch * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int> live, dst(batch, 0), dit(batch, 0), plat(batch, 0);
  std::vector<double> mm(batch, INFINITY);
  for (int b = 0; b < batch; ++b) {
    if (bad[b]) dst[b] = LGM_NONFINITE;
    else live.push_back(b);
  }
  if (G.sqrt_db(live, tol, maxiter, dst, dit, mm, plat)) return LGM_ERR_CUDA;
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), store_kernel<<<G.ew_grid(batch), 256, 0, st>>>(G.S, G.d_ids, G_B, X, ld);
  CK(cudaMemcpyAsync(iters, dit.data(), batch * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(status, dst.data(), batch * 4, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int lgm_grid_est(const double* M1, int p1, const double* M2, int64_t n64, int64_t batch64, int64_t ld, int itmax,
                 int zero_shortcut, double* est, int* passes, cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  Scratch sc(st);
  CK(cudaMallocAsync(&sc.p, Grid::bytes(n, batch), st));
  Grid G;
  G.st = st;
  G.carve(sc.p, n, batch);
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(M1, ld, G.S, G.d_ids, G.d_iflag);
  if (M2) {  // second operand into slot G_AM via the B slot
    G.ew(all, 1, G_AP, G_B, G_B);
    lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(M2, ld, G.S, G.d_ids, G.d_iflag);
    G.ew(all, 1, G_AM, G_B, G_B);
    G.ew(all, 1, G_B, G_AP, G_AP);
  }
  std::vector<int> nz;
  if (zero_shortcut) {
    if (G.any_nonzero(all, G_B, nz)) return LGM_ERR_CUDA;
  } else {
    nz.assign(batch, 1);
  }
  std::vector<const double*> m1, m2;
  std::vector<int> pp, zero;
  for (int b = 0; b < batch; ++b) {
    m1.push_back(G.S.buf(b, G_B));
    m2.push_back(M2 ? G.S.buf(b, G_AM) : nullptr);
    pp.push_back(p1);
    zero.push_back(nz[b] ? 0 : 1);
  }
  std::vector<double> e, mm;
  std::vector<int> ps;
  if (G.estimate(m1, pp, m2, zero, itmax, e, ps, mm)) return LGM_ERR_CUDA;
  CK(cudaMemcpyAsync(est, e.data(), batch * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(passes, ps.data(), batch * 4, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int lgm_grid_balance(const double* A, double* B, double* scale, int64_t n64, int64_t batch64, int64_t ld,
                     int max_sweeps, int* sweeps, cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  Scratch sc(st);
  CK(cudaMallocAsync(&sc.p, Grid::bytes(n, batch), st));
  Grid G;
  G.st = st;
  G.carve(sc.p, n, batch);
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(A, ld, G.S, G.d_ids, G.d_iflag);
  std::vector<double> mm0(batch, INFINITY);
  CK(cudaMemcpyAsync(G.d_margin, mm0.data(), batch * 8, cudaMemcpyHostToDevice, st));
  lgm_count_launch(), balance_kernel_g<<<batch, bal_threads(n), bal_smem(n), st>>>(G.S, G.d_ids, scale, sweeps, max_sweeps, G.d_margin);
  lgm_count_launch(), store_kernel<<<G.ew_grid(batch), 256, 0, st>>>(G.S, G.d_ids, G_B, B, ld);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return 0;
}

int lgm_grid_degopt(const double* X, const double* FP, double* Z, int64_t n64, int64_t batch64, int64_t ld, int k,
                    int* products, const LgmParams& P, cudaStream_t st) {
  const int n = (int)n64, batch = (int)batch64;
  Scratch sc(st);
  CK(cudaMallocAsync(&sc.p, Grid::bytes(n, batch), st));
  Grid G;
  G.st = st;
  G.carve(sc.p, n, batch);
  std::vector<int> all(batch);
  for (int b = 0; b < batch; ++b) all[b] = b;
  if (G.upload_ids(all)) return LGM_ERR_CUDA;
  lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(X, ld, G.S, G.d_ids, G.d_iflag);
  int prods = 0;
  const int tiles = (n + TM - 1) / TM;
  if (FP) {
    G.ew(all, 1, G_Y, G_B, G_B);
    lgm_count_launch(), load_kernel<<<G.ew_grid(batch), 256, 0, st>>>(FP, ld, G.S, G.d_ids, G.d_iflag);
    G.ew(all, 1, G_AP, G_B, G_B);
    G.ew(all, 1, G_B, G_Y, G_Y);
  } else {
    CombSpec cs{};
    cs.nterm = 1;
    cs.node[0] = G_B;
    cs.coef[0] = 1.0;
    lgm_count_launch(), gemm_comb_kernel<<<dim3(tiles, tiles, batch), 128, 0, st>>>(G.S, G.d_ids, cs, G_B, G_AP);
    prods++;
  }
  const int node_slot[8] = {-1, -1, G_B, G_AP, G_XI, G_YI, G_P6, G_P7};
  const double* base = P.coef + P.coef_off[k - 1];
  auto spec = [&](const double* row, int nn) {
    CombSpec cs{};
    cs.c0 = row[0];
    for (int t = 2; t <= nn; ++t)
      if (row[t - 1] != 0.0) { cs.node[cs.nterm] = node_slot[t]; cs.coef[cs.nterm] = row[t - 1]; cs.nterm++; }
    return cs;
  };
  int nn = 3;
  for (int j = 1; j < k; ++j) {
    const double* lrow = base + j * (j + 3) / 2;
    const double* rrow = base + k * (k + 3) / 2 + j * (j + 3) / 2;
    CombSpec rs = spec(rrow, nn);
    lgm_count_launch(), combine_kernel<<<G.ew_grid(batch), 256, 0, st>>>(G.S, G.d_ids, rs, G_Y);
    CombSpec ls = spec(lrow, nn);
    lgm_count_launch(), gemm_comb_kernel<<<dim3(tiles, tiles, batch), 128, 0, st>>>(G.S, G.d_ids, ls, G_Y, node_slot[nn + 1]);
    nn++;
    prods++;
  }
  CombSpec os = spec(base + k * (k + 3), nn);
  std::vector<double> mult(batch, 1.0);
  CK(cudaMemcpyAsync(G.d_scal, mult.data(), batch * 8, cudaMemcpyHostToDevice, st));
  lgm_count_launch(), final_kernel<<<G.ew_grid(batch), 256, 0, st>>>(G.S, G.d_ids, os, G.d_scal, G.d_scale, 0, Z, ld,
                                                                      nullptr);
  CK(cudaGetLastError());
  std::vector<int> pr(batch, prods);
  CK(cudaMemcpyAsync(products, pr.data(), batch * 4, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

extern "C" int lgm_debug_panel_cycles(unsigned long long* out) {
#ifdef LGM_PANEL_PROF
  cudaMemcpyFromSymbol(out, g_panel_cyc, sizeof(g_panel_cyc));
  return 6;
#else
  (void)out;
  return 0;
#endif
}

extern "C" int lgm_debug_grid_phase_ms(double* out, int reset) {
  for (int i = 0; i < PH_N; ++i) {
    out[i] = g_phase_ms[i];
    if (reset) g_phase_ms[i] = 0.0;
  }
  return PH_N;
}
