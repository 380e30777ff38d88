// Engine F: the whole logm pipeline for one matrix per CTA, n <= NMAX (32 or 64).
//
// Layout: the CTA is two *teams* of T = NMAX/32 warps; inside a
// team thread `row` owns matrix row `row`.  Matrices live in shared memory with a padded
// row stride LDM = NMAX + 1 doubles, which makes both row-per-thread accesses
// (M[row][j], lanes = rows) and column-per-thread accesses (M[i][col], lanes = cols)
// bank-conflict free.  The pivoted Gauss-Jordan inversion keeps the row being eliminated
// in registers (NMAX doubles per thread, fully unrolled); the two teams invert X and Y of
// the Denman-Beavers step concurrently, and the two columns of the block 1-norm
// estimator run on the two teams.  All threads execute the (uniform) Algorithm-1 driver
// code; data-dependent decisions are broadcast through shared memory.
//
// Reference (relative to /root/reference/pkg/src/logmpoly/): balance matcore.py:180-215;
// onenorm :84-87; est_product_norm :234-297; est_power_norm :300-311; sqrt_db
// sqrtm.py:27-78; eval_degopt schemes.py:91-126; driver SPEC.md:429-502 / PAPER.md:724-840
// as restated in oracle/driver.py.
#pragma once
#include "lgm_common.cuh"

namespace lgm {

#ifdef LGM_PHASE_PROF
// cycles per phase summed over CTAs: 0 balance, 1 scaling-loop alpha, 2 sqrt_db, 3 select, 4 poly
__device__ unsigned long long lgm_phase_cycles[8];
#define LGM_PHASE_BEGIN(c) long long _lgm_t0 = clock64()
#define LGM_PHASE_END(c, ph) do { if ((c).tid == 0) atomicAdd(&lgm_phase_cycles[ph], (unsigned long long)(clock64() - _lgm_t0)); } while (0)
#else
#define LGM_PHASE_BEGIN(c) do {} while (0)
#define LGM_PHASE_END(c, ph) do {} while (0)
#endif

// Dynamic shared memory, referenced by symbol so every access compiles to LDS/STS.
extern __shared__ __align__(16) double lgm_smem[];

template <int NMAX>
struct Cfg {
  static constexpr int T = NMAX / 32;     // warps per team
  static constexpr int NT = 64 * T;       // threads per CTA
  static constexpr int LDM = NMAX + 1;    // padded row stride (doubles)
  static constexpr int MAT = NMAX * LDM;  // doubles per matrix buffer
  static constexpr int NBUF = 2;          // B (X) and Y; A_prev / A_I2 and P4..P6 live in L2
  // shared-memory carve-up (in doubles)
  static constexpr int OFF_PROW = NBUF * MAT;                // [2 teams][2][NMAX+2]
  static constexpr int PROW = NMAX + 2;
  static constexpr int OFF_VEC = OFF_PROW + 2 * 2 * PROW;    // [8][NMAX]
  static constexpr int OFF_SCALE = OFF_VEC + 9 * NMAX;       // [NMAX] balancing scales
  static constexpr int OFF_RED = OFF_SCALE + NMAX;           // [64] reduction scratch
  static constexpr int OFF_INT = OFF_RED + 64;               // ints: piv[2][NMAX], misc[64]
  static constexpr int SMEM_DOUBLES = OFF_INT + (2 * NMAX + 64 + 1) / 2 + 1;
  static constexpr size_t SMEM_BYTES = (size_t)SMEM_DOUBLES * sizeof(double);
  // kernels that keep the polynomial nodes P4..P6 in shared memory too (building blocks)
  static constexpr size_t SMEM_BYTES_X = SMEM_BYTES + 4 * MAT * sizeof(double);
};

// misc int slots
enum { MI_STATUS = 0, MI_STATUS2, MI_J, MI_NPICK, MI_ORDER = 8 /* 9 slots */, MI_PICK = 20,
       MI_FLAG = 24, MI_COUNT = 64 };
// red double slots
enum { RD_LOGDET = 0 /* 2 */, RD_KEY = 4 /* [2 teams][4 slots] */, RD_CN = 12 /* 2 */,
       RD_CHANGE = 16, RD_SCALE = 20 /* [2 warps] */, RD_MARGIN = 24, RD_EST = 28,
       RD_NORM = 32 /* [4] */, RD_H = 40 /* 9 sorted h values */ };

// The matrix order as seen by the kernel code: a runtime int, or the compile-time NMAX when
// the kernel is instantiated for n == NMAX (FULL), which folds every `row < n` / `j < n`
// guard and trip count away.
template <int NMAX, bool FULL>
struct NVal {
  int v;
  __device__ __forceinline__ operator int() const { return FULL ? NMAX : v; }
  __device__ __forceinline__ NVal& operator=(int x) { v = x; return *this; }
};

template <int NMAX, bool FULL = false>
struct Ctx {
  using C = Cfg<NMAX>;
  NVal<NMAX, FULL> n;
  int tid, warp, lane, team, wit, row;  // wit = warp index in team, row = wit*32 + lane
  const LgmParams* P;
  double mm;       // running min margin (uniform)
  int plateau;     // DB stop tests in the noise band [tol/10, 10 tol] (uniform)

  __device__ __forceinline__ static double* sm() { return lgm_smem; }
  // a matrix operand: shared buffer (row stride LDM) or global workspace slot (row stride n)
  struct MRef {
    double* p;
    int ld;
  };
  __device__ MRef bref(int b) const { return MRef{buf(b), C::LDM}; }
  __device__ double* buf(int b) const { return sm() + b * C::MAT; }
  __device__ double* prow(int tm, int parity) const { return sm() + C::OFF_PROW + (tm * 2 + parity) * C::PROW; }
  __device__ double* vec(int v) const { return sm() + C::OFF_VEC + v * NMAX; }
  __device__ double* scale() const { return sm() + C::OFF_SCALE; }
  __device__ double* red() const { return sm() + C::OFF_RED; }
  __device__ int* ints() const { return reinterpret_cast<int*>(sm() + C::OFF_INT); }
  __device__ int* piv(int tm) const { return ints() + tm * NMAX; }
  __device__ int* misc() const { return ints() + 2 * NMAX; }

  __device__ void init(double* smem, int n_, const LgmParams* p) {
    (void)smem; n = n_; P = p;
    tid = threadIdx.x; warp = tid >> 5; lane = tid & 31;
    team = warp / C::T; wit = warp % C::T; row = wit * 32 + lane;
    mm = INFINITY;
    plateau = 0;
  }

  __device__ __forceinline__ void team_sync() const {
    if (C::T == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(C::T * 32) : "memory");
  }

  // ---- margins (uniform) -------------------------------------------------------------
  __device__ __forceinline__ void note(double x, double thr) {
    double den = fabs(thr);
    double m = den > 0.0 ? fabs(x - thr) * lgm_rcp_rough(den) : fabs(x - thr);
    mm = fmin(mm, m);
  }
  __device__ __forceinline__ void gap(double a, double b) {
    double den = fmax(fabs(a), fabs(b));
    mm = fmin(mm, den > 0.0 ? fabs(a - b) * lgm_rcp_rough(den) : 0.0);
  }
  __device__ __forceinline__ bool le(double x, double thr) { note(x, thr); return x <= thr; }

  // ---- elementwise helpers ------------------------------------------------------------
  // Estimator restart column (matcore.py:265-271): v_i = (-1)^i (1 + i/max(1, n-1)),
  // normalised by numpy's pairwise sum of |v|; built once per matrix into vec(8).
  __device__ void init_ramp() {
    if (tid == 0) {
      red()[RD_EST] = lgm_pairwise_sum(
          [&](int i) { return fabs(((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))); }, n);
    }
    __syncthreads();
    const double rsum = red()[RD_EST];
    for (int i = tid; i < n; i += C::NT)
      vec(8)[i] = (((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(n > 1 ? n - 1 : 1))) / rsum;
    __syncthreads();
  }

  __device__ void zero_all() {
    // matrices, pivot rows, estimator vectors and scales (padding must read as 0)
    static_assert(C::OFF_RED % 2 == 0, "double2 zeroing");
    double2* p = reinterpret_cast<double2*>(sm());
    for (int i = tid; i < C::OFF_RED / 2; i += C::NT) p[i] = make_double2(0.0, 0.0);
  }
  __device__ void copy_buf(int dst, int src) {
    double* d = buf(dst);
    const double* s = buf(src);
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
      d[i * C::LDM + j] = s[i * C::LDM + j];
    }
  }
  __device__ void set_identity(int b) {
    double* d = buf(b);
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
      d[i * C::LDM + j] = (i == j) ? 1.0 : 0.0;
    }
  }

  // onenorm of a referenced matrix (numpy order: column sums over rows in order)
  __device__ double onenorm_ref(MRef M) {
    double cs = 0.0;
    for (int j = tid; j < n; j += C::NT) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc = (i == 0) ? fabs(M.p[i * M.ld + j]) : acc + fabs(M.p[i * M.ld + j]);
      cs = fmax(cs, acc);
    }
    cs = lgm_warp_max(cs);
    __syncthreads();
    if (lane == 0) red()[RD_NORM + warp] = cs;
    __syncthreads();
    double r = red()[RD_NORM];
    for (int w = 1; w < C::NT / 32; ++w) r = fmax(r, red()[RD_NORM + w]);
    __syncthreads();
    return r;
  }

  // onenorm(M - shift*I) exactly as numpy: column sums accumulated over rows in order.
  __device__ double onenorm(int b, double shift) {
    const double* M = buf(b);
    double cs = 0.0;
    for (int j = tid; j < n; j += C::NT) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        double v = M[i * C::LDM + j];
        if (i == j) v = v - shift;
        acc = (i == 0) ? fabs(v) : acc + fabs(v);
      }
      cs = fmax(cs, acc);
    }
    cs = lgm_warp_max(cs);
    __syncthreads();
    if (lane == 0) red()[RD_NORM + warp] = cs;
    __syncthreads();
    double r = red()[RD_NORM];
    for (int w = 1; w < C::NT / 32; ++w) r = fmax(r, red()[RD_NORM + w]);
    __syncthreads();
    return r;
  }

  // ---- balancing (matcore.py:180-215), bit-identical decisions --------------------------
  // numpy pairwise sum of |p[i*stride]|, i < n <= 128 (lgm_common.cuh lgm_pairwise_block).
  __device__ __forceinline__ double pw_abs_sum(const double* p, int stride) const {
    if (n < 8) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += fabs(p[i * stride]);
      return s;
    }
    double r0 = fabs(p[0]), r1 = fabs(p[stride]), r2 = fabs(p[2 * stride]), r3 = fabs(p[3 * stride]);
    double r4 = fabs(p[4 * stride]), r5 = fabs(p[5 * stride]), r6 = fabs(p[6 * stride]), r7 = fabs(p[7 * stride]);
    int i = 8;
    const int m8 = n - (n % 8);
    for (; i < m8; i += 8) {
      const double* q = p + i * stride;
      r0 += fabs(q[0]); r1 += fabs(q[stride]); r2 += fabs(q[2 * stride]); r3 += fabs(q[3 * stride]);
      r4 += fabs(q[4 * stride]); r5 += fabs(q[5 * stride]); r6 += fabs(q[6 * stride]); r7 += fabs(q[7 * stride]);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += fabs(p[i * stride]);
    return res;
  }

  // Non-inlined entry points work on a register copy of the context: member accesses
  // through `this` would otherwise be local-memory loads inside the hot loops.
  __device__ __noinline__ int balance(int b, int max_sweeps) {
    Ctx s = *this;
    const int r = s.balance_impl(b, max_sweeps);
    mm = s.mm;
    return r;
  }
  __device__ __forceinline__ int balance_impl(int b, int max_sweeps) {
    double* B = buf(b);
    double* sc = scale();
    for (int i = tid; i < n; i += C::NT) sc[i] = 1.0;
    __syncthreads();
    int sweeps = 0;
    for (int sw = 0; sw < max_sweeps; ++sw) {
      sweeps++;
      bool moved = false;
      const int m8 = n - (n % 8);
      for (int i = 0; i < n; ++i) {
        // numpy pairwise sums of |B[:, i]| (lanes 0-7) and |B[i, :]| (lanes 8-15) of warp 0:
        // the 8 interleaved accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by
        // xor-shuffles (commutative adds), tail added in order by lane 0.  Lane 0 decides;
        // only its margin record is reported.
        if (warp == 0) {
          const int q = lane & 7;
          const bool colside = lane < 8;
          const double* base = colside ? B + i : B + i * C::LDM;
          const int stride = colside ? C::LDM : 1;
          double acc = 0.0;
          if (n >= 8 && lane < 16) {
            acc = fabs(base[q * stride]);
            for (int k = 8 + q; k < m8; k += 8) acc += fabs(base[k * stride]);
          }
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          acc += __shfl_xor_sync(0xffffffffu, acc, 4);
          double csum = __shfl_sync(0xffffffffu, acc, 0);
          double rsum = __shfl_sync(0xffffffffu, acc, 8);
          if (lane == 0) {
            if (n < 8) {
              csum = 0.0;
              rsum = 0.0;
              for (int k = 0; k < n; ++k) csum += fabs(B[k * C::LDM + i]);
              for (int k = 0; k < n; ++k) rsum += fabs(B[i * C::LDM + k]);
            } else {
              for (int k = m8; k < n; ++k) csum += fabs(B[k * C::LDM + i]);
              for (int k = m8; k < n; ++k) rsum += fabs(B[i * C::LDM + k]);
            }
            const double dg = fabs(B[i * C::LDM + i]);
            double c = csum - dg, r = rsum - dg, f = 0.0;
            if (!(c == 0.0 || r == 0.0)) {
              double tot = c + r;
              f = 1.0;
              while (true) {
                note(c, r / 2.0);
                if (!(c < r / 2.0)) break;
                c *= 2.0; r /= 2.0; f *= 2.0;
              }
              while (true) {
                note(c, r * 2.0);
                if (!(c >= r * 2.0)) break;
                c /= 2.0; r *= 2.0; f /= 2.0;
              }
              note(c + r, 0.95 * tot);
              if (!(c + r < 0.95 * tot && 1e-300 < f && f < 1e300)) f = 0.0;
            }
            red()[RD_MARGIN + (i & 1)] = f;  // 0: leave row/column i alone (double-buffered)
          }
        }
        __syncthreads();
        const double f = red()[RD_MARGIN + (i & 1)];
        if (f != 0.0) {
          double inv = 1.0 / f;  // exact: f is a power of two in (1e-300, 1e300)
          for (int q = tid; q < n; q += C::NT) B[q * C::LDM + i] *= f;
          __syncthreads();
          for (int q = tid; q < n; q += C::NT) B[i * C::LDM + q] *= inv;
          if (tid == 0) sc[i] *= f;
          moved = true;
          __syncthreads();
        }
      }
      if (!moved) break;
    }
    __syncthreads();
    return sweeps;
  }

  // ---- pivoted Gauss-Jordan inversion of the team's matrix, row in registers -------------
  // On entry r[] holds row `row` of M (zeros beyond n; rows >= n all zero).  On exit r[]
  // holds storage row `row` of the in-place result: Minv[q(row)][p_j] = r[j], where p_j is
  // the pivot row of step j (piv(team)[j]) and q(row) = my_step.  Returns 1 if an exact zero
  // pivot is met (matcore.py:124-125), else 0; logabsdet = sum log|pivot| (team-uniform).
  // Implementation notes: every pivot step reads the pivot column from r[0] and writes the
  // eliminated row back shifted by one register (r[j] <- r[j+1] - g * prow[j+1]), so the
  // pivot column of the next step is again r[0]: static register indexing inside a small
  // runtime loop (no unrolling over steps, no rotation moves -- the shift rides in the FMA's
  // destination).  After NMAX steps (steps k >= n are pure rotations) the frame is back to
  // the identity.  Row scaling is deferred: the pivot row is broadcast unscaled together with
  // 1/pivot, the other rows fold 1/pivot into their multiplier, and the pivot row keeps raw
  // values (its column-k entry set to 1) and is scaled once at the end -- the elimination is
  // linear in each row, so this is the same Gauss-Jordan recurrence with different rounding.
#ifndef LGM_F_PUBFIRST
#define LGM_F_PUBFIRST 1  // A/B: config 1 1.845 -> 1.762 ms, config 2 2.454 -> 2.445 ms, bit-identical
#endif
  __device__ int gj_invert(double (&r)[NMAX], double& logabsdet, int& my_step) {
    bool used = false;
    my_step = -1;
    double mylog = 0.0, rowscale = 1.0;
    int* pv = piv(team);
    double* kslot = red() + RD_KEY + team * 4;
    int status = 0;
#pragma unroll 1
    for (int k = 0; k < NMAX; ++k) {
      const double r0 = r[0];
      double g = 0.0, last = r0;        // defaults: pure rotation (steps k >= n)
      const double* pr = prow(team, k & 1);
      if (k < n) {                      // team-uniform
        // argmax |r0| over the remaining rows on a single 32-bit key: the high word of |r0|
        // (exponent and 20 mantissa bits) with its low RB bits replaced by (2 NMAX - 1 - row),
        // so one redux picks a row whose |value| is within 2^-13 relative of the largest
        // (ties -> lowest row).  That is partial pivoting with a 1 - 2^-13 threshold, as
        // stable as the exact argmax; the exact signed pivot then comes by shuffle.  Exact
        // zeros are not candidates: an all-zero key means an exactly singular step.
        constexpr int RB = (NMAX == 32) ? 6 : 7;
        constexpr unsigned RMASK = (1u << RB) - 1u;
        const bool cand = (row < n) && !used && r0 != 0.0;
        const unsigned key = cand ? ((((unsigned)__double2hiint(r0) & 0x7fffffffu) & ~RMASK) |
                                     (unsigned)(2 * NMAX - 1 - row)) : 0u;
        unsigned kmax = __reduce_max_sync(0xffffffffu, key);
        int prow_idx = 2 * NMAX - 1 - (int)(kmax & RMASK);
        double pval = __shfl_sync(0xffffffffu, r0, prow_idx & 31);  // exact signed pivot
        if (C::T > 1) {
          if (lane == 0) {
            reinterpret_cast<unsigned*>(kslot)[wit] = kmax;
            kslot[2 + wit] = pval;
          }
          team_sync();
          const unsigned k0 = reinterpret_cast<unsigned*>(kslot)[0];
          const unsigned k1 = reinterpret_cast<unsigned*>(kslot)[1];
          const int w = k1 > k0 ? 1 : 0;
          kmax = w ? k1 : k0;
          pval = kslot[2 + w];
          prow_idx = 2 * NMAX - 1 - (int)(kmax & RMASK);
        }
        const unsigned mhi = kmax, mlo = 0u;
        if ((mhi | mlo) == 0u) { status = 1; break; }  // all remaining candidates exactly zero
        double* pw = prow(team, k & 1);
        const bool own = (row == prow_idx);
#if LGM_F_PUBFIRST
        // the owner's stores first: the reciprocal's slow-path call is a scheduling barrier,
        // so in source order after it the publish would wait for the whole Newton chain
        if (own) {  // one lane publishes its raw row (current frame)
          used = true;
          my_step = k;
          mylog = r0;  // log|p| taken once after the loop (one pivot per row)
#pragma unroll
          for (int j = 0; j < NMAX; j += 2) *reinterpret_cast<double2*>(pw + j) = make_double2(r[j], r[j + 1]);
        }
        if (lane == 0 && wit == 0) pv[k] = prow_idx;
        const double rp = lgm_rcp(pval);
        if (own) rowscale = rp;
        team_sync();
#else
        const double rp = lgm_rcp(pval);  // every lane, in parallel with the owner's stores
        if (own) {  // one lane publishes its raw row (current frame)
          used = true;
          my_step = k;
          mylog = r0;  // log|p| taken once after the loop (one pivot per row)
          rowscale = rp;
#pragma unroll
          for (int j = 0; j < NMAX; j += 2) *reinterpret_cast<double2*>(pw + j) = make_double2(r[j], r[j + 1]);
        }
        if (lane == 0 && wit == 0) pv[k] = prow_idx;
        team_sync();
#endif
        g = own ? 0.0 : r0 * rp;  // branch-free: the owner keeps its raw row
        last = own ? 1.0 : -g;
      }
      // shifted elimination: r[j] <- r[j+1] - g * prow[j+1]; g == 0 -> exact rotation
#pragma unroll
      for (int j = 0; j < NMAX; j += 2) {
        const double2 p2 = *reinterpret_cast<const double2*>(pr + j);  // prow[j], prow[j+1]
        if (j > 0) r[j - 1] = fma(-g, p2.x, r[j]);
        r[j] = fma(-g, p2.y, r[j + 1 < NMAX ? j + 1 : j]);
      }
      r[NMAX - 1] = last;
    }
    if (rowscale != 1.0) {
#pragma unroll
      for (int j = 0; j < NMAX; ++j) r[j] *= rowscale;
    }
    // team sum of the pivots' log|.| (one per valid row)
    double s = lgm_warp_sum(my_step >= 0 ? log(fabs(mylog)) : 0.0);
    if (C::T > 1) {
      team_sync();
      if (lane == 0) red()[RD_LOGDET + team * 2 + wit] = s;
      team_sync();
      s = red()[RD_LOGDET + team * 2] + red()[RD_LOGDET + team * 2 + 1];
      team_sync();
    }
    logabsdet = s;
    return status;
  }

  // butterfly reduce-scatter of v[NMAX] over the warp: lane l ends holding the sums of
  // register indices {l*(NMAX/32) + e}; returns max over those per-lane sums (warp-reduced
  // to a single value for the whole team).
  __device__ double colsum_max(double (&v)[NMAX]) {
#pragma unroll
    for (int off = 16, len = NMAX; off >= 1; off >>= 1, len >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < NMAX / 2; ++i) {
        if (i < len / 2) {
          double send = up ? v[i] : v[i + len / 2];
          double keep = up ? v[i + len / 2] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
    }
    // lane holds NMAX/32 column partial sums in v[0..NMAX/32-1] (this warp's rows)
    if (C::T == 1) {
      double m = v[0];
#pragma unroll
      for (int e = 1; e < NMAX / 32; ++e) m = fmax(m, v[e]);
      return lgm_warp_max(m);
    }
    // T == 2: add the other warp's partial column sums
    double* scr = vec(6);  // [NMAX] scratch
    team_sync();
    if (wit == 1) {
#pragma unroll
      for (int e = 0; e < NMAX / 32; ++e) scr[lane * (NMAX / 32) + e] = v[e];
    }
    team_sync();
    double m = 0.0;
    if (wit == 0) {
#pragma unroll
      for (int e = 0; e < NMAX / 32; ++e) m = fmax(m, v[e] + scr[lane * (NMAX / 32) + e]);
    }
    m = lgm_warp_max(m);
    team_sync();
    return m;  // valid in warp wit == 0
  }

  // ---- scaled coupled Denman-Beavers square root (sqrtm.py:27-78) ------------------------
  // X (buffer bx) is replaced by X^(1/2); buffer by is workspace (Y).  Returns status
  // (0, LGM_SINGULAR, LGM_DB_NOCONV, LGM_NONFINITE); iters = iterations performed.
  __device__ __noinline__ int sqrt_db(int bx, int by, double tol, int maxiter, int& iters) {
    Ctx s = *this;
    int it = 0;
    const int r = s.sqrt_db_impl(bx, by, tol, maxiter, it);
    iters = it;
    mm = s.mm;
    plateau = s.plateau;
    return r;
  }
  __device__ __forceinline__ int sqrt_db_impl(int bx, int by, double tol, int maxiter, int& iters) {
    double* X = buf(bx);
    double* Y = buf(by);
    set_identity(by);
    __syncthreads();
    bool scaling = true;
    const double two_n = 2.0 * n;
    iters = 0;
    for (int it = 1; it <= maxiter; ++it) {
      iters = it;
      double r[NMAX];
      // team 0 loads X, team 1 loads Y (skipped at it == 1: Y = I, Y^-1 = I, log|det| = 0)
      const bool active = (team == 0) || (it > 1);
      bool bad = false;
      if (!active) {
#pragma unroll
        for (int j = 0; j < NMAX; ++j) r[j] = 0.0;
      } else {
        const double* S = team == 0 ? X : Y;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
          double v = (row < n && j < n) ? S[row * C::LDM + j] : 0.0;
          bad |= !isfinite(v);
          r[j] = v;
        }
      }
      int st = __syncthreads_or(bad) ? 4 : 0;
      if (st) { iters = it - 1; return LGM_NONFINITE; }  // as_square inside lu_factor (matcore.py:122)
      double logdet = 0.0;
      int my_step = -1, sing = 0;
      {
        LGM_PHASE_BEGIN(*this);
        if (active) sing = gj_invert(r, logdet, my_step);
        LGM_PHASE_END(*this, 7);
      }
      if (tid == 0) { misc()[MI_STATUS] = 0; }
      __syncthreads();
      if (active && row == 0 && wit == 0) {
        red()[RD_LOGDET + 2 * team] = logdet;
        if (sing) atomicOr(&misc()[MI_STATUS], 1);
      }
      if (!active && row == 0 && wit == 0) red()[RD_LOGDET + 2 * team] = 0.0;
      __syncthreads();
      if (misc()[MI_STATUS]) { iters = it - 1; return LGM_SINGULAR; }
      const double lx = red()[RD_LOGDET], ly = red()[RD_LOGDET + 2];
      double mu = 1.0;
      if (scaling) mu = fmin(fmax(exp(-(lx + ly) / two_n), LGM_MU_MIN), LGM_MU_MAX);
      const double inv_mu = 1.0 / mu;
      // team 0 (holds X^-1, permuted) forms Y' = (mu Y + X^-1/mu)/2 in place;
      // team 1 (holds Y^-1, permuted; or I at it == 1) forms X' = (mu X + Y^-1/mu)/2 in place
      // and the column sums of |X' - X| and |X'|.
      // (register-lean: the inverse row in r[] is overwritten by |X' - X|, then by |X'|)
      const int* pv = piv(team);
      if (team == 0) {
        if (row < n) {
          const int q = my_step;
#pragma unroll
          for (int j = 0; j < NMAX; ++j) {
            if (j < n) {
              double* y = &Y[q * C::LDM + pv[j]];
              *y = 0.5 * (mu * *y + r[j] * inv_mu);
            }
          }
        }
      } else {
        const int q = (it == 1) ? row : my_step;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
          double dj = 0.0;
          if (row < n && j < n) {
            const int col = (it == 1) ? j : pv[j];
            double* x = &X[q * C::LDM + col];
            double xo = *x;
            double yi = (it == 1) ? ((col == row) ? inv_mu : 0.0) : r[j] * inv_mu;
            double xn = 0.5 * (mu * xo + yi);
            *x = xn;
            dj = fabs(xn - xo);
          }
          r[j] = dj;
        }
      }
      __syncthreads();  // X' and Y' complete
      // ||X' - X||_1 (team 1, butterfly over the registers) and ||X'||_1 (team 0: column per
      // thread, rows in order -- numpy's axis-0 reduction order) in parallel
      if (team == 1) {
        const double change = colsum_max(r);
        if (wit == 0 && lane == 0) red()[RD_CHANGE] = change;
      } else {
        double acc = 0.0;
        if (row < n) {
          for (int i = 0; i < n; ++i) acc += fabs(X[i * C::LDM + row]);
        }
        double m = lgm_warp_max(acc);
        if (C::T > 1) {
          if (lane == 0) red()[RD_SCALE + wit] = m;
          team_sync();
          m = fmax(red()[RD_SCALE], red()[RD_SCALE + 1]);
        }
        if (wit == 0 && lane == 0) red()[RD_SCALE + 2] = m;
      }
      __syncthreads();
      const double change = red()[RD_CHANGE], size = red()[RD_SCALE + 2];
      __syncthreads();
      if (size == 0.0) return LGM_DB_NOCONV;  // sqrtm.py:69-70
      const double rel = change / size;
      note(rel, LGM_SCALING_SWITCH);
      if (rel < LGM_SCALING_SWITCH) scaling = false;
      note(rel, tol);
      if (tol / 10.0 <= rel && rel <= 10.0 * tol) plateau++;
      if (rel <= tol) return 0;
    }
    return LGM_DB_NOCONV;  // sqrtm.py:76-78
  }

  // ---- block 1-norm estimator (matcore.py:234-311) -------------------------------------
  // Operator = M1^p1 [* AmI] where M1 = buf(b1) - sh1*I and AmI = buf(bA) - I (if has2).
  // Returns the estimate (uniform); passes += total_power per apply.
  __device__ double mat_el(const double* M, int i, int j, double sh) const {
    double v = M[i * C::LDM + j];
    return (i == j) ? v - sh : v;
  }

  // p successive thin products x <- M x (row-per-thread; M^T x: column-per-thread) for the
  // team's estimator column.  The thread's row (column) of M is held in registers across
  // the p products; x ping-pongs between xa and xb (smem, zero beyond n); on return xa
  // holds the result.  Inlined at a single call site in estimate_impl (a non-inlined callee
  // gets a reduced register budget under the ABI and serialises the x loads).
  __device__ __forceinline__ void apply_pow(MRef M, int p, bool trans, double*& xa, double*& xb) {
    double m[NMAX];
    const bool ok = row < n;
    if (trans) {
#pragma unroll
      for (int j = 0; j < NMAX; ++j) m[j] = (ok && j < n) ? M.p[j * M.ld + row] : 0.0;
    } else {
#pragma unroll
      for (int j = 0; j < NMAX; ++j) m[j] = (ok && j < n) ? M.p[row * M.ld + j] : 0.0;
    }
    for (int q = 0; q < p; ++q) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int j = 0; j < NMAX; j += 4) {
        const double2 x01 = *reinterpret_cast<const double2*>(xa + j);
        const double2 x23 = *reinterpret_cast<const double2*>(xa + j + 2);
        a0 = fma(m[j], x01.x, a0);
        a1 = fma(m[j + 1], x01.y, a1);
        a2 = fma(m[j + 2], x23.x, a2);
        a3 = fma(m[j + 3], x23.y, a3);
      }
      if (ok) xb[row] = (a0 + a1) + (a2 + a3);
      team_sync();
      double* tt = xa;
      xa = xb;
      xb = tt;
    }
  }

  // op = M1^p1 [* MA]: forward applies MA (if has2) then M1^p1; the adjoint applies
  // (M1^T)^p1 then MA^T.  One loop over the two stages so apply_pow is inlined once.
  // (x vectors passed as shared-memory offsets so the accesses compile to LDS/STS, not
  // generic loads through an address-taken pointer)
  __device__ __noinline__ void apply_seq(MRef b1, int p1, bool has2, MRef bA, bool trans, int& oa, int& ob) {
    Ctx s = *this;
    double* xa = sm() + oa;
    double* xb = sm() + ob;
#pragma unroll 1
    for (int st = 0; st < 2; ++st) {
      const bool use_a = trans ? (st == 1) : (st == 0);
      if (use_a && !has2) continue;
      s.apply_pow(use_a ? bA : b1, use_a ? 1 : p1, trans, xa, xb);
    }
    oa = (int)(xa - sm());
    ob = (int)(xb - sm());
  }

  // buf(dst) = buf(src) - I, element-exact like numpy's B - I
  __device__ void minus_identity(int dst, int src) {
    double* D = buf(dst);
    const double* S = buf(src);
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
        double v = S[i * C::LDM + j];
        D[i * C::LDM + j] = (i == j) ? v - 1.0 : v;
      }
  }

  __device__ bool any_nonzero_ref(MRef M) {
    bool nz = false;
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) nz |= M.p[i * M.ld + j] != 0.0;
    return __syncthreads_or(nz);
  }

  __device__ bool any_nonzero(int b, double sh) {
    bool nz = false;
    const double* M = buf(b);
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
      nz |= mat_el(M, i, j, sh) != 0.0;
    }
    return __syncthreads_or(nz);
  }

  // Operator = M1^p1 [* MA] with M1 = buf(b1), MA = buf(bA) (matrices stored explicitly,
  // e.g. A - I materialised like numpy's B - I).
  __device__ __noinline__ double estimate(MRef b1, int p1, bool has2, MRef bA, int itmax, int& passes) {
    Ctx s = *this;
    int ps = passes;
    LGM_PHASE_BEGIN(*this);
    const double e = s.estimate_impl(b1, p1, has2, bA, itmax, ps);
    LGM_PHASE_END(*this, 6);
    passes = ps;
    mm = s.mm;
    return e;
  }
  __device__ __forceinline__ double estimate_impl(MRef b1, int p1, bool has2, MRef bA, int itmax, int& passes) {
    const int t = n < 2 ? n : 2;
    const int total = p1 + (has2 ? 1 : 0);
    // vec layout: col c uses vec(2c) / vec(2c+1) ping-pong; vec(4), vec(5) = Z cols; vec(7) = h
    double* h = vec(7);
    int* order = misc() + MI_ORDER;
    // initial block X (matcore.py:265-271)
    {
      const double inv_n = 1.0 / n;
      for (int i = tid; i < n; i += C::NT) {
        vec(0)[i] = inv_n;
        if (t > 1) vec(2)[i] = vec(8)[i];  // normalised ramp, built once per matrix (init_ramp)
      }
    }
    __syncthreads();
    double est = 0.0;
    int best_j = 0, ncols = t;
    uint64_t hist = 0ull;
    for (int sweep = 0; sweep < itmax; ++sweep) {
      // ---- forward: Y = op(X), team c handles column c
      int cur = 0;
      if (team < ncols) {
        double* xa = vec(2 * team);
        double* xb = vec(2 * team + 1);
        {
          LGM_PHASE_BEGIN(*this);
          int oa = (int)(xa - sm()), ob = (int)(xb - sm());
          apply_seq(b1, p1, has2, bA, false, oa, ob);
          xa = sm() + oa;
          xb = sm() + ob;
          LGM_PHASE_END(*this, 5);
        }
        cur = (p1 + (has2 ? 1 : 0)) & 1;
        // column 1-norm (axis-0 sum); team reduction
        double v = (row < n) ? fabs(xa[row]) : 0.0;
        v = lgm_warp_sum(v);
        if (lane == 0) red()[RD_CN + team * 2 + wit] = v;
      }
      passes += total;
      __syncthreads();
      double cn[2] = {0.0, 0.0};
      for (int c = 0; c < ncols; ++c) {
        cn[c] = red()[RD_CN + c * 2];
        if (C::T > 1) cn[c] += red()[RD_CN + c * 2 + 1];
      }
      const int yb = cur;  // Y column c is in vec(2c + yb)
      int j = (ncols > 1 && cn[1] > cn[0]) ? 1 : 0;
      if (ncols > 1) gap(cn[0], cn[1]);
      double cand = cn[j];
      if (est > 0.0) gap(cand, est);
      if (cand > est) { est = cand; best_j = j; }
      else if (sweep > 0) break;
      // ---- adjoint: Z = op^T(sign(Y))
      if (team < ncols) {
        double* ya = vec(2 * team + yb);
        double* yb2 = vec(2 * team + (yb ^ 1));
        if (row < n) ya[row] = (ya[row] >= 0.0) ? 1.0 : -1.0;  // matcore.py:231
        team_sync();
        double* xa = ya;
        double* xb = yb2;
        {
          LGM_PHASE_BEGIN(*this);
          int oa = (int)(xa - sm()), ob = (int)(xb - sm());
          apply_seq(b1, p1, has2, bA, true, oa, ob);
          xa = sm() + oa;
          xb = sm() + ob;
          LGM_PHASE_END(*this, 5);
        }
        if (row < n) vec(4 + team)[row] = xa[row];
      }
      passes += total;
      __syncthreads();
      // h = row max |Z|, top-(4t+1) order (desc, ties -> lowest index) by warp 0
      for (int i = tid; i < n; i += C::NT) {
        double hv = fabs(vec(4)[i]);
        if (ncols > 1) hv = fmax(hv, fabs(vec(5)[i]));
        h[i] = hv;
      }
      __syncthreads();
      const int ntop = n < 4 * t + 1 ? n : 4 * t + 1;
      if (warp == 0) {
        uint64_t taken = 0ull;
        for (int q = 0; q < ntop; ++q) {
          // lane examines rows lane and lane + 32
          uint64_t kbest = 0ull;
          int rbest = 1 << 30;
#pragma unroll
          for (int e = 0; e < NMAX / 32; ++e) {
            int i = lane + 32 * e;
            if (i < n && !((taken >> i) & 1ull)) {
              uint64_t kk = lgm_key(h[i]);
              if (kk > kbest) { kbest = kk; rbest = i; }
            }
          }
          int wl;
          uint64_t kmax = lgm_warp_argmax(kbest, wl);
          unsigned tie = __ballot_sync(0xffffffffu, kbest == kmax);
          int rsel = (kbest == kmax) ? rbest : (1 << 30);
          rsel = __reduce_min_sync(0xffffffffu, (unsigned)rsel);
          (void)tie; (void)wl;
          taken |= 1ull << rsel;
          if (lane == 0) { order[q] = rsel; red()[RD_H + q] = lgm_unkey(kmax); }
        }
      }
      __syncthreads();
      for (int a = 0; a + 1 < ntop && a < 4 * t; ++a) gap(red()[RD_H + a], red()[RD_H + a + 1]);
      int picks[2], npick = 0;
      for (int q = 0; q < (ntop < 4 * t ? ntop : 4 * t) && npick < t; ++q) {
        int i = order[q];
        if (!((hist >> i) & 1ull)) picks[npick++] = i;
      }
      const double h0 = h[order[0]], hb = h[best_j];
      if (sweep > 0 && order[0] != best_j) gap(h0, hb);
      if (npick == 0 || (sweep > 0 && h0 <= hb)) break;
      __syncthreads();
      for (int c = 0; c < npick; ++c) hist |= 1ull << picks[c];
      ncols = npick;
      for (int i = tid; i < n; i += C::NT) {
        vec(0)[i] = (i == picks[0]) ? 1.0 : 0.0;
        if (npick > 1) vec(2)[i] = (i == picks[1]) ? 1.0 : 0.0;
      }
      __syncthreads();
    }
    __syncthreads();
    return est;
  }

  // ---- degree-optimal polynomial (schemes.py:104-126) -----------------------------------
  // Nodes P1 = I, P2 = buf(bX), P3 = buf(b3), P4..P6 = ext + (t-4)*ext_stride (row stride
  // ext_ld; shared or a global workspace slot).  All node addressing is arithmetic on the
  // (compile-time) slot index t, so no local-memory arrays are involved.
  struct Nodes {
    const double* p2;
    const double* p3;
    int p3_ld;
    double* ext;
    int ext_ld, ext_stride;
    __device__ __forceinline__ const double* ptr(int t) const {
      return t == 2 ? p2 : (t == 3 ? p3 : ext + (t - 4) * ext_stride);
    }
    __device__ __forceinline__ int ld(int t) const { return t == 2 ? C::LDM : (t == 3 ? p3_ld : ext_ld); }
  };
  // nodes P2..P_{TM}: TM = 7 for the shipped schemes k <= 5, LGM_K_MAX + 2 for k = 6..9 (a
  // separate instantiation so the k <= 5 path keeps its register allocation)
  static constexpr int TM5 = 7, TM9 = LGM_K_MAX + 2;

  // Polynomial GEMMs on the FP64 tensor cores (mma.sync m8n8k4 -> DMMA): warp w owns output
  // rows 16w .. 16w+15 (two 8-row tiles) x all NMAX/8 column tiles, so every left-operand
  // element is formed once per CTA; acc[(mi * FT + ni) * 2 + e] = C[frow(mi)][fcol(ni, e)].
  // A right operand materialised by combine_rhs uses a swizzled layout (row stride NMAX,
  // column c of row k stored at c ^ 4(k & 3)): the row-per-warp writes and the B fragment
  // reads (rows t, columns g) are both bank-conflict free.
  static constexpr int FT = NMAX / 8;  // column tiles
  __device__ __forceinline__ static int swz(int k, int c) { return k * NMAX + (c ^ ((k & 3) << 2)); }
  __device__ __forceinline__ int frow(int mi) const { return 16 * warp + 8 * mi + (lane >> 2); }
  __device__ __forceinline__ int fcol(int ni, int e) const { return 8 * ni + 2 * (lane & 3) + e; }

  // acc = L * R with L = sum_{t=2..nn} crow[t-1] * P_t + crow[0] * I formed on the fly with
  // numpy's _combine rounding (schemes.py:91-101: sequential over t, zero coefficients
  // skipped, products and sums rounded separately).  R: swizzled (rswz) or row stride LDM.
  template <int TMAX>
  __device__ void gemm_comb(const Nodes& nd, int nn, const double* crow, const double* R, bool rswz,
                            double (&acc)[NMAX / 2]) {
#pragma unroll
    for (int q = 0; q < NMAX / 2; ++q) acc[q] = 0.0;
    double cf[TMAX - 1];
#pragma unroll
    for (int t = 2; t <= TMAX; ++t) cf[t - 2] = (t <= nn) ? crow[t - 1] : 0.0;
    const double l0 = crow[0];
    const int t4 = lane & 3;
#pragma unroll 2
    for (int k0 = 0; k0 < n; k0 += 4) {
      const int kk = k0 + t4;
      double a[2], b[FT];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int i = frow(mi);
        double l = 0.0;
        if (i < n && kk < n) {
#pragma unroll
          for (int t = 2; t <= TMAX; ++t)
            if (cf[t - 2] != 0.0) l = __dadd_rn(l, __dmul_rn(cf[t - 2], nd.ptr(t)[i * nd.ld(t) + kk]));
          if (kk == i && l0 != 0.0) l = __dadd_rn(l, l0);
        }
        a[mi] = l;
      }
#pragma unroll
      for (int ni = 0; ni < FT; ++ni) {
        const int c = 8 * ni + (lane >> 2);
        b[ni] = (kk < n && c < n) ? R[rswz ? swz(kk, c) : kk * C::LDM + c] : 0.0;
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < FT; ++ni)
          lgm_dmma(*reinterpret_cast<double(*)[2]>(&acc[(mi * FT + ni) * 2]), a[mi], b[ni]);
    }
  }

  // D (swizzled) = sum_{t=2..nn} crow[t-1] P_t + crow[0] I (schemes.py:91-101 order)
  template <int TMAX>
  __device__ void combine_rhs(double* D, const Nodes& nd, int nn, const double* crow) {
    double cf[TMAX - 1];
#pragma unroll
    for (int t = 2; t <= TMAX; ++t) cf[t - 2] = (t <= nn) ? crow[t - 1] : 0.0;
    const double c0 = crow[0];
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
        double v = 0.0;
#pragma unroll
        for (int t = 2; t <= TMAX; ++t)
          if (cf[t - 2] != 0.0) v = __dadd_rn(v, __dmul_rn(cf[t - 2], nd.ptr(t)[i * nd.ld(t) + j]));
        if (i == j && c0 != 0.0) v = __dadd_rn(v, c0);
        D[swz(i, j)] = v;
      }
  }

  __device__ void store_frag(double* D, int ld, const double (&acc)[NMAX / 2]) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < FT; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = frow(mi), c = fcol(ni, e);
          if (i < n && c < n) D[i * ld + c] = acc[(mi * FT + ni) * 2 + e];
        }
  }

  // P2 = X in buf(bX), P3 = X^2 in buf(b3) (computed here if !have_fp: one product), R temp
  // buf(bR), P4..P6 in `ext`.  The last node stays in registers; the epilogue forms z,
  // scales by `mult` (= -2^s), reverts the balancing (matcore.py:175-177) when `unbal` is
  // set, stages through R and writes row-major to Lg (ld).
  __device__ __noinline__ void degopt(int k, int bX, MRef b3, bool have_fp, int bR, double* ext, int ext_ld,
                                      int ext_stride, double mult, bool unbal, double* Lg, long long ldg,
                                      int& products) {
    Ctx s = *this;
    if (k <= 5) s.degopt_impl<TM5>(k, bX, b3, have_fp, bR, ext, ext_ld, ext_stride, mult, unbal, Lg, ldg, products);
    else s.degopt_impl<TM9>(k, bX, b3, have_fp, bR, ext, ext_ld, ext_stride, mult, unbal, Lg, ldg, products);
  }
  template <int TMAX>
  __device__ __forceinline__ void degopt_impl(int k, int bX, MRef b3, bool have_fp, int bR, double* ext, int ext_ld,
                                              int ext_stride, double mult, bool unbal, double* Lg, long long ldg,
                                              int& products) {
    Nodes nd{buf(bX), b3.p, b3.ld, ext, ext_ld, ext_stride};
    double* R = buf(bR);
    double acc[NMAX / 2];
    if (!have_fp) {  // P3 = P2 * P2
      const double one[2] = {0.0, 1.0};
      gemm_comb<TMAX>(nd, 2, one, buf(bX), false, acc);
      products++;
      __syncthreads();
      store_frag(b3.p, b3.ld, acc);
      __syncthreads();
    }
    int nn = 3;  // nodes P1..P3 available
    bool last_in_regs = false;
    for (int j = 1; j < k; ++j) {
      combine_rhs<TMAX>(R, nd, nn, lgm_rhs(*P, k, j));
      __syncthreads();
      gemm_comb<TMAX>(nd, nn, lgm_lhs(*P, k, j), R, true, acc);
      products++;
      nn++;
      __syncthreads();
      if (j < k - 1) {
        store_frag(const_cast<double*>(nd.ptr(nn)), nd.ld(nn), acc);
        __syncthreads();
      } else {
        last_in_regs = true;
      }
    }
    // epilogue (fragment layout): z = sum out[t] P_t + out[0] I, L = mult * z * (scale_i /
    // scale_j) into R (row stride LDM); per element the operation order over t is numpy's
    const double* orow = lgm_out(*P, k);
    const double* sc = scale();
    {
      double cf[TMAX - 1];
#pragma unroll
      for (int t = 2; t <= TMAX; ++t) cf[t - 2] = (t <= nn) ? orow[t - 1] : 0.0;
      double z[NMAX / 2];
#pragma unroll
      for (int q = 0; q < NMAX / 2; ++q) z[q] = 0.0;
#pragma unroll
      for (int t = 2; t <= TMAX; ++t) {
        if (cf[t - 2] != 0.0) {
          const bool regs = (t == nn && last_in_regs);
          const double* src = nd.ptr(t);
          const int sld = nd.ld(t);
          double pv[NMAX / 2];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < FT; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int q = (mi * FT + ni) * 2 + e, i = frow(mi), c = fcol(ni, e);
                pv[q] = regs ? acc[q] : ((i < n && c < n) ? src[i * sld + c] : 0.0);
              }
#pragma unroll
          for (int q = 0; q < NMAX / 2; ++q) z[q] = __dadd_rn(z[q], __dmul_rn(cf[t - 2], pv[q]));
        }
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int i = frow(mi);
        const double si = unbal && i < n ? sc[i] : 1.0;
#pragma unroll
        for (int ni = 0; ni < FT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = (mi * FT + ni) * 2 + e, c = fcol(ni, e);
            if (i < n && c < n) {
              double v = z[q];
              if (i == c && orow[0] != 0.0) v = __dadd_rn(v, orow[0]);
              v = mult * v;
              // sc[] are powers of two within (1e-300, 1e300) (radix-2 balancing), so
              // sc[i] / sc[c] == sc[i] * 2^-e(c) exactly: the reciprocal is an exponent flip
              if (unbal) v = v * (si * __hiloint2double(0x7fe00000 - __double2hiint(sc[c]), 0));
              R[i * C::LDM + c] = v;
            }
          }
      }
    }
    __syncthreads();
    for (int i = warp; i < n; i += C::NT / 32)
      for (int jcol = lane; jcol < n; jcol += 32) Lg[(long long)i * ldg + jcol] = R[i * C::LDM + jcol];
  }

  // ---- load / store --------------------------------------------------------------------
  __device__ bool load(int b, const double* Ag, long long ldg) {
    double* D = buf(b);
    bool bad = false;
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
      double v = Ag[(long long)i * ldg + j];
      bad |= !isfinite(v);
      D[i * C::LDM + j] = v;
    }
    return __syncthreads_or(bad);
  }
  __device__ void store(int b, double* Dg, long long ldg) {
    const double* S = buf(b);
    for (int i = warp; i < n; i += C::NT / 32)
      for (int j = lane; j < n; j += 32) {
      Dg[(long long)i * ldg + j] = S[i * C::LDM + j];
    }
  }

  // ---- Algorithm 1 (oracle/driver.py logm_status) ----------------------------------------
  // bB: A - I (shared), bAI2: A_I2 (global workspace slot), nI2 = ||A_I2||_1 (cached per root)
  __device__ __noinline__ double alpha(MRef bB, bool have_ai2, MRef bAI2, double nA, double nI2, int m, double theta,
                          double (&cache)[32], unsigned& cvalid, int& nest, int& passes) {
    const int itmax = P->est_itmax;
    double t1, Pm;
    if (have_ai2) {
      double r2 = sqrt(nI2);
      if (le(r2, theta)) {  // Eq. 27
        t1 = r2;
        Pm = pow(nI2, (double)(m / 2));
      } else {
        if (!((cvalid >> m) & 1u)) {
          nest++;
          double e = 0.0;
          if (any_nonzero_ref(bAI2)) e = estimate(bAI2, m / 2, false, bB, itmax, passes);
          cache[m] = e; cvalid |= 1u << m;
        }
        Pm = cache[m];
        t1 = pow(Pm, 1.0 / m);
      }
    } else {
      if (!((cvalid >> m) & 1u)) {
        nest++;
        double e = 0.0;
        if (any_nonzero_ref(bB)) e = estimate(bB, m, false, bB, itmax, passes);
        cache[m] = e; cvalid |= 1u << m;
      }
      Pm = cache[m];
      t1 = pow(Pm, 1.0 / m);
    }
    note(t1, theta);
    if (t1 > theta) return t1;
    double bound = pow(Pm * nA, 1.0 / (m + 1));  // Eq. 28
    double t2;
    if (le(bound, theta)) {
      t2 = bound;
    } else {
      if (!((cvalid >> (m + 1)) & 1u)) {
        nest++;
        double e;
        if (have_ai2) {
          e = estimate(bAI2, m / 2, true, bB, itmax, passes);
        } else {
          e = 0.0;
          if (any_nonzero_ref(bB)) e = estimate(bB, m + 1, false, bB, itmax, passes);
        }
        cache[m + 1] = e; cvalid |= 1u << (m + 1);
      }
      t2 = pow(cache[m + 1], 1.0 / (m + 1));
    }
    return fmax(t1, t2);
  }

  __device__ int first_index(double x, int K) {
    for (int j = 1; j <= K; ++j)
      if (le(x, P->theta[j - 1])) return j;
    return K;
  }

  // returns k; cert = alpha certifying k
  __device__ __noinline__ int select(MRef bB, MRef bAI2, double nA, double nI2, double alpha_loop, double (&cache)[32],
                        unsigned& cvalid, int& nest, int& passes, double& cert) {
    const int K = P->max_k;
    const double* th = P->theta;
    const int* mk = P->order;
    double r2 = sqrt(nI2);
    int mK = mk[K - 1];
    int min_im;
    if ((cvalid >> mK) & 1u) {
      min_im = first_index(pow(cache[mK], 1.0 / mK), K);
      if ((cvalid >> (mK + 1)) & 1u) {
        int m2 = first_index(pow(cache[mK + 1], 1.0 / (mK + 1)), K);
        min_im = min_im > m2 ? min_im : m2;
      }
    } else {
      min_im = first_index(r2, K);
    }
    const int tabmin[LGM_K_MAX] = LGM_TABMIN_IM;
    min_im = tabmin[min_im - 1];
    note(r2, th[0]);
    min_im = (r2 > th[0]) ? (min_im > 2 ? min_im : 2) : 1;
    int max_in = K;
    double max_bound = -1.0;
    bool found = false;
    for (int j = 1; j <= K; ++j) {
      int m = mk[j - 1];
      double bnd = pow(pow(nI2, (double)(m / 2)) * nA, 1.0 / (m + 1));
      if (le(bnd, th[j - 1])) { max_in = j; max_bound = bnd; found = true; break; }
    }
    double cert_max = found ? max_bound : alpha_loop;
    if (min_im >= max_in) { cert = cert_max; return max_in; }
    for (int j = min_im; j < max_in; ++j) {
      double a = alpha(bB, true, bAI2, nA, nI2, mk[j - 1], th[j - 1], cache, cvalid, nest, passes);
      if (le(a, th[j - 1])) { cert = a; return j; }
      if (le(a, th[j])) { cert = a; return j + 1; }
    }
    cert = cert_max;
    return max_in;
  }
};

// Buffer roles in the fused logm kernel
enum { BUF_B = 0, BUF_Y = 1 };

template <int NMAX, bool FULL>
__device__ void logm_one(Ctx<NMAX, FULL>& c, const double* Ag, double* Lg, long long ld, lgm_report* rep, double* ws) {
  const LgmParams& P = *c.P;
  lgm_report R = {};
  R.balanced = P.balance;
  int n = c.n;
  c.zero_all();
  __syncthreads();
  c.init_ramp();
  // a failed matrix gets an all-NaN L: a caller ignoring the status never reads stale data
  auto fail_fill = [&]() {
    for (int i = c.warp; i < n; i += Cfg<NMAX>::NT / 32)
      for (int j = c.lane; j < n; j += 32) Lg[(long long)i * ld + j] = __longlong_as_double(0x7ff8000000000000LL);
  };
  if (c.load(BUF_B, Ag, ld)) {
    R.status = LGM_NONFINITE;
    fail_fill();
    if (c.tid == 0) *rep = R;
    return;
  }
  if (P.balance) {
    LGM_PHASE_BEGIN(c);
    R.balance_sweeps = c.balance(BUF_B, 100);
    LGM_PHASE_END(c, 0);
  } else {
    for (int i = c.tid; i < n; i += Cfg<NMAX>::NT) c.scale()[i] = 1.0;
    __syncthreads();
  }
  const int K = P.max_k;
  const double thK = P.theta[K - 1];
  const int mK = P.order[K - 1];
  const double tol = P.db_tol > 0.0 ? P.db_tol : 10.0 * n * LGM_UNIT_ROUNDOFF;
  double cache[32];  // estimates by power m (<= m_K + 1 = 29 with k = 9)
  unsigned cvalid = 0u;
  int nest = 0, passes = 0, s = 0, db_iters = 0, products = 0;
  bool have_ai2 = false;
  // A_prev / A_I2 in this matrix's workspace slot 3 (row stride n)
  const typename Ctx<NMAX, FULL>::MRef AI2{ws + (LGM_FUSED_WS - 1) * n * n, n};
  double nI2 = 0.0;
  double alpha_loop = c.onenorm(BUF_B, 1.0);
  bool finish = c.le(alpha_loop, thK);
  int status = 0;
  while (!finish && s < P.maxiter_s) {
    double nA = c.onenorm(BUF_B, 1.0);
    double a;
    {
      LGM_PHASE_BEGIN(c);
      c.minus_identity(BUF_Y, BUF_B);  // A - I materialised as numpy does (estimator operand)
      __syncthreads();
      a = c.alpha(c.bref(BUF_Y), have_ai2, AI2, nA, nI2, mK, thK, cache, cvalid, nest, passes);
      LGM_PHASE_END(c, 1);
    }
    alpha_loop = a;
    finish = c.le(a, thK);
    if (!finish) {
      {  // A_prev = B
        const double* Bm = c.buf(BUF_B);
        for (int i = c.warp; i < n; i += Cfg<NMAX>::NT / 32)
          for (int j = c.lane; j < n; j += 32) AI2.p[i * n + j] = Bm[i * Cfg<NMAX>::LDM + j];
      }
      __syncthreads();
      int its = 0;
      {
        LGM_PHASE_BEGIN(c);
        status = c.sqrt_db(BUF_B, BUF_Y, tol, P.db_maxiter, its);
        LGM_PHASE_END(c, 2);
      }
      db_iters += its;
      if (status) break;
      s++;
      // A_I2 = A_prev - 2 B + I, in place over A_prev; its 1-norm (numpy
      // order: column sums over rows in order) is cached for the next alpha / select
      {
        const double* Bm = c.buf(BUF_B);
        double cs = 0.0;
        for (int j = c.tid; j < n; j += Cfg<NMAX>::NT) {
          double acc = 0.0;
          for (int i = 0; i < n; ++i) {
            double v = AI2.p[i * n + j] - 2.0 * Bm[i * Cfg<NMAX>::LDM + j];
            if (i == j) v = v + 1.0;
            AI2.p[i * n + j] = v;
            acc = (i == 0) ? fabs(v) : acc + fabs(v);
          }
          cs = fmax(cs, acc);
        }
        cs = lgm_warp_max(cs);
        __syncthreads();
        if (c.lane == 0) c.red()[RD_NORM + c.warp] = cs;
        __syncthreads();
        nI2 = c.red()[RD_NORM];
        for (int w = 1; w < Cfg<NMAX>::NT / 32; ++w) nI2 = fmax(nI2, c.red()[RD_NORM + w]);
      }
      have_ai2 = true;
      cvalid = 0u;
      __syncthreads();
    }
  }
  R.s = s;
  R.db_iters = db_iters;
  R.divisions = 2 * db_iters;
  R.norm_estimations = nest;
  R.estimation_passes = passes;
  if (status || !finish) {
    R.status = status ? status : LGM_SCALING_MAXITER;
    R.min_margin = c.mm;
    R.db_plateau = c.plateau;
    fail_fill();
    if (c.tid == 0) *rep = R;
    return;
  }
  const double nA = c.onenorm(BUF_B, 1.0);
  c.minus_identity(BUF_Y, BUF_B);  // A - I: estimator operand in select, GEMM operand below
  __syncthreads();
  if (!have_ai2) {  // s = 0: A_I2 = (B - I)(B - I), one product
    typename Ctx<NMAX, FULL>::Nodes nd{c.buf(BUF_Y), c.buf(BUF_Y), Cfg<NMAX>::LDM, nullptr, 0, 0};  // P2 := A - I
    const double one[2] = {0.0, 1.0};
    double acc[NMAX / 2];
    c.template gemm_comb<Ctx<NMAX, FULL>::TM5>(nd, 2, one, c.buf(BUF_Y), false, acc);
    products++;
    c.store_frag(AI2.p, AI2.ld, acc);
    __syncthreads();
    nI2 = c.onenorm_ref(AI2);
  }
  double cert = 0.0;
  int k;
  {
    LGM_PHASE_BEGIN(c);
    k = c.select(c.bref(BUF_Y), AI2, nA, nI2, alpha_loop, cache, cvalid, nest, passes, cert);
    LGM_PHASE_END(c, 3);
  }
  // P2 = I - B (the schemes approximate -log(I - X), schemes.py:129-131); B is dead now.
  {
    double* Bm = c.buf(BUF_B);
    for (int i = c.warp; i < n; i += Cfg<NMAX>::NT / 32)
      for (int j = c.lane; j < n; j += 32) {
      double v = Bm[i * Cfg<NMAX>::LDM + j];
      Bm[i * Cfg<NMAX>::LDM + j] = (i == j) ? 1.0 - v : -v;
    }
  }
  __syncthreads();
  // P4..P6: this matrix's workspace slot (3 n^2 doubles, row stride n)
  {
    LGM_PHASE_BEGIN(c);
    c.degopt(k, BUF_B, AI2, true, BUF_Y, ws, n, n * n, -ldexp(1.0, s), P.balance != 0, Lg, ld, products);
    LGM_PHASE_END(c, 4);
  }
  // a non-finite logarithm (only when the estimator overflowed upstream: norms ~1e300, where
  // Algorithm 1's decisions are meaningless) is reported, not returned as a success; the
  // final L is still staged in BUF_Y
  bool bad = false;
  {
    const double* Lm = c.buf(BUF_Y);
    for (int i = c.warp; i < n; i += Cfg<NMAX>::NT / 32)
      for (int j = c.lane; j < n; j += 32) bad |= !isfinite(Lm[i * Cfg<NMAX>::LDM + j]);
  }
  bad = __syncthreads_or(bad);
  R.k = k;
  R.alpha_used = cert;
  R.products = products;
  R.norm_estimations = nest;
  R.estimation_passes = passes;
  R.min_margin = c.mm;
  R.db_plateau = c.plateau;
  R.status = bad ? LGM_NONFINITE : 0;
  if (c.tid == 0) *rep = R;
}

}  // namespace lgm
