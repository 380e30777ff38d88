// Engine G (n > 64): host-orchestrated batched kernels.  Declarations used by lgm_api.cu.
#pragma once
#include "lgm_common.cuh"

size_t lgm_grid_workspace_bytes(int64_t n, int64_t batch);
int lgm_grid_logm(const double* A, double* L, int64_t n, int64_t batch, int64_t ld, const LgmParams& P,
                  lgm_report* rep, void* ws, cudaStream_t s);
int lgm_grid_sqrt_db(const double* A, double* X, int64_t n, int64_t batch, int64_t ld, double tol, int maxiter,
                     int* iters, int* status, cudaStream_t s);
int lgm_grid_est(const double* M1, int p1, const double* M2, int64_t n, int64_t batch, int64_t ld, int itmax,
                 int zero_shortcut, double* est, int* passes, cudaStream_t s);
int lgm_grid_balance(const double* A, double* B, double* scale, int64_t n, int64_t batch, int64_t ld,
                     int max_sweeps, int* sweeps, cudaStream_t s);
int lgm_grid_degopt(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld, int k,
                    int* products, const LgmParams& P, cudaStream_t s);
