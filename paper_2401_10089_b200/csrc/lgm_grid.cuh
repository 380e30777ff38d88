// Engine G (n > 64): device-driven batched kernels captured into a CUDA graph.  Declarations
// used by lgm_api.cu.  Every entry point is stream-ordered (no host synchronisation) and uses
// only the caller's workspace (lgm_grid_workspace_bytes).
#pragma once
#include "lgm_common.cuh"

size_t lgm_grid_workspace_bytes(int64_t n, int64_t batch);
int lgm_grid_logm(const double* A, double* L, int64_t n, int64_t batch, int64_t ld, const LgmParams& P,
                  lgm_report* rep, void* ws, cudaStream_t s);
int lgm_grid_sqrt_db(const double* A, double* X, int64_t n, int64_t batch, int64_t ld, double tol, int maxiter,
                     int* iters, int* status, void* ws, cudaStream_t s);
int lgm_grid_est(const double* M1, int p1, const double* M2, int64_t n, int64_t batch, int64_t ld, int itmax,
                 int zero_shortcut, double* est, int* passes, void* ws, cudaStream_t s);
int lgm_grid_balance(const double* A, double* B, double* scale, int64_t n, int64_t batch, int64_t ld,
                     int max_sweeps, int* sweeps, void* ws, cudaStream_t s);
int lgm_grid_degopt(const double* X, const double* FP, double* Z, int64_t n, int64_t batch, int64_t ld, int k,
                    int* products, const LgmParams& P, void* ws, cudaStream_t s);
int lgm_grid_expm(const double* A, double* E, int64_t n, int64_t batch, int64_t ld, void* ws, cudaStream_t s);
// LGM_WS_GUARD=1: guard band (bytes) after every workspace region / slot (0 otherwise)
size_t lgm_ws_guard_bytes();
int lgm_grid_ws_guard(int64_t n, int64_t batch, void* ws, int check, unsigned long long* bad, cudaStream_t s);
// kernels executed inside Engine G graphs on the current device (synchronous read; stats only)
unsigned long long lgm_grid_exec_nodes();
