// Engine G (n > 64) -- placeholder until the batched large-n path lands.
#include "lgm_grid.cuh"

size_t lgm_grid_workspace_bytes(int64_t, int64_t) { return 0; }
int lgm_grid_logm(const double*, double*, int64_t, int64_t, int64_t, const LgmParams&, lgm_report*, void*,
                  cudaStream_t) { return LGM_ERR_UNSUPPORTED; }
int lgm_grid_sqrt_db(const double*, double*, int64_t, int64_t, int64_t, double, int, int*, int*, cudaStream_t) {
  return LGM_ERR_UNSUPPORTED;
}
int lgm_grid_est(const double*, int, const double*, int64_t, int64_t, int64_t, int, int, double*, int*,
                 cudaStream_t) { return LGM_ERR_UNSUPPORTED; }
int lgm_grid_balance(const double*, double*, double*, int64_t, int64_t, int64_t, int, int*, cudaStream_t) {
  return LGM_ERR_UNSUPPORTED;
}
int lgm_grid_degopt(const double*, const double*, double*, int64_t, int64_t, int64_t, int, int*, const LgmParams&,
                    cudaStream_t) { return LGM_ERR_UNSUPPORTED; }
