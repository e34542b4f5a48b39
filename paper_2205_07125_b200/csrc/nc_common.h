// Shared helpers for libneurocomm_b200: error reporting and CUDA checks.
#pragma once
#include <cstdarg>
#include <cstdio>
#include "../../include/neurocomm_b200.h"

void nc_set_error(const char* fmt, ...);

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define NC_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t nc_err_ = (expr);                                                \
    if (nc_err_ != cudaSuccess) {                                                \
      nc_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                   \
                   cudaGetErrorString(nc_err_));                                 \
      return NC_E_CUDA;                                                          \
    }                                                                            \
  } while (0)
#define NC_LAUNCH_CHECK() NC_CUDA_TRY(cudaGetLastError())
#endif

/* Force-load a module's kernels (cudaFuncGetAttributes) -- called by nc_sim_prepare,
 * see there.  One per translation unit on the step path. */
int ncx_load_exchange_kernels(void);
int ncx_load_local_kernels(void);
int ncx_load_persistent_kernels(void);
