// Host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/rbf_b200.h"

namespace rbf {

int set_error(int code, const char* fmt, ...);

inline int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RBF_OK;
  return set_error(RBF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count(int device);

}  // namespace rbf

#define RBF_CUDA_TRY(expr)                                  \
  do {                                                      \
    int _rc = ::rbf::cuda_check((expr), #expr);             \
    if (_rc != RBF_OK) return _rc;                          \
  } while (0)

#define RBF_LAUNCH_CHECK(what) RBF_CUDA_TRY(cudaPeekAtLastError())
