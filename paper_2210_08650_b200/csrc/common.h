// Shared host helpers: thread-local error message, CUDA error checks.
#pragma once

#include <cstdarg>
#include <cstdio>

#include "hapi.h"

namespace hapi {

hapi_status set_error(hapi_status st, const char* fmt, ...);
void clear_error();
const char* last_error_cstr();

}  // namespace hapi

#define HAPI_CUDA_TRY(expr)                                                               \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ::hapi::set_error(e_ == cudaErrorMemoryAllocation ? HAPI_ERR_OUT_OF_MEMORY   \
                                                               : HAPI_ERR_CUDA,           \
                               "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),    \
                               __FILE__, __LINE__);                                       \
  } while (0)
