// Shared helpers for the engine's CUDA sources (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>

namespace stda {

// thread-local last-error string behind stda_last_error()
void set_error(const std::string& msg);

struct Error {
  std::string msg;
};

#define STDA_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::stda::Error{std::string(#call) + ": " + cudaGetErrorString(e_)};       \
  } while (0)

#define STDA_CHECK(cond, msg)                                                        \
  do {                                                                               \
    if (!(cond)) throw ::stda::Error{std::string(msg)};                              \
  } while (0)

// After kernel launches: surface configuration errors immediately.
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error{std::string(what) + ": " + cudaGetErrorString(e)};
}

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

__device__ __forceinline__ float bf16_round(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}

}  // namespace stda
