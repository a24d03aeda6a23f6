// Shared helpers for the engine's CUDA sources (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>
#include <utility>

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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) once per (kernel, device);
// thread-safe (plans may be used from several host threads)
inline void ensure_dyn_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> done;  // ((fn, device), bytes)
  int dev = 0;
  STDA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& e : done)
    if (e.first.first == fn && e.first.second == dev && e.second >= bytes) return;
  STDA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.push_back({{fn, dev}, bytes});
}
template <typename... A>
inline void ensure_dyn_smem(void (*kern)(A...), int bytes) {
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), bytes);
}

// After kernel launches: surface configuration errors immediately.
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error{std::string(what) + ": " + cudaGetErrorString(e)};
}

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

__device__ __forceinline__ float bf16_round(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}

// ---- packed fp32 (sm_100 FFMA2): two independent round-to-nearest fp32 FMAs per instruction,
// bit-identical to two fmaf() calls; halves the issue slots of FMA-bound SIMT loops.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void f2_fma(unsigned long long& acc, unsigned long long a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}

// ---- programmatic dependent launch (PDL) -------------------------------------------
// Forward kernels are launched with launch_pdl: a kernel may become resident while the
// previous kernel of the stream drains, run its prologue (barrier init, TMEM alloc,
// weight loads), and block in grid_dep_wait() until the previous grid has completed and
// its writes are visible.  Every kernel calls grid_dep_wait() before it reads or writes
// activation memory.  Without a programmatic edge grid_dep_wait() returns immediately.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel of the stream start launching (its CTAs still wait in grid_dep_wait)
__device__ __forceinline__ void grid_dep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Programmatic dependent launch for a launch on stream st (stda_abi.cu): by default on for
// eager launches and off inside CUDA-graph capture; env STDA_PDL=1 / 0 forces it.
bool pdl_enabled(cudaStream_t st);

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                const char* what, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled(st) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw Error{std::string(what) + ": " + cudaGetErrorString(e)};
}

}  // namespace stda
