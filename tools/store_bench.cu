// Global store throughput per SM on B200 (round 2): how fast can one persistent CTA per SM
// push coalesced 16-byte stores (STG.128), as a function of the warps issuing them, vs
// cp.async.bulk shared->global stores.  The conv epilogues store ~14 B/clk/SM; this
// measures whether that is a hardware ceiling or a concurrency limit.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_bench tools/store_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stg_kernel(uint4* out, size_t n_per_cta, int iters) {
  uint4* base = out + blockIdx.x * n_per_cta;
  const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
  for (int it = 0; it < iters; ++it)
    for (size_t i = threadIdx.x; i < n_per_cta; i += blockDim.x) base[i] = v;
}

// one warp store instruction = 32 / LPR runs of LPR consecutive 16-byte lanes, the runs in
// 32 / LPR regions of the CTA's range far apart (the gate kernels' plane stores: a warp's 8
// pixels x 4 channel groups go to 4 plane blocks as 128-byte runs, LPR = 8; phase planes: 64-byte
// runs, LPR = 4)
template <int LPR>
__global__ void stg_runs_kernel(uint4* out, size_t n_per_cta, int iters) {
  constexpr int NR = 32 / LPR;
  uint4* base = out + blockIdx.x * n_per_cta;
  const size_t region = n_per_cta / NR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int run = lane / LPR, w = lane % LPR;
  const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
  for (int it = 0; it < iters; ++it)
    for (size_t i = (size_t)warp * LPR; i < region; i += (size_t)nw * LPR) base[run * region + i + w] = v;
}

__global__ void bulk_kernel(uint8_t* out, size_t bytes_per_cta, int chunk, int iters) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint8_t* base = out + blockIdx.x * bytes_per_cta;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
  for (int it = 0; it < iters; ++it) {
    for (size_t o = 0; o < bytes_per_cta; o += chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + o), "r"(src), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_cta = 1 << 20;  // 1 MB per CTA per iteration (148 MB total: beyond L2)
  const size_t small = 256 << 10;  // 256 KB per CTA (37 MB total: L2-resident)
  uint8_t* buf;
  cudaMalloc(&buf, (size_t)sms * per_cta);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t pc : {per_cta, small}) {
    const int iters = pc == per_cta ? 4 : 16;
    for (int warps : {2, 4, 8, 16, 32}) {
      stg_kernel<<<sms, warps * 32>>>((uint4*)buf, pc / 16, 1);
      cudaEventRecord(a);
      stg_kernel<<<sms, warps * 32>>>((uint4*)buf, pc / 16, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * pc * iters;
      printf("STG.128  %4zu KB/CTA warps %2d: %7.1f GB/s  %5.1f B/clk/SM (at 1.965 GHz)\n", pc >> 10, warps,
             bytes / ms / 1e6, bytes / ms / 1e-3 / sms / 1.965e9);
    }
    for (int lpr : {8, 4, 2}) {
      auto kern = lpr == 8 ? stg_runs_kernel<8> : lpr == 4 ? stg_runs_kernel<4> : stg_runs_kernel<2>;
      kern<<<sms, 512>>>((uint4*)buf, pc / 16, 1);
      cudaEventRecord(a);
      kern<<<sms, 512>>>((uint4*)buf, pc / 16, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * pc * iters;
      printf("STG.128  %4zu KB/CTA 16 warps, %3d-byte runs in %2d regions: %7.1f GB/s  %5.1f B/clk/SM\n", pc >> 10,
             lpr * 16, 32 / lpr, bytes / ms / 1e6, bytes / ms / 1e-3 / sms / 1.965e9);
    }
    for (int chunk : {4096, 16384, 32768}) {
      cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
      bulk_kernel<<<sms, 128, chunk>>>(buf, pc, chunk, 1);
      cudaEventRecord(a);
      bulk_kernel<<<sms, 128, chunk>>>(buf, pc, chunk, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * pc * iters;
      printf("bulk S2G %4zu KB/CTA chunk %5d: %7.1f GB/s  %5.1f B/clk/SM\n", pc >> 10, chunk, bytes / ms / 1e6,
             bytes / ms / 1e-3 / sms / 1.965e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
