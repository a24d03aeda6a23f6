// Does tcgen05.mma issue rate scale with the number of issuing warps (each warp owns its
// own TMEM accumulators and commits its own MMAs)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_multiwarp tools/mma_multiwarp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

__global__ void bench(int n, int nwarps, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nwarps));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  const uint32_t tmem = tmem_holder;
  long long t0 = clock64();
  if (warp < nwarps) {
    uint32_t e;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
    const bool leader = e != 0;
    const uint32_t idesc = idesc_bf16(n);
    const uint64_t ad0 = desc(smem_u32(smem) + warp * 4096, 128 * 16 * 2 * 4, 128);
    const uint64_t bd = desc(smem_u32(smem + 48 * 1024), n * 16, 128);
    const uint32_t d = tmem + (uint32_t)(warp * n);
    uint64_t ad = ad0;
    for (int i = 0; i < iters / nwarps; ++i) {
      if (leader)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd),
                     "r"(idesc), "r"((uint32_t)(i > 0)));
      ad += 1;
      if ((i & 7) == 7) ad = ad0;
    }
    __syncwarp();
    if (leader)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  if (warp == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 8192;
  printf("N  warps  cycles/mma (aggregate per SM)\n");
  for (int n : {16, 32, 64, 128})
    for (int w : {1, 2, 4}) {
      if (w * n > 512) continue;
      bench<<<1, 128, 64 * 1024>>>(n, w, iters, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h;
      cudaMemcpy(&h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%3d %4d %8.1f\n", n, w, (double)h / iters);
    }
  return 0;
}
