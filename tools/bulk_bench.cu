// cp.async.bulk command cost: one CTA per SM, a warp issues N copies of S bytes each from a
// (L2-resident) global buffer into shared memory, waits on one mbarrier; cycles per round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_bench tools/bulk_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bench(const uint8_t* src, size_t src_bytes, int n, int s, int rounds, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  unsigned long long t0 = clock64();
  uint32_t phase = 0;
  for (int r = 0; r < rounds; ++r) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(n * s));
    __syncwarp();
    for (int c = lane; c < n; c += 32) {
      const size_t off = ((size_t)(blockIdx.x * 7919 + r * 104729 + c * 6151) * 4096) % (src_bytes - s);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + (size_t)c * s)), "l"(src + (off & ~15ull)), "r"(s), "r"(su32(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)), "r"(phase) : "memory");
    phase ^= 1;
  }
  unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = (t1 - t0) / rounds;
}

int main() {
  size_t bytes = 64ull << 20;  // L2-resident source
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int cfgs[][2] = {{1, 2752}, {2, 2752}, {4, 2752}, {8, 2752}, {16, 2752}, {1, 22016}, {2, 11008},
                   {4, 5504}, {8, 2752}, {16, 1376}, {4, 12352}, {1, 49408}, {8, 6176}};
  for (auto& c : cfgs) {
    for (int grid : {1, 148}) {
      bench<<<grid, 64, 200 * 1024>>>(src, bytes, c[0], c[1], 200, out);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < grid; ++i) avg += h[i];
      avg /= grid;
      printf("grid %3d  n %2d x %6d B = %6d B : %8.0f cycles/round  %6.1f B/clk/SM  %6.0f cyc/copy\n", grid, c[0],
             c[1], c[0] * c[1], avg, c[0] * c[1] / avg, avg / c[0]);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
