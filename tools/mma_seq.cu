// Replays the stride-1 conv's per-item MMA stream (9 taps x G tiles x {A_hi x [B_hi|B_lo]
// (N'=2N), A_lo x B_hi (N)}) in isolation, to compare with the in-kernel rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_seq tools/mma_seq.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ bool g_leader;
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, bool leader) {
  if (leader)
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

template <int N, int MODE>  // MODE 0: concat pair, 1: 3 passes, 2: single hi*hi
__global__ void bench(int items, int G, int L, int P, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  const uint32_t tmem = tmem_holder;
  if (warp == 0) {
    uint32_t e;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
    const bool leader = e != 0;
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 160 * 1024);
    const uint32_t lboA = P * 16;
    const uint64_t a0 = desc(sa, lboA, 128);
    const uint64_t b0 = desc(sb, (MODE == 0 ? 2 * N : N) * 16, 128);
    const uint32_t lo_units = 2 * P;
    long long t0 = clock64();
    for (int it = 0; it < items; ++it) {
      const uint32_t dslot = tmem + (it & 1) * 256;
#pragma unroll 1
      for (int t = 0; t < 9; ++t) {
        const uint64_t ad0 = a0 + (uint32_t)((t / 3) * L + (t % 3));
        const uint64_t bd = b0 + (uint32_t)t * (MODE == 2 ? 32 * N : 64 * N) / 16;
        uint64_t ad = ad0;
        uint32_t dcol = dslot;
        for (int g = 0; g < G; ++g, ad += 128, dcol += (MODE == 0 ? 2 * N : N)) {
          if (MODE == 0) {
            mma(dcol, ad, bd, idesc_bf16(2 * N), t > 0, leader);
            mma(dcol, ad + lo_units, bd, idesc_bf16(N), 1, leader);
          } else if (MODE == 1) {
            mma(dcol, ad, bd, idesc_bf16(N), t > 0, leader);
            mma(dcol, ad + lo_units, bd, idesc_bf16(N), 1, leader);
            mma(dcol, ad, bd + 2 * N, idesc_bf16(N), 1, leader);
          } else {
            mma(dcol, ad, bd, idesc_bf16(N), t > 0, leader);
          }
        }
      }
    }
    __syncwarp();
    if (leader) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    if (leader) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int MODE>
void run(int G, int L, int P, const char* name) {
  long long* d_out;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int items = 64;
  bench<N, MODE><<<148, 128, 210 * 1024>>>(items, G, L, P, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const int mmas_per_tapg = MODE == 0 ? 2 : MODE == 1 ? 3 : 1;
  const double per_item = (double)mx / items;
  printf("%-24s N=%2d G=%d  cycles/item %8.0f  cycles/(tap,g) %6.1f  cycles/MMA %5.1f\n", name, N, G, per_item,
         per_item / (9 * G), per_item / (9 * G * mmas_per_tapg));
  cudaFree(d_out);
}

int main() {
  run<16, 0>(4, 129, 776, "S1 concat (enc0.s1)");
  run<16, 1>(4, 129, 776, "S1 3-pass");
  run<16, 2>(4, 129, 776, "S1 1-pass bf16");
  run<32, 0>(4, 65, 648, "S1 concat N=32");
  run<32, 1>(4, 65, 648, "S1 3-pass N=32");
  run<64, 0>(2, 33, 328, "S1 concat N=64");
  run<64, 1>(2, 33, 328, "S1 3-pass N=64");
  return 0;
}
