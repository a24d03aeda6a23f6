// Transposed-conv MMA stream (2 sources x 16 taps x {A_hi x [B_hi|B_lo] (N=32), A_lo x B_hi
// (N=16)}) with optional background traffic: (a) bulk copies into shared memory, (b) four
// warps draining TMEM with tcgen05.ld — to find what slows the in-kernel MMA rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_interf tools/mma_interf.cu
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
__device__ __forceinline__ void mma(bool leader, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (leader)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
                 "r"(idesc), "r"(acc));
}

__global__ void bench(int items, int L, int P, int bg_copy, int bg_ldtm, const uint8_t* gsrc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar, cbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int i = threadIdx.x; i < 190 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  const uint32_t tmem = tmem_holder;
  if (warp == 0) {
    uint32_t e;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
    const bool leader = e != 0;
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 100 * 1024);
    const uint32_t lboA = P * 16, src_units = (2 * 2 * P * 16) >> 4, lo_units = 2 * P;
    const uint64_t a0 = desc(sa, lboA, 128), b0 = desc(sb, 32 * 16, 128);
    long long t0 = clock64();
    for (int it = 0; it < items; ++it) {
      const uint32_t dslot = tmem + (it & 1) * 256;
#pragma unroll 1
      for (int s = 0; s < 2; ++s)
#pragma unroll 1
        for (int t = 0; t < 16; ++t) {
          const int ph = t >> 2, a = (t >> 1) & 1, bb = t & 1;
          const int dy = (ph >> 1) + a - 1, dx = (ph & 1) + bb - 1;
          const uint64_t ad = a0 + s * src_units + (uint32_t)(dy * L + dx + L + 1);
          const uint64_t bd = b0 + (uint32_t)(s * 16 + t) * 64;
          const uint32_t d = dslot + (uint32_t)((s * 4 + ph) * 32);
          mma(leader, d, ad, bd, idesc_bf16(32), (t & 3) != 0 || s);
          mma(leader, d, ad + lo_units, bd, idesc_bf16(16), 1);
        }
    }
    __syncwarp();
    if (leader) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    if (leader) {
      out[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else if (warp == 1 && bg_copy) {
    // background: repeated 32 KB bulk copies global -> smem (region at 150 KB)
    if (lane == 0) {
      uint32_t ph = 0;
      while (!done) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cbar)), "r"(32768));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem + 150 * 1024)),
                     "l"(gsrc + (blockIdx.x % 64) * 32768), "r"(32768), "r"(smem_u32(&cbar)));
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&cbar)), "r"(ph));
        ph ^= 1;
      }
    }
  } else if (warp >= 2 && bg_ldtm) {
    // background: epilogue-like TMEM loads of the other slot
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256;
    float acc = 0.f;
    while (!done) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(trow));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[0]);
    }
    if (acc == 12345.f) out[1000] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d_out;
  uint8_t* gsrc;
  cudaMalloc(&d_out, 2048 * sizeof(long long));
  cudaMalloc(&gsrc, 64 * 32768);
  cudaMemset(gsrc, 0, 64 * 32768);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  const int items = 64;
  for (int bgc : {0, 1})
    for (int bgl : {0, 1}) {
      bench<<<148, 192, 190 * 1024>>>(items, 65, 264, bgc, bgl, gsrc, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("T dual concat  bg_copy=%d bg_ldtm=%d  cycles/item %8.0f  cycles/MMA-pair %6.1f\n", bgc, bgl,
             (double)mx / items, (double)mx / items / 32);
    }
  return 0;
}
