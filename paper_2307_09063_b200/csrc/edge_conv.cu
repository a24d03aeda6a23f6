// Edge layers of the tensor-core path: the stem (F frames -> c0 channels, temporal
// fusion, reference model.py:144-147) and the head (c0 -> 1, model.py:158,199).  Both
// are too narrow for the tensor cores (Cin = 3 / Cout = 1) and bandwidth-shaped, so
// they are dedicated FP32 SIMT kernels around the NHWC layout of the tcgen05 layers.
//
// Tile = 8 rows x 64 columns, 256 threads, 2 output pixels (rows r and r+4) per thread.
#include <algorithm>

#include "edge_conv.cuh"

namespace stda {
namespace {

constexpr int kTH = 8, kTW = 64, kThreads = 256;
constexpr int kIH = kTH + 2, kIW = kTW + 2;  // staged halo tile

// stem: x (Src: NCHW or window strides) -> relu(conv) written as operand planes:
// PL over H x W (stage-1 conv input) and PP phase planes (stage-2 residual input).
// weights: SIMT layout with cob = 16: [blk][ci][tap][16], bias [C0].
__global__ void __launch_bounds__(kThreads) stem_planes_kernel(const float* __restrict__ w,
                                                               const float* __restrict__ bias, Src x,
                                                               int F, int C0, PlBuf pl, PlBuf pp,
                                                               int H, int W, int bf16, int64_t b_base) {
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                       // [F][kIH][kIW]
  float* ws = xs + F * kIH * kIW;       // [F][9][16]
  const int tid = threadIdx.x;
  const int ty0 = blockIdx.y * kTH, tx0 = blockIdx.x * kTW;
  const int64_t b = b_base + blockIdx.z;
  for (int e = tid; e < F * kIH * kIW; e += kThreads) {
    const int ci = e / (kIH * kIW);
    const int rem = e - ci * kIH * kIW;
    const int r = rem / kIW, c = rem - r * kIW;
    const int iy = ty0 - 1 + r, ix = tx0 - 1 + c;
    float v = 0.f;
    if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
      v = __ldg(x.x + b * x.xb + (int64_t)ci * x.xc + ((int64_t)iy * W + ix) * x.xp);
      if (bf16) v = bf16_round(v);
    }
    xs[e] = v;
  }
  const int c = tid & (kTW - 1), r0 = tid / kTW;  // rows r0 and r0 + 4
  const int ox = tx0 + c;
  for (int blk = 0; blk < C0 / 16; ++blk) {
    __syncthreads();
    for (int e = tid; e < F * 144; e += kThreads) ws[e] = __ldg(w + (size_t)blk * F * 144 + e);
    __syncthreads();
    float acc[2][16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[0][q] = acc[1][q] = __ldg(bias + blk * 16 + q);
    for (int ci = 0; ci < F; ++ci) {
      const float* xc = xs + ci * kIH * kIW;
      float v[6][3];
#pragma unroll
      for (int rr = 0; rr < 3; ++rr)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          v[rr][kx] = xc[(r0 + rr) * kIW + c + kx];
          v[rr + 3][kx] = xc[(r0 + 4 + rr) * kIW + c + kx];
        }
      const float4* wc = reinterpret_cast<const float4*>(ws + ci * 144);
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const int ky = t / 3, kx = t % 3;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 w4 = wc[t * 4 + q];
          acc[0][4 * q + 0] = fmaf(v[ky][kx], w4.x, acc[0][4 * q + 0]);
          acc[0][4 * q + 1] = fmaf(v[ky][kx], w4.y, acc[0][4 * q + 1]);
          acc[0][4 * q + 2] = fmaf(v[ky][kx], w4.z, acc[0][4 * q + 2]);
          acc[0][4 * q + 3] = fmaf(v[ky][kx], w4.w, acc[0][4 * q + 3]);
          acc[1][4 * q + 0] = fmaf(v[ky + 3][kx], w4.x, acc[1][4 * q + 0]);
          acc[1][4 * q + 1] = fmaf(v[ky + 3][kx], w4.y, acc[1][4 * q + 1]);
          acc[1][4 * q + 2] = fmaf(v[ky + 3][kx], w4.z, acc[1][4 * q + 2]);
          acc[1][4 * q + 3] = fmaf(v[ky + 3][kx], w4.w, acc[1][4 * q + 3]);
        }
      }
    }
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
      const int oy = ty0 + r0 + 4 * pr;
      if (oy >= H || ox >= W) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(acc[pr][8 * h + i], 0.f);
        pl_store8(pl, b, 0, 2 * blk + h, oy * pl.L + ox, v);
        pl_store8(pp, b, (oy & 1) * 2 + (ox & 1), 2 * blk + h, (oy >> 1) * pp.L + (ox >> 1), v);
      }
    }
  }
}

// head: u = d*g (+ s*gs) over NHWC C0 channels -> y [B][H][W] (one output channel).
// weights [9][C0] (tap-major, channel fastest), bias[1].
__global__ void __launch_bounds__(kThreads) head_nhwc_kernel(const float* __restrict__ w,
                                                             const float* __restrict__ bias,
                                                             const float* __restrict__ d,
                                                             const float* __restrict__ g,
                                                             const float* __restrict__ s,
                                                             const float* __restrict__ gs, int C0,
                                                             float* __restrict__ y, int H, int W,
                                                             int bf16, int64_t b_base) {
  extern __shared__ __align__(16) float sm[];
  const int CP = C0 + 4;                 // padded pixel stride: conflict-free float4 reads
  const int Q = C0 / 4;
  float* us = sm;                        // [kIH*kIW][CP]
  float* ws = us + kIH * kIW * CP;       // [9][C0]
  const int tid = threadIdx.x;
  const int ty0 = blockIdx.y * kTH, tx0 = blockIdx.x * kTW;
  const int64_t b = b_base + blockIdx.z;
  for (int e = tid; e < 9 * C0; e += kThreads) ws[e] = __ldg(w + e);
  for (int e = tid; e < kIH * kIW * Q; e += kThreads) {
    const int pix = e / Q, j = e - pix * Q;
    const int r = pix / kIW, c = pix - r * kIW;
    const int iy = ty0 - 1 + r, ix = tx0 - 1 + c;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
      const size_t off = (((size_t)b * H + iy) * W + ix) * C0 + 4 * j;
      const float4 dv = __ldg(reinterpret_cast<const float4*>(d + off));
      u = dv;
      if (g) {
        const float4 gv = __ldg(reinterpret_cast<const float4*>(g + (size_t)b * C0 + 4 * j));
        u = make_float4(dv.x * gv.x, dv.y * gv.y, dv.z * gv.z, dv.w * gv.w);
      }
      if (s) {
        float4 sv = __ldg(reinterpret_cast<const float4*>(s + off));
        if (gs) {
          const float4 h = __ldg(reinterpret_cast<const float4*>(gs + (size_t)b * C0 + 4 * j));
          sv = make_float4(sv.x * h.x, sv.y * h.y, sv.z * h.z, sv.w * h.w);
        }
        u = make_float4(u.x + sv.x, u.y + sv.y, u.z + sv.z, u.w + sv.w);
      }
      if (bf16)
        u = make_float4(bf16_round(u.x), bf16_round(u.y), bf16_round(u.z), bf16_round(u.w));
    }
    *reinterpret_cast<float4*>(us + pix * CP + 4 * j) = u;
  }
  __syncthreads();
  const int c = tid & (kTW - 1), r0 = tid / kTW;
  float a0 = 0.f, a1 = 0.f;
  for (int t = 0; t < 9; ++t) {
    const int ky = t / 3, kx = t % 3;
    const float* p0 = us + ((r0 + ky) * kIW + c + kx) * CP;
    const float* p1 = p0 + 4 * kIW * CP;
    const float* wt = ws + t * C0;
    for (int j = 0; j < C0; j += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(wt + j);
      const float4 u0 = *reinterpret_cast<const float4*>(p0 + j);
      const float4 u1 = *reinterpret_cast<const float4*>(p1 + j);
      a0 = fmaf(u0.x, w4.x, a0); a0 = fmaf(u0.y, w4.y, a0);
      a0 = fmaf(u0.z, w4.z, a0); a0 = fmaf(u0.w, w4.w, a0);
      a1 = fmaf(u1.x, w4.x, a1); a1 = fmaf(u1.y, w4.y, a1);
      a1 = fmaf(u1.z, w4.z, a1); a1 = fmaf(u1.w, w4.w, a1);
    }
  }
  const float bv = __ldg(bias);
  const int ox = tx0 + c;
  if (ox < W) {
    const int oy0 = ty0 + r0, oy1 = oy0 + 4;
    if (oy0 < H) y[((size_t)b * H + oy0) * W + ox] = a0 + bv;
    if (oy1 < H) y[((size_t)b * H + oy1) * W + ox] = a1 + bv;
  }
}

template <typename K>
void set_smem(K kern, size_t bytes) {
  static uint64_t configured = 0;
  int dev = 0;
  STDA_CUDA(cudaGetDevice(&dev));
  if (!(configured >> (dev & 63) & 1)) {
    STDA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured |= 1ull << (dev & 63);
  }
  (void)bytes;
}

}  // namespace

void launch_stem_planes(const float* w, const float* bias, const Src& x, int F, int C0,
                        const PlBuf& pl, const PlBuf& pp, int64_t B, int H, int W, bool bf16,
                        cudaStream_t st) {
  STDA_CHECK(C0 % 16 == 0, "stem kernel needs stem_channels % 16 == 0");
  const size_t smem = sizeof(float) * (F * kIH * kIW + F * 144);
  set_smem(stem_planes_kernel, smem);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kTH), (unsigned)std::min<int64_t>(65535, B - b0));
    stem_planes_kernel<<<grid, kThreads, smem, st>>>(w, bias, x, F, C0, pl, pp, H, W, bf16, b0);
    check_launch("stem_planes_kernel");
  }
}

void launch_head_nhwc(const float* w, const float* bias, const float* d, const float* g,
                      const float* s, const float* gs, int C0, float* y, int64_t B, int H, int W,
                      bool bf16, cudaStream_t st) {
  STDA_CHECK(C0 % 4 == 0, "head kernel needs stem_channels % 4 == 0");
  const size_t smem = sizeof(float) * ((size_t)kIH * kIW * (C0 + 4) + 9 * C0);
  set_smem(head_nhwc_kernel, smem);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kTH), (unsigned)std::min<int64_t>(65535, B - b0));
    head_nhwc_kernel<<<grid, kThreads, smem, st>>>(w, bias, d, g, s, gs, C0, y, H, W, bf16, b0);
    check_launch("head_nhwc_kernel");
  }
}

}  // namespace stda
