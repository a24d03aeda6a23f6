// Operand-plane helpers: border zeroing and the fused ECA gate + apply kernel.
#include <algorithm>

#include "planes.cuh"

namespace stda {
namespace {

__global__ void zero_borders_kernel(ZeroList zl, int64_t B) {
  // unit = one 16-byte position slot of one (image, plane, cg16, pass, cg8) block
  for (int i = 0; i < zl.n; ++i) {
    const PlBuf& p = zl.buf[i];
    const int per_block = 2 * (p.L + 8) + p.Hp;  // top margin, bottom margin, pad column
    const int blocks = p.planes * (p.C / 16) * p.np * 2;
    const int64_t total = B * blocks * (int64_t)per_block;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
      const int64_t bb = u / per_block;
      const int r = (int)(u - bb * per_block);
      const int64_t b = bb / blocks;
      const int blk = (int)(bb - b * blocks);
      const int plane = blk / ((p.C / 16) * p.np * 2);
      const int inner = blk - plane * ((p.C / 16) * p.np * 2);
      int q;
      if (r < p.L + 8) q = -(p.L + 8) + r;                    // rows -2/-1 region
      else if (r < 2 * (p.L + 8)) q = p.Hp * p.L + (r - (p.L + 8));  // row Hp (+ margin)
      else q = (r - 2 * (p.L + 8)) * p.L + p.Wp;              // pad column of row y
      uint16_t* dst = p.base + b * p.img_stride + (int64_t)plane * p.plane_stride +
                      ((size_t)inner * p.Q + q + p.off) * 8;
      *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  }
}

constexpr int kGateThreads = 256;
constexpr int kPixPerCta = 512;

__global__ void __launch_bounds__(kGateThreads) gate_apply_kernel(
    const float* __restrict__ gap, int items, const float* __restrict__ eca_w, int k,
    const float* __restrict__ x, PlBuf skip, int has_skip, PlBuf out_pl, int has_pl, PlBuf out_pp,
    int has_pp, float* __restrict__ out_f32, int C, int H, int W) {
  __shared__ float mean[1024];
  __shared__ float gate[1024];
  const int64_t b = blockIdx.y;
  // gate for this image: fixed-order reduction of the producer's per-item partial sums
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int t = 0; t < items; ++t) s += __ldg(gap + (b * items + t) * C + c);
    mean[c] = s / (float)(H * W);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float z = 0.f;
    for (int j = 0; j < k; ++j) {
      const int cc = c + j - k / 2;
      if (cc >= 0 && cc < C) z = fmaf(__ldg(eca_w + j), mean[cc], z);
    }
    gate[c] = 1.f / (1.f + expf(-z));
  }
  __syncthreads();
  const int G8 = C / 8;
  const int pix0 = blockIdx.x * kPixPerCta;
  const int npix = min(kPixPerCta, H * W - pix0);
  for (int u = threadIdx.x; u < npix * G8; u += blockDim.x) {
    const int pl = u / G8, c8 = u - pl * G8;
    const int pix = pix0 + pl;
    const int y = pix / W, xx = pix - y * W;
    const float* xp = x + ((size_t)b * H * W + pix) * C + c8 * 8;
    const float4 a0 = __ldg(reinterpret_cast<const float4*>(xp));
    const float4 a1 = __ldg(reinterpret_cast<const float4*>(xp) + 1);
    float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = v[i] * gate[c8 * 8 + i];  // eca(x) = x * gate
    if (has_skip) {
      float s[8];
      pl_load8(skip, b, 0, c8, y * skip.L + xx, s);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = v[i] + s[i];             // + skip (model.py:197-198)
    }
    if (has_pl) pl_store8(out_pl, b, 0, c8, y * out_pl.L + xx, v);
    if (has_pp) pl_store8(out_pp, b, (y & 1) * 2 + (xx & 1), c8, (y >> 1) * out_pp.L + (xx >> 1), v);
    if (out_f32) {
      float* op = out_f32 + ((size_t)b * H * W + pix) * C + c8 * 8;
      *reinterpret_cast<float4*>(op) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(op + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

}  // namespace

void launch_zero_borders(const ZeroList& zl, int64_t B, cudaStream_t st) {
  if (zl.n == 0 || B == 0) return;
  zero_borders_kernel<<<148 * 4, 256, 0, st>>>(zl, B);
  check_launch("zero_borders_kernel");
}

void launch_gate_apply(const float* gap, int items, const float* eca_w, int k, const float* x,
                       const PlBuf* skip, const PlBuf* out_pl, const PlBuf* out_pp, float* out_f32,
                       int64_t B, int C, int H, int W, cudaStream_t st) {
  STDA_CHECK(C % 8 == 0 && C <= 1024, "gate_apply: channel count");
  STDA_CHECK(B <= 65535, "gate_apply: batch too large for one launch");
  dim3 grid(cdiv(H * W, kPixPerCta), (unsigned)B);
  gate_apply_kernel<<<grid, kGateThreads, 0, st>>>(
      gap, items, eca_w, k, x, skip ? *skip : PlBuf{}, skip != nullptr, out_pl ? *out_pl : PlBuf{},
      out_pl != nullptr, out_pp ? *out_pp : PlBuf{}, out_pp != nullptr, out_f32, C, H, W);
  check_launch("gate_apply_kernel");
}

}  // namespace stda
