// Operand-plane helpers: border zeroing and the fused ECA gate + apply kernel.
#include <algorithm>

#include "planes.cuh"

namespace stda {
namespace {

// One CTA per (buffer, image, plane, cg16/pass/cg8 block); its threads zero the border
// positions of that block: the top margin (rows -2/-1), the bottom margin (row Hp) and
// the pad column of every row.  blocks_before[i] = first CTA index of buffer i.
__global__ void zero_borders_kernel(ZeroList zl, ZeroOffsets zo) {
  int i = 0;
  while (i + 1 < zl.n && (int64_t)blockIdx.x >= zo.blocks_before[i + 1]) ++i;
  const PlBuf& p = zl.buf[i];
  const int64_t blk = blockIdx.x - zo.blocks_before[i];  // b * blocks_per_img + inner
  uint16_t* base = p.base + blk * (int64_t)p.Q * 8;      // blocks are contiguous per image
  const int margin = p.L + 8;
  const int per_block = 2 * margin + p.Hp;
  for (int r = threadIdx.x; r < per_block; r += blockDim.x) {
    int q;
    if (r < margin) q = -margin + r;                       // rows -2/-1 region
    else if (r < 2 * margin) q = p.Hp * p.L + (r - margin);  // row Hp (+ margin)
    else q = (r - 2 * margin) * p.L + p.Wp;                // pad column of row y
    *reinterpret_cast<uint4*>(base + (size_t)(q + p.off) * 8) = make_uint4(0, 0, 0, 0);
  }
}

constexpr int kGateThreads = 256;
constexpr int kPixPerCta = 128;

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
  if (blockIdx.x == 0) {  // top / bottom margins of the output planes, once per image
    if (has_pl) pl_zero_margins(out_pl, b, threadIdx.x, blockDim.x);
    if (has_pp) pl_zero_margins(out_pp, b, threadIdx.x, blockDim.x);
  }
  constexpr int kB = 4;  // units whose loads are issued before any is consumed
  const int n = npix * G8;
  for (int u0 = threadIdx.x; u0 < n; u0 += kB * blockDim.x) {
    float4 xa[kB][2];
    float sk[kB][8];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int u = u0 + j * blockDim.x;
      if (u >= n) break;
      const int pl = u / G8, c8 = u - pl * G8;
      const int pix = pix0 + pl;
      const float* xp = x + ((size_t)b * H * W + pix) * C + c8 * 8;
      xa[j][0] = __ldg(reinterpret_cast<const float4*>(xp));
      xa[j][1] = __ldg(reinterpret_cast<const float4*>(xp) + 1);
      if (has_skip) {
        const int y = pix / W, xx = pix - y * W;
        pl_load8(skip, b, 0, c8, y * skip.L + xx, sk[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int u = u0 + j * blockDim.x;
      if (u >= n) break;
      const int pl = u / G8, c8 = u - pl * G8;
      const int pix = pix0 + pl;
      const int y = pix / W, xx = pix - y * W;
      float v[8] = {xa[j][0].x, xa[j][0].y, xa[j][0].z, xa[j][0].w,
                    xa[j][1].x, xa[j][1].y, xa[j][1].z, xa[j][1].w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = v[i] * gate[c8 * 8 + i];                 // eca(x) = x * gate
        if (has_skip) v[i] = v[i] + sk[j][i];           // + skip (model.py:197-198)
      }
      if (has_pl) pl_store8(out_pl, b, 0, c8, y * out_pl.L + xx, v);
      if (has_pp) pl_store8(out_pp, b, (y & 1) * 2 + (xx & 1), c8, (y >> 1) * out_pp.L + (xx >> 1), v);
      if (c8 == 0 && xx >= W - 2) {  // pad columns of the rows ending here
        if (has_pl && xx == W - 1) pl_zero_pos(out_pl, b, 0, y * out_pl.L + W);
        if (has_pp) pl_zero_pos(out_pp, b, (y & 1) * 2 + (xx & 1), (y >> 1) * out_pp.L + W / 2);
      }
      if (out_f32) {
        float* op = out_f32 + ((size_t)b * H * W + pix) * C + c8 * 8;
        *reinterpret_cast<float4*>(op) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(op + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
  }
}

}  // namespace

void launch_zero_borders(const ZeroList& zl, int64_t B, cudaStream_t st) {
  if (zl.n == 0 || B == 0) return;
  // (b, plane, cg16, pass, cg8) blocks of an image buffer are contiguous Q*8-element
  // blocks: img_stride = planes * blocks_per_plane * Q * 8
  ZeroOffsets zo;
  int64_t total = 0;
  for (int i = 0; i < zl.n; ++i) {
    const PlBuf& p = zl.buf[i];
    zo.blocks_before[i] = total;
    total += B * (int64_t)p.planes * (p.C / 16) * p.np * 2;
  }
  STDA_CHECK(total < (1ll << 31), "zero_borders: too many blocks");
  zero_borders_kernel<<<(unsigned)total, 128, 0, st>>>(zl, zo);
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
