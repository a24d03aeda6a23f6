// Edge layers of the tensor-core path: the stem (F frames -> c0 channels, temporal
// fusion, reference model.py:144-147) and the head (c0 -> 1, model.py:158,199).  Both
// are too narrow for the tensor cores (Cin = 3 / Cout = 1) and bandwidth-shaped, so
// they are dedicated FP32 SIMT kernels.  The head is fused with the last ECA gate and
// skip add (model.py:197-199): it reduces the GAP partials itself and stages
// u = d * gate + skip straight from the decoder output and the stem's operand plane.
//
// Tile = 8 rows x 64 columns, 256 threads, 2 output pixels (rows r and r+4) per thread.
// Staging loops issue kBatch independent loads per thread before consuming them.
#include <algorithm>

#include "edge_conv.cuh"
#include "ptx.cuh"

namespace stda {
namespace {

constexpr int kTH = 8, kTW = 64, kThreads = 256;
constexpr int kIH = kTH + 2, kIW = kTW + 2;  // staged halo tile
constexpr int kBatch = 8;
constexpr int kHeadTH = 16;  // head tile rows (4 per thread x 4 thread rows)

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
  const int n = F * kIH * kIW;
  for (int e0 = tid; e0 < n; e0 += kBatch * kThreads) {
    float v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = e0 + u * kThreads;
      v[u] = 0.f;
      if (e < n) {
        const int ci = e / (kIH * kIW);
        const int rem = e - ci * kIH * kIW;
        const int r = rem / kIW, c = rem - r * kIW;
        const int iy = ty0 - 1 + r, ix = tx0 - 1 + c;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W)
          v[u] = __ldg(x.x + b * x.xb + (int64_t)ci * x.xc + ((int64_t)iy * W + ix) * x.xp);
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = e0 + u * kThreads;
      if (e < n) xs[e] = bf16 ? bf16_round(v[u]) : v[u];
    }
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
      // pad columns of the rows this thread ends (planes.cuh border contract)
      if (blk == 0 && ox >= W - 2) {
        if (ox == W - 1) pl_zero_pos(pl, b, 0, oy * pl.L + W);
        pl_zero_pos(pp, b, (oy & 1) * 2 + (ox & 1), (oy >> 1) * pp.L + W / 2);
      }
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0) {  // top / bottom margins, once per image
    pl_zero_margins(pl, b, tid, kThreads);
    pl_zero_margins(pp, b, tid, kThreads);
  }
}

// head fused with the last ECA gate and skip add:
//   y = bias + conv3x3(d * gate(d) + skip) over C0 channels, one output channel.
// d: NHWC fp32 [B][H][W][C0] (decoder output); gap: its per-item channel sums
// [B][items][C0]; skip: operand plane (PL over H x W) of the stem output.
// weights [9][C0] (tap-major, channel fastest), bias[1].
__global__ void __launch_bounds__(kThreads) head_fused_kernel(
    const float* __restrict__ w, const float* __restrict__ bias, const float* __restrict__ gap, int items,
    const float* __restrict__ eca_w, int k, const float* __restrict__ d, PlBuf skip, int C0,
    float* __restrict__ y, int H, int W, int bf16, int64_t b_base) {
  extern __shared__ __align__(16) float sm[];
  constexpr int kIH = kHeadTH + 2;       // head tile: 16 rows x 64 columns
  const int CP = C0 + 4;                 // padded pixel stride: conflict-free float4 reads
  const int G8 = C0 / 8;
  float* us = sm;                        // [kIH*kIW][CP]
  float* ws = us + kIH * kIW * CP;       // [9][C0]
  float* gate = ws + 9 * C0;             // [C0]
  float* mean = gate + C0;               // [C0]
  const int tid = threadIdx.x;
  const int ty0 = blockIdx.y * kHeadTH, tx0 = blockIdx.x * kTW;
  const int64_t b = b_base + blockIdx.z;
  for (int e = tid; e < 9 * C0; e += kThreads) ws[e] = __ldg(w + e);
  // ECA gate of this image (fixed-order reduction: identical in every CTA)
  for (int ch = tid; ch < C0; ch += kThreads) {
    float s = 0.f;
    for (int t = 0; t < items; ++t) s += __ldg(gap + (b * items + t) * C0 + ch);
    mean[ch] = s / (float)(H * W);
  }
  __syncthreads();
  for (int ch = tid; ch < C0; ch += kThreads) {
    float z = 0.f;
    for (int j = 0; j < k; ++j) {
      const int cc = ch + j - k / 2;
      if (cc >= 0 && cc < C0) z = fmaf(__ldg(eca_w + j), mean[cc], z);
    }
    gate[ch] = 1.f / (1.f + expf(-z));
  }
  __syncthreads();
  const int n = kIH * kIW * G8;
  for (int e0 = tid; e0 < n; e0 += 4 * kThreads) {
    float4 dv[4][2];
    float sv[4][8];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kThreads;
      const int pix = e / G8, c8 = e - pix * G8;
      const int r = pix / kIW, cc = pix - r * kIW;
      const int iy = ty0 - 1 + r, ix = tx0 - 1 + cc;
      ok[u] = e < n && iy >= 0 && iy < H && ix >= 0 && ix < W;
      if (ok[u]) {
        const float4* dp = reinterpret_cast<const float4*>(d + (((size_t)b * H + iy) * W + ix) * C0 + c8 * 8);
        dv[u][0] = __ldg(dp);
        dv[u][1] = __ldg(dp + 1);
        pl_load8(skip, b, 0, c8, iy * skip.L + ix, sv[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kThreads;
      if (e >= n) break;
      const int pix = e / G8, c8 = e - pix * G8;
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (ok[u]) {
        const float dd[8] = {dv[u][0].x, dv[u][0].y, dv[u][0].z, dv[u][0].w,
                             dv[u][1].x, dv[u][1].y, dv[u][1].z, dv[u][1].w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = dd[i] * gate[c8 * 8 + i] + sv[u][i];  // eca(d) + skip (model.py:197-198)
          if (bf16) v[i] = bf16_round(v[i]);
        }
      }
      float* dst = us + pix * CP + c8 * 8;
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  __syncthreads();
  // 4 consecutive output rows per thread: the 6 staged rows they need are read once
  // per (column tap, channel quad) and reused by every row tap
  const int c = tid & (kTW - 1), r0 = (tid / kTW) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int j = 0; j < C0; j += 4) {
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      float4 u[6];
#pragma unroll
      for (int rr = 0; rr < 6; ++rr)
        u[rr] = *reinterpret_cast<const float4*>(us + ((r0 + rr) * kIW + c + kx) * CP + j);
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        const float4 w4 = *reinterpret_cast<const float4*>(ws + (ky * 3 + kx) * C0 + j);
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const float4 v = u[o + ky];
          acc[o] = fmaf(v.x, w4.x, acc[o]);
          acc[o] = fmaf(v.y, w4.y, acc[o]);
          acc[o] = fmaf(v.z, w4.z, acc[o]);
          acc[o] = fmaf(v.w, w4.w, acc[o]);
        }
      }
    }
  }
  const float bv = __ldg(bias);
  const int ox = tx0 + c;
  if (ox < W) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int oy = ty0 + r0 + o;
      if (oy < H) y[((size_t)b * H + oy) * W + ox] = acc[o] + bv;
    }
  }
}

// ---- row-block versions on the bulk-copy (TMA) engine --------------------------------
// One CTA = R rows of one image; inputs are bulk-loaded contiguous row ranges, outputs of
// the stem are staged as operand-plane row images and bulk-stored (pad columns included).
constexpr int kRowThreads = 256;

__device__ __forceinline__ void split_store(uint8_t* dst_hi, uint8_t* dst_lo, const float (&v)[8], int np) {
  float hi[8], lo[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    hi[i] = bf16_round(v[i]);
    lo[i] = v[i] - hi[i];
  }
  *reinterpret_cast<uint4*>(dst_hi) = make_uint4(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]),
                                                 pack_bf16x2(hi[4], hi[5]), pack_bf16x2(hi[6], hi[7]));
  if (np == 2)
    *reinterpret_cast<uint4*>(dst_lo) = make_uint4(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]),
                                                   pack_bf16x2(lo[4], lo[5]), pack_bf16x2(lo[6], lo[7]));
}

// stem: rows [y0, y0+R) of relu(conv3x3(x)) -> PL rows (H x W grid) and PP rows (planes).
// x rows must be contiguous (x.xp == 1): frame ci row iy at x.x + b*xb + ci*xc + iy*W.
__global__ void __launch_bounds__(kRowThreads) stem_rows_kernel(const float* __restrict__ w,
                                                                const float* __restrict__ bias, Src x, int F,
                                                                int C0, PlBuf pl, PlBuf pp, int H, int W, int R,
                                                                int bf16, int64_t b_base) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t b = b_base + blockIdx.y;
  const int y0 = blockIdx.x * R;
  const int np = pl.np, nblk = (C0 / 16) * np * 2, L = W + 1, Lp = W / 2 + 1;
  auto al = [](size_t v) { return (v + 127) / 128 * 128; };
  float* xs = reinterpret_cast<float*>(smem_raw);                 // [F][R+2][W]
  float* ws = reinterpret_cast<float*>(smem_raw + al((size_t)F * (R + 2) * W * 4));  // [C0/16][F][9][16]
  uint8_t* po = reinterpret_cast<uint8_t*>(ws) + al((size_t)C0 * F * 9 * 4);
  const size_t po_blk = (size_t)R * L * 16;
  uint8_t* pp_s = po + al(nblk * po_blk);
  const size_t pp_blk = (size_t)(R / 2) * Lp * 16;
  const int r_lo = max(y0 - 1, 0), r_hi = min(y0 + R + 1, H);  // rows present in the image
  if (tid == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t rb = (uint32_t)(r_hi - r_lo) * W * 4;
    ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), rb * F);
    for (int ci = 0; ci < F; ++ci)
      ptx::bulk_g2s(ptx::smem_u32(xs + ((size_t)ci * (R + 2) + (r_lo - (y0 - 1))) * W),
                    x.x + b * x.xb + (int64_t)ci * x.xc + (int64_t)r_lo * W, rb, ptx::smem_u32(&bar));
  }
  for (int e = tid; e < C0 * F * 9; e += kRowThreads) ws[e] = __ldg(w + e);
  // rows outside the image are zero (bulk copies only cover the present rows)
  for (int ci = 0; ci < F; ++ci)
    for (int e = tid; e < W; e += kRowThreads) {
      if (y0 - 1 < 0) xs[((size_t)ci * (R + 2)) * W + e] = 0.f;
      if (y0 + R >= H) xs[((size_t)ci * (R + 2) + R + 1) * W + e] = 0.f;
    }
  if (blockIdx.x == 0) {  // top / bottom margins of the output planes, once per image
    pl_zero_margins(pl, b, tid, kRowThreads);
    pl_zero_margins(pp, b, tid, kRowThreads);
  }
  ptx::mbar_wait(ptx::smem_u32(&bar), 0);
  __syncthreads();
  for (int pix = tid; pix < R * W; pix += kRowThreads) {
    const int r = pix / W, xx = pix - r * W;
    for (int blk = 0; blk < C0 / 16; ++blk) {
      float acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = __ldg(bias + blk * 16 + q);
      for (int ci = 0; ci < F; ++ci) {
        const float* xc = xs + (size_t)ci * (R + 2) * W;
        const float4* wc = reinterpret_cast<const float4*>(ws + ((size_t)blk * F + ci) * 144);
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const int ix = xx + kx - 1;
            float v = (ix >= 0 && ix < W) ? xc[(r + ky) * W + ix] : 0.f;
            if (bf16) v = bf16_round(v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 w4 = wc[(ky * 3 + kx) * 4 + q];
              acc[4 * q + 0] = fmaf(v, w4.x, acc[4 * q + 0]);
              acc[4 * q + 1] = fmaf(v, w4.y, acc[4 * q + 1]);
              acc[4 * q + 2] = fmaf(v, w4.z, acc[4 * q + 2]);
              acc[4 * q + 3] = fmaf(v, w4.w, acc[4 * q + 3]);
            }
          }
      }
      const int plane = ((y0 + r) & 1) * 2 + (xx & 1);
      const size_t pos_pl = (size_t)(r * L + xx) * 16, pos_pp = (size_t)((r >> 1) * Lp + (xx >> 1)) * 16;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(acc[8 * h + i], 0.f);
        const int kh = (blk * np) * 2 + h;  // hi block of channel group 2*blk+h
        split_store(po + kh * po_blk + pos_pl, po + (kh + 2) * po_blk + pos_pl, v, np);
        uint8_t* ppl = pp_s + (size_t)plane * nblk * pp_blk;
        split_store(ppl + kh * pp_blk + pos_pp, ppl + (kh + 2) * pp_blk + pos_pp, v, np);
      }
    }
  }
  for (int u = tid; u < R * nblk; u += kRowThreads) {  // pad columns of the staged rows
    const int r = u / nblk, kb = u - r * nblk;
    *reinterpret_cast<uint4*>(po + kb * po_blk + (size_t)(r * L + W) * 16) = make_uint4(0, 0, 0, 0);
    if ((r & 1) == 0)
      for (int plane = 0; plane < 4; ++plane)
        *reinterpret_cast<uint4*>(pp_s + ((size_t)plane * nblk + kb) * pp_blk + (size_t)((r >> 1) * Lp + W / 2) * 16) =
            make_uint4(0, 0, 0, 0);
  }
  ptx::fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    uint16_t* img = pl.base + b * pl.img_stride;
    for (int kb = 0; kb < nblk; ++kb)
      ptx::bulk_s2g(img + ((size_t)kb * pl.Q + y0 * L + pl.off) * 8, ptx::smem_u32(po + kb * po_blk),
                    (uint32_t)po_blk);
    for (int plane = 0; plane < 4; ++plane) {
      uint16_t* pimg = pp.base + b * pp.img_stride + (int64_t)plane * pp.plane_stride;
      for (int kb = 0; kb < nblk; ++kb)
        ptx::bulk_s2g(pimg + ((size_t)kb * pp.Q + (y0 / 2) * Lp + pp.off) * 8,
                      ptx::smem_u32(pp_s + ((size_t)plane * nblk + kb) * pp_blk), (uint32_t)pp_blk);
    }
    ptx::bulk_commit();
    ptx::bulk_wait_read();
  }
}

template <typename K>
void set_smem(K kern) {
  static uint64_t configured = 0;
  int dev = 0;
  STDA_CUDA(cudaGetDevice(&dev));
  if (!(configured >> (dev & 63) & 1)) {
    STDA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured |= 1ull << (dev & 63);
  }
}

}  // namespace

void launch_stem_planes(const float* w, const float* bias, const Src& x, int F, int C0,
                        const PlBuf& pl, const PlBuf& pp, int64_t B, int H, int W, bool bf16,
                        cudaStream_t st) {
  STDA_CHECK(C0 % 16 == 0, "stem kernel needs stem_channels % 16 == 0");
  if (x.xp == 1 && H % 2 == 0 && W % 2 == 0 && W <= 1024) {
    // bulk-copy row-block path: R rows (even, dividing H) with R*W ~ 256 pixels
    int R = 2;
    while (R * 2 * W <= 256 && H % (R * 2) == 0) R *= 2;
    const int np = pl.np, nblk = (C0 / 16) * np * 2, L = W + 1, Lp = W / 2 + 1;
    auto al = [](size_t v) { return (v + 127) / 128 * 128; };
    const size_t smem = al((size_t)F * (R + 2) * W * 4) + al((size_t)C0 * F * 9 * 4) +
                        al((size_t)nblk * R * L * 16) + al((size_t)4 * nblk * (R / 2) * Lp * 16);
    STDA_CHECK(smem <= 200 * 1024, "stem: rows do not fit shared memory");
    set_smem(stem_rows_kernel);
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      dim3 grid(H / R, (unsigned)std::min<int64_t>(65535, B - b0));
      stem_rows_kernel<<<grid, kRowThreads, smem, st>>>(w, bias, x, F, C0, pl, pp, H, W, R, bf16, b0);
      check_launch("stem_rows_kernel");
    }
    return;
  }
  const size_t smem = sizeof(float) * (F * kIH * kIW + F * 144);
  set_smem(stem_planes_kernel);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kTH), (unsigned)std::min<int64_t>(65535, B - b0));
    stem_planes_kernel<<<grid, kThreads, smem, st>>>(w, bias, x, F, C0, pl, pp, H, W, bf16, b0);
    check_launch("stem_planes_kernel");
  }
}

void launch_head_fused(const float* w, const float* bias, const float* gap, int items,
                       const float* eca_w, int k, const float* d, const PlBuf& skip, int C0, float* y,
                       int64_t B, int H, int W, bool bf16, cudaStream_t st) {
  STDA_CHECK(C0 % 8 == 0, "head kernel needs stem_channels % 8 == 0");
  const size_t smem = sizeof(float) * ((size_t)(kHeadTH + 2) * kIW * (C0 + 4) + 9 * C0 + 2 * C0);
  STDA_CHECK(smem <= 200 * 1024, "head kernel: stem_channels too large for the smem tile");
  set_smem(head_fused_kernel);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kHeadTH), (unsigned)std::min<int64_t>(65535, B - b0));
    head_fused_kernel<<<grid, kThreads, smem, st>>>(w, bias, gap, items, eca_w, k, d, skip, C0, y, H, W, bf16,
                                                    b0);
    check_launch("head_fused_kernel");
  }
}

}  // namespace stda
