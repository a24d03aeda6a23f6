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
#include <cstdlib>
#include <string>
#include <type_traits>

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
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
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
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
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
  if (items == kGatesReady) {
    for (int ch = tid; ch < C0; ch += kThreads) gate[ch] = __ldg(gap + b * C0 + ch);
  } else {
    for (int ch = tid; ch < C0; ch += kThreads) mean[ch] = eca_channel_sum(gap, items, C0, b, ch) / (float)(H * W);
    __syncthreads();
    for (int ch = tid; ch < C0; ch += kThreads) gate[ch] = eca_gate_of(mean, C0, ch, eca_w, k);
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
          v[i] = gate_fma(dd[i], gate[c8 * 8 + i], sv[u][i]);  // eca(d) + skip (model.py:197-198)
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
__global__ void __launch_bounds__(kRowThreads, 4) stem_rows_kernel(const float* __restrict__ w,
                                                                const float* __restrict__ bias, Src x, int F,
                                                                int C0, PlBuf pl, PlBuf pp, int H, int W, int R,
                                                                int bf16, int64_t b_base, int direct) {
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
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
  // two vertically adjacent pixels per thread: every weight read from smem feeds both
  // (the kernel is bound by shared-memory wavefronts, not FMA issue)
  for (int it = tid; it < (R / 2) * W; it += kRowThreads) {
    const int r0 = (it / W) * 2, xx = it - (it / W) * W;
    for (int blk = 0; blk < C0 / 16; ++blk) {
      // channel pairs packed for FFMA2 (same per-channel fmaf sequence, half the issues)
      unsigned long long acc2[2][8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        acc2[0][q] = acc2[1][q] = f2_pack(__ldg(bias + blk * 16 + 2 * q), __ldg(bias + blk * 16 + 2 * q + 1));
      for (int ci = 0; ci < F; ++ci) {
        const float* xc = xs + (size_t)ci * (R + 2) * W;
        const ulonglong2* wc = reinterpret_cast<const ulonglong2*>(ws + ((size_t)blk * F + ci) * 144);
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const int ix = xx + kx - 1;
          unsigned long long vv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float v = (ix >= 0 && ix < W) ? xc[(r0 + k) * W + ix] : 0.f;
            if (bf16) v = bf16_round(v);
            vv[k] = f2_pack(v, v);
          }
#pragma unroll
          for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const ulonglong2 w4 = wc[(ky * 3 + kx) * 4 + q];
              f2_fma(acc2[0][2 * q], vv[ky], w4.x);
              f2_fma(acc2[0][2 * q + 1], vv[ky], w4.y);
              f2_fma(acc2[1][2 * q], vv[ky + 1], w4.x);
              f2_fma(acc2[1][2 * q + 1], vv[ky + 1], w4.y);
            }
        }
      }
#pragma unroll
      for (int o = 0; o < 2; ++o) {
      const int r = r0 + o;
      float acc[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) f2_unpack(acc2[o][q], acc[2 * q], acc[2 * q + 1]);
      const int plane = ((y0 + r) & 1) * 2 + (xx & 1);
      const size_t pos_pl = (size_t)(r * L + xx) * 16, pos_pp = (size_t)((r >> 1) * Lp + (xx >> 1)) * 16;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(acc[8 * h + i], 0.f);
        if (direct) {  // coalesced 16-byte stores straight to the planes
          const int oy = y0 + r;
          pl_store8(pl, b, 0, 2 * blk + h, oy * L + xx, v);
          pl_store8(pp, b, plane, 2 * blk + h, (oy >> 1) * Lp + (xx >> 1), v);
          continue;
        }
        const int kh = (blk * np) * 2 + h;  // hi block of channel group 2*blk+h
        split_store(po + kh * po_blk + pos_pl, po + (kh + 2) * po_blk + pos_pl, v, np);
        uint8_t* ppl = pp_s + (size_t)plane * nblk * pp_blk;
        split_store(ppl + kh * pp_blk + pos_pp, ppl + (kh + 2) * pp_blk + pos_pp, v, np);
      }
      if (direct && blk == 0 && xx >= W - 2) {  // pad columns (planes.cuh border contract)
        const int oy = y0 + r;
        if (xx == W - 1) pl_zero_pos(pl, b, 0, oy * L + W);
        pl_zero_pos(pp, b, plane, (oy >> 1) * Lp + W / 2);
      }
      }
    }
  }
  if (direct) return;
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

// ---- stem with weights in the kernel-parameter (constant) bank (C0 = 16, F <= 4) --------
// Same row blocks and direct plane stores as stem_rows_kernel, but the 16 x F x 9 weights
// and the bias are a __grid_constant__ parameter: every FMA takes its weight straight
// from the constant bank (uniform across the warp), so the only shared-memory traffic is
// the frame rows.  ncu on stem_rows_kernel: LSU wavefronts ~80 % busy, mostly weights.
constexpr int kStemC = 16, kStemMaxF = 4;
struct alignas(16) StemConst {
  float w[kStemMaxF * 9 * kStemC];  // [ci][ky][kx][co]: channel pairs (co, co+1) are 8-byte units
  float b[kStemC];
};

// NP = 1: bf16 operands (inputs rounded, hi plane only); PL = false: phase planes only (the
// consumers of the PL copy — enc0.s1 and the head — read the phase planes instead)
template <int F, int PX, int NP, bool PL = true>
__global__ void __launch_bounds__(kRowThreads, 4) stem_const_kernel(const __grid_constant__ StemConst cw, Src x,
                                                                   PlBuf pl, PlBuf pp, int H, int W, int R,
                                                                   int64_t b_base) {
  constexpr bool bf16 = NP == 1;
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t b = b_base + blockIdx.y;
  const int y0 = blockIdx.x * R;
  const int L = W + 1, Lp = W / 2 + 1;
  float* xs = reinterpret_cast<float*>(smem_raw);  // [F][R+2][W]
  const int r_lo = max(y0 - 1, 0), r_hi = min(y0 + R + 1, H);
  if (tid == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t rb = (uint32_t)(r_hi - r_lo) * W * 4;
    ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), rb * F);
#pragma unroll
    for (int ci = 0; ci < F; ++ci)
      ptx::bulk_g2s(ptx::smem_u32(xs + ((size_t)ci * (R + 2) + (r_lo - (y0 - 1))) * W),
                    x.x + b * x.xb + (int64_t)ci * x.xc + (int64_t)r_lo * W, rb, ptx::smem_u32(&bar));
  }
#pragma unroll
  for (int ci = 0; ci < F; ++ci)  // rows outside the image are zero
    for (int e = tid; e < W; e += kRowThreads) {
      if (y0 - 1 < 0) xs[((size_t)ci * (R + 2)) * W + e] = 0.f;
      if (y0 + R >= H) xs[((size_t)ci * (R + 2) + R + 1) * W + e] = 0.f;
    }
  if (blockIdx.x == 0) {  // top / bottom margins of the output planes, once per image
    if (PL) pl_zero_margins(pl, b, tid, kRowThreads);
    pl_zero_margins(pp, b, tid, kRowThreads);
  }
  ptx::mbar_wait(ptx::smem_u32(&bar), 0);
  __syncthreads();
  // C0 = 16: one cg16, blocks (pass, cg8) at (pass * 2 + cg8) * Q (planes.cuh)
  const size_t QB = (size_t)pl.Q * 8, QBp = (size_t)pp.Q * 8;
  uint16_t* plb = PL ? pl.base + b * pl.img_stride + (size_t)pl.off * 8 : nullptr;
  uint16_t* ppb = pp.base + b * pp.img_stride + (size_t)pp.off * 8;
  for (int it = tid; it < (R / PX) * W; it += kRowThreads) {  // PX vertically adjacent pixels
    const int r0 = (it / W) * PX, xx = it - (it / W) * W;
    // channel-pair accumulators: one FFMA2 = (x broadcast) x (uniform weight pair) + pair,
    // bit-identical to two fmaf() in the same order, half the issue slots
    unsigned long long acc2[PX][kStemC / 2];
#pragma unroll
    for (int o = 0; o < PX; ++o)
#pragma unroll
      for (int j = 0; j < kStemC / 2; ++j) acc2[o][j] = *reinterpret_cast<const unsigned long long*>(&cw.b[2 * j]);
#pragma unroll
    for (int ci = 0; ci < F; ++ci) {
      const float* xc = xs + (size_t)ci * (R + 2) * W;
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int ix = xx + kx - 1;
        unsigned long long v2[PX + 2];
#pragma unroll
        for (int k = 0; k < PX + 2; ++k) {
          float t = (ix >= 0 && ix < W) ? xc[(r0 + k) * W + ix] : 0.f;
          if (bf16) t = bf16_round(t);
          v2[k] = f2_pack(t, t);
        }
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
          for (int j = 0; j < kStemC / 2; ++j) {
            const unsigned long long w2 =
                *reinterpret_cast<const unsigned long long*>(&cw.w[((ci * 3 + ky) * 3 + kx) * kStemC + 2 * j]);
#pragma unroll
            for (int o = 0; o < PX; ++o) f2_fma(acc2[o][j], v2[ky + o], w2);
          }
      }
    }
    float acc[PX][kStemC];
#pragma unroll
    for (int o = 0; o < PX; ++o)
#pragma unroll
      for (int j = 0; j < kStemC / 2; ++j) f2_unpack(acc2[o][j], acc[o][2 * j], acc[o][2 * j + 1]);
#pragma unroll
    for (int o = 0; o < PX; ++o) {
      const int oy = y0 + r0 + o;
      const int plane = (oy & 1) * 2 + (xx & 1);
      uint16_t* po = plb + (size_t)(oy * L + xx) * 8;
      uint16_t* pq = ppb + (int64_t)plane * pp.plane_stride + (size_t)((oy >> 1) * Lp + (xx >> 1)) * 8;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v8[i] = fmaxf(acc[o][8 * h + i], 0.f);
        if (PL) store8_split<NP>(po + h * QB, 2 * QB, v8);
        store8_split<NP>(pq + h * QBp, 2 * QBp, v8);
      }
      if (xx >= W - 2) {  // pad columns (planes.cuh border contract)
        if (PL && xx == W - 1) pl_zero_pos(pl, b, 0, oy * L + W);
        pl_zero_pos(pp, b, plane, (oy >> 1) * Lp + W / 2);
      }
    }
  }
}

// ---- persistent strip head (C0 = 16, W in {32, 64, 128}) ------------------------------
// One CTA per SM walks a contiguous range of strips (R = 512 / W rows x W columns; an
// image's ECA gate is computed once per CTA-image, halo rows of neighbouring strips hit
// L2).  A producer warp bulk-copies rows y0-1 .. y0+R of d (NHWC fp32: one contiguous
// range) and of the skip plane (per (pass, cg8) block one contiguous range of rows with
// their zero pad column) into a 2-stage ring, so strip i+1 is in flight while the 8
// compute warps transform and convolve strip i.  u = d * gate + skip is formed in place
// over d, channel quad j of stage pixel p stored at quad slot j ^ ((p >> 1) & 3): the
// conv's float4 reads of 8 consecutive pixels then hit 8 distinct 16-byte bank groups.
// Each compute thread produces 2 output rows of one column.
constexpr int kHsCompute = 256;              // 8 compute warps
constexpr int kHsThreads = kHsCompute + 32;  // + producer warp
constexpr int kHsC = 16;

struct HeadStrips {
  int R, SR, L, dbytes, sblk, stage;  // rows, staged rows, plane row stride, d / skip-block / stage bytes
  size_t smem;
};

__host__ __device__ constexpr HeadStrips head_strips_geom(int W) {
  HeadStrips g{};
  g.R = 2 * kHsCompute / W;
  g.SR = g.R + 2;
  g.L = W + 1;
  g.dbytes = g.SR * W * kHsC * 4;
  // (a phase-plane skip stages ceil(SR/2) rows x (W/2 + 1) positions for each of 4 planes)
  g.sblk = g.SR * g.L * 16 > 4 * ((g.SR + 1) / 2) * (W / 2 + 1) * 16 ? g.SR * g.L * 16
                                                                      : 4 * ((g.SR + 1) / 2) * (W / 2 + 1) * 16;
  g.stage = g.dbytes + 4 * g.sblk;
  g.smem = 2 * (size_t)g.stage + (9 * kHsC + kHsC + 16 * kHsC + kHsC) * 4 + 4 * 8;
  return g;
}

__device__ __forceinline__ int hs_swz(int p) { return (p >> 1) & 3; }

// d / u values of a head stage: fp32, or bf16 (DBF: the bf16 variant's d, and u — which that
// variant rounds to bf16 before the conv — stored in place at the same value index)
template <bool DBF>
__device__ __forceinline__ float4 hd_load(const float* base, size_t idx) {
  if constexpr (DBF) {
    const uint2 r = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(base) + idx);
    return make_float4(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xFFFF0000u), __uint_as_float(r.y << 16),
                       __uint_as_float(r.y & 0xFFFF0000u));
  } else {
    return *reinterpret_cast<const float4*>(base + idx);
  }
}
template <bool DBF>
__device__ __forceinline__ void hd_store(float* base, size_t idx, float4 u) {
  if constexpr (DBF)
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(base) + idx) =
        make_uint2(pack_bf16x2(u.x, u.y), pack_bf16x2(u.z, u.w));
  else
    *reinterpret_cast<float4*>(base + idx) = u;
}

// the same by byte address inside a stage
template <bool DBF>
__device__ __forceinline__ float4 hd_load_b(const uint8_t* p) {
  if constexpr (DBF) {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    return make_float4(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xFFFF0000u), __uint_as_float(r.y << 16),
                       __uint_as_float(r.y & 0xFFFF0000u));
  } else {
    return *reinterpret_cast<const float4*>(p);
  }
}
template <bool DBF>
__device__ __forceinline__ void hd_store_b(uint8_t* p, float4 u) {
  if constexpr (DBF)
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(u.x, u.y), pack_bf16x2(u.z, u.w));
  else
    *reinterpret_cast<float4*>(p) = u;
}

struct HeadConst {
  float w[9 * kHsC];  // [tap][channel]: read by the conv from the kernel-parameter bank
};

// SKIP_PP: the skip (stem output) comes as phase planes: staged per row and px plane as
// [block][row][px][W/2] (2 copies per row and block, issued by the producer warp's lanes)
template <int W, bool SKIP_PP = false, bool DBF = false>
__global__ void __launch_bounds__(kHsThreads, 1) head_strips_kernel(
    const __grid_constant__ HeadConst cw, const float* __restrict__ bias, const float* __restrict__ gap, int items,
    const float* __restrict__ eca_w, int k, const float* __restrict__ d, PlBuf skip, float* __restrict__ y,
    int64_t B, int H, int bf16) {
  using namespace ptx;
  extern __shared__ __align__(128) uint8_t hsm[];
  constexpr HeadStrips g = head_strips_geom(W);
  constexpr int R = g.R, SR = g.SR, L = g.L;
  float* ws = reinterpret_cast<float*>(hsm + 2 * (size_t)g.stage);  // [9][16]
  float* gate = ws + 9 * kHsC;                                       // [16]
  float* part = gate + kHsC;                                         // [16 groups][16]
  float* mean = part + 16 * kHsC;                                    // [16]
  uint64_t* full = reinterpret_cast<uint64_t*>(mean + kHsC);         // [2]
  uint64_t* empty = full + 2;                                        // [2]
  const int tid = threadIdx.x, warp = tid >> 5;
  const int spi = H / R;  // strips per image
  const int64_t n_strips = B * spi;
  const int64_t s_begin = blockIdx.x * n_strips / gridDim.x;
  const int64_t s_end = (blockIdx.x + 1) * n_strips / gridDim.x;
  const int np = skip.np;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kHsCompute / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  grid_dep_wait();  // d, gap and skip come from the previous kernels

  if (warp == kHsCompute / 32 && SKIP_PP) {
    // ===== producer warp, phase-plane skip: lane 0 posts the bytes, lanes issue the copies.
    // The strip's staged rows of one parity py are consecutive rows of the py planes, so
    // per (block, py, px) ONE copy of those plane rows (with their pad column): the stage
    // holds [block][py*2+px][plane row][Lp] (hs_pp_row() maps a staged row to its slot)
    const int lane = tid & 31;
    constexpr int Lp = W / 2 + 1;
    int i = 0;
    for (int64_t s = s_begin; s < s_end; ++s, ++i) {
      const int st = i & 1;
      mbar_wait(smem_u32(&empty[st]), ((i >> 1) & 1) ^ 1);
      const int64_t b = s / spi;
      const int y0 = (int)(s - b * spi) * R;
      const int r0 = y0 == 0 ? 1 : 0;
      const int r1 = y0 + R == H ? SR - 1 : SR;
      const int nr = r1 - r0, iy0 = y0 - 1 + r0;
      const int n0 = (nr + 1 - (iy0 & 1)) / 2, n1 = nr - n0;  // staged rows of parity 0 / 1
      const uint32_t bar = smem_u32(&full[st]);
      uint8_t* base = hsm + (size_t)st * g.stage;
      if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(nr * W * kHsC * (DBF ? 2 : 4) + np * 2 * 2 * nr * Lp * 16));
      __syncwarp();
      const uint16_t* simg = skip.base + b * skip.img_stride;
      const int ncp = 1 + np * 2 * 4;
      for (int c = lane; c < ncp; c += 32) {
        if (c == 0) {
          bulk_g2s(smem_u32(base + (size_t)r0 * W * kHsC * (DBF ? 2 : 4)),
                   reinterpret_cast<const uint8_t*>(d) + ((size_t)b * H + iy0) * W * kHsC * (DBF ? 2 : 4),
                   (uint32_t)(nr * W * kHsC * (DBF ? 2 : 4)), bar);
          continue;
        }
        const int u = c - 1, plane = u & 3, blk = u >> 2, py = plane >> 1;
        const int pass = blk >> 1, cg8 = blk & 1;
        const int iyf = iy0 + ((iy0 & 1) != py ? 1 : 0);  // first staged row of parity py
        const int n = py ? n1 : n0;
        bulk_g2s(smem_u32(base + g.dbytes + (size_t)blk * g.sblk + (size_t)plane * ((SR + 1) / 2) * Lp * 16),
                 simg + (int64_t)plane * skip.plane_stride +
                     (skip.block_index(0, pass, cg8) + skip.off + (size_t)(iyf >> 1) * Lp) * 8,
                 (uint32_t)(n * Lp * 16), bar);
      }
    }
    return;
  }
  if (warp == kHsCompute / 32) {
    // ===== producer warp: one bulk copy per tensor (and skip block) per strip =====
    if ((tid & 31) == 0) {
      int i = 0;
      for (int64_t s = s_begin; s < s_end; ++s, ++i) {
        const int st = i & 1;
        mbar_wait(smem_u32(&empty[st]), ((i >> 1) & 1) ^ 1);
        const int64_t b = s / spi;
        const int y0 = (int)(s - b * spi) * R;
        const int r0 = y0 == 0 ? 1 : 0;                // first staged row inside the image
        const int r1 = y0 + R == H ? SR - 1 : SR;      // one past the last
        const int nr = r1 - r0, iy0 = y0 - 1 + r0;
        const uint32_t bar = smem_u32(&full[st]);
        uint8_t* base = hsm + (size_t)st * g.stage;
        mbar_arrive_expect_tx(bar, (uint32_t)(nr * W * kHsC * (DBF ? 2 : 4) + np * 2 * nr * L * 16));
        bulk_g2s(smem_u32(base + (size_t)r0 * W * kHsC * (DBF ? 2 : 4)),
                 reinterpret_cast<const uint8_t*>(d) + ((size_t)b * H + iy0) * W * kHsC * (DBF ? 2 : 4),
                 (uint32_t)(nr * W * kHsC * (DBF ? 2 : 4)), bar);
        const uint16_t* simg = skip.base + b * skip.img_stride;
        for (int pass = 0; pass < np; ++pass)
          for (int cg8 = 0; cg8 < 2; ++cg8)
            bulk_g2s(smem_u32(base + g.dbytes + (size_t)(pass * 2 + cg8) * g.sblk + (size_t)r0 * L * 16),
                     simg + (skip.block_index(0, pass, cg8) + skip.off + (size_t)iy0 * L) * 8,
                     (uint32_t)(nr * L * 16), bar);
      }
    }
    return;
  }

  // ===== 8 compute warps =====
  const float bv = __ldg(bias);
  const int cx = tid % W, rp = tid / W;  // conv: column, row pair
  // Index arithmetic hoisted out of the strip loop (the kernel is issue-bound: 2 warps per
  // scheduler, and integer address math was ~60 % of its instructions).  Transform step `it`
  // of a thread touches stage pixel p = it * 64 + tid / 4; for W >= 64 its row (it * 64) / W
  // is a compile-time constant of the unrolled loop and its column is a per-thread constant
  // plus (it * 64) % W, so every shared-memory address is base register + immediate.
  const int q = tid & 3, t4 = tid >> 2;
  constexpr bool kCtRows = W >= 64;
  // byte offsets inside a stage: d / u value quad q of pixel t4, skip bytes of pixel t4, the
  // swizzled quad of the u store (hs_swz(p) = (column >> 1) & 3: W % 8 == 0)
  const uint32_t t_d = (uint32_t)t4 * (kHsC * (DBF ? 2 : 4)) + (uint32_t)q * (DBF ? 8 : 16);
  const uint32_t t_u = (uint32_t)t4 * (kHsC * (DBF ? 2 : 4)) + (uint32_t)(q ^ ((t4 >> 1) & 3)) * (DBF ? 8 : 16);
  constexpr int SH = (SR + 1) / 2, LP = W / 2 + 1;
  const uint32_t t_s = (uint32_t)(q >> 1) * g.sblk + (uint32_t)(q & 1) * 8 +
                       (SKIP_PP ? (uint32_t)((t4 & 1) * SH * LP + (t4 >> 1)) * 16 : (uint32_t)t4 * 16);
  // conv: column cx + kx - 1 of rows 2rp .. 2rp + 3: pixel byte offset and swizzle per kx
  uint32_t c_px[3], c_sw[3];
#pragma unroll
  for (int kx = 0; kx < 3; ++kx) {
    const int xx = min(max(cx + kx - 1, 0), W - 1);
    c_px[kx] = (uint32_t)((2 * rp) * W + xx) * (kHsC * (DBF ? 2 : 4));
    c_sw[kx] = (uint32_t)((xx >> 1) & 3) * (DBF ? 8 : 16);
  }
  int64_t cur_b = -1, pre_b = -1;  // image of gate slot 0 / of slot 1 (formed ahead)
  int gsel = 0;
  int i = 0;
  for (int64_t s = s_begin; s < s_end; ++s, ++i) {
    const int st = i & 1;
    const int64_t b = s / spi;
    const int y0 = (int)(s - b * spi) * R;
    if (b != cur_b && b == pre_b) {
      gsel = 1;  // formed together with the previous image
      cur_b = b;
    } else if (b != cur_b) {
      // ECA gates (model.py:128-135) of image b and — when this CTA's strips reach it — of
      // image b + 1 in the same pass: the second image's loads fly with the first's, so the
      // CTAs whose strips span two images stop once (2-3 us) instead of twice.  Per image:
      // kEcaGroups group sums in parallel, added in group order (planes.cuh: the one
      // reduction order of every gate).  Threads 0..127 take image b, 128..255 image b + 1.
      const bool two = b + 1 <= (s_end - 1) / spi;
      const int im = tid >> 7, t7 = tid & 127;
      static_assert(kHsCompute == 2 * kEcaGroups * kHsC, "one (image, group, channel) per thread");
      float* gate2 = ws;              // [2][16] (the weight slots are unused: weights sit in the parameter bank)
      float* mean2 = ws + 2 * kHsC;   // [2][16]
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");  // previous images' gate readers
      if (items == kGatesReady) {
        if (tid < kHsC * (two ? 2 : 1)) gate2[tid] = __ldg(gap + b * kHsC + tid);
      } else {
        if (im == 0 || two) part[tid] = eca_group_sum(gap, items, kHsC, b + im, t7 % kHsC, t7 / kHsC);
        asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
        if (tid < kHsC * (two ? 2 : 1)) {
          const int mi = tid / kHsC, c = tid % kHsC;
          float a = 0.f;
          for (int grp = 0; grp < kEcaGroups; ++grp) a += part[mi * 128 + grp * kHsC + c];
          mean2[tid] = a / (float)(H * W);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
        if (tid < kHsC * (two ? 2 : 1)) {
          const int mi = tid / kHsC, c = tid % kHsC;
          gate2[tid] = eca_gate_of(mean2 + mi * kHsC, kHsC, c, eca_w, k);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
      gsel = 0;
      cur_b = b;
      pre_b = two ? b + 1 : -1;
    }
    mbar_wait(smem_u32(&full[st]), (i >> 1) & 1);
    float* ubase = reinterpret_cast<float*>(hsm + (size_t)st * g.stage);
    const uint8_t* sbase = hsm + (size_t)st * g.stage + g.dbytes;
    // transform: one (stage pixel, channel quad) per thread step, NB steps per batch: all
    // loads of a batch, one __syncwarp (the 4 quads of a pixel are lanes of one warp and
    // are rewritten in place; steps touch disjoint pixels), then all stores
    constexpr int NIT = SR * W * 4 / kHsCompute;
    static_assert(NIT * kHsCompute == SR * W * 4, "transform steps");
    constexpr int NB = NIT % 4 == 0 ? 4 : NIT % 3 == 0 ? 3 : 2;
    static_assert(NIT % NB == 0, "transform batches");
    const float4 g4 = *reinterpret_cast<const float4*>(ws + gsel * kHsC + q * 4);
    const bool top = y0 == 0, bot = y0 + R == H;  // staged row 0 / SR - 1 lies outside the image
    // phase-plane skip: staged row r sits in plane row slot r >> 1 of its parity's planes,
    // one slot earlier for even r in an image's first strip (no row above the image is staged)
    const uint32_t zoff = SKIP_PP && top ? (uint32_t)LP * 16 : 0u;
    uint8_t* ub = reinterpret_cast<uint8_t*>(ubase);
#pragma unroll
    for (int it0 = 0; it0 < NIT; it0 += NB) {
      float4 dv[NB];
      uint2 hv[NB], lv[NB];
      bool in[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if constexpr (kCtRows) {
          constexpr int VB = kHsC * (DBF ? 2 : 4);  // bytes per stage pixel
          const int it = it0 + j;
          const int r = (it * 64) / W, xc = (it * 64) % W;  // compile-time under the unroll
          in[j] = !(r == 0 && top) && !(r == SR - 1 && bot);
          dv[j] = hd_load_b<DBF>(ub + t_d + (uint32_t)(r * W + xc) * VB);
          uint32_t so;
          if (SKIP_PP)  // plane ((r + 1) & 1, column & 1), slot r >> 1 (y0 is a multiple of R, R even)
            so = (uint32_t)(((((r + 1) & 1) * 2) * SH + (r >> 1)) * LP + xc / 2) * 16 - ((r & 1) == 0 ? zoff : 0u);
          else
            so = (uint32_t)(r * L + xc) * 16;
          hv[j] = *reinterpret_cast<const uint2*>(sbase + t_s + so);
          lv[j] = np == 2 ? *reinterpret_cast<const uint2*>(sbase + t_s + so + 2 * g.sblk) : make_uint2(0u, 0u);
        } else {
          const int p = ((it0 + j) * kHsCompute + tid) >> 2;
          const int r = p / W, x = p - r * W;
          const int iy = y0 - 1 + r;
          in[j] = iy >= 0 && iy < H;
          dv[j] = hd_load<DBF>(ubase, (size_t)p * kHsC + q * 4);
          // channels 4q..4q+3: cg8 block (q >> 1), bytes (q & 1) * 8 of position r*L + x
          // (phase-plane skip: plane (iy%2, x%2), plane-row slot of iy, column x/2)
          size_t so;
          if (SKIP_PP) {
            const int py = iy & 1, iy0s = y0 - 1 + (y0 == 0 ? 1 : 0);
            const int slot = (iy >> 1) - ((iy0s + ((iy0s & 1) != py ? 1 : 0)) >> 1);
            so = ((size_t)((py * 2 + (x & 1)) * ((SR + 1) / 2) + slot) * (W / 2 + 1) + (x >> 1)) * 16 + (q & 1) * 8;
          } else {
            so = (size_t)(r * L + x) * 16 + (q & 1) * 8;
          }
          hv[j] = *reinterpret_cast<const uint2*>(sbase + (size_t)(q >> 1) * g.sblk + so);
          lv[j] = np == 2 ? *reinterpret_cast<const uint2*>(sbase + (size_t)(2 + (q >> 1)) * g.sblk + so)
                          : make_uint2(0u, 0u);
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
        if (in[j]) {
          float s4[4];
          s4[0] = __uint_as_float(hv[j].x << 16);
          s4[1] = __uint_as_float(hv[j].x & 0xFFFF0000u);
          s4[2] = __uint_as_float(hv[j].y << 16);
          s4[3] = __uint_as_float(hv[j].y & 0xFFFF0000u);
          if (np == 2) {
            s4[0] += __uint_as_float(lv[j].x << 16);
            s4[1] += __uint_as_float(lv[j].x & 0xFFFF0000u);
            s4[2] += __uint_as_float(lv[j].y << 16);
            s4[3] += __uint_as_float(lv[j].y & 0xFFFF0000u);
          }
          u.x = gate_fma(dv[j].x, g4.x, s4[0]);  // eca(d) + skip (model.py:197-198)
          u.y = gate_fma(dv[j].y, g4.y, s4[1]);
          u.z = gate_fma(dv[j].z, g4.z, s4[2]);
          u.w = gate_fma(dv[j].w, g4.w, s4[3]);
          if (bf16) {
            u.x = bf16_round(u.x);
            u.y = bf16_round(u.y);
            u.z = bf16_round(u.z);
            u.w = bf16_round(u.w);
          }
        }
        if constexpr (kCtRows) {
          const int it = it0 + j;
          hd_store_b<DBF>(ub + t_u + (uint32_t)(((it * 64) / W) * W + (it * 64) % W) * (kHsC * (DBF ? 2 : 4)), u);
        } else {
          const int p = ((it0 + j) * kHsCompute + tid) >> 2;
          hd_store<DBF>(ubase, (size_t)p * kHsC + (q ^ hs_swz(p)) * 4, u);
        }
      }
    }
    fence_proxy_async();  // generic writes of this stage before its next async refill
    asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
    // conv3x3 (model.py:158,199): rows 2rp, 2rp+1 of the strip at column cx
    // 4 independent chains per output (channel quads j), summed at the end
    float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      // a column outside the image contributes exact zeros: skip it (the border lane idles)
      if ((kx == 0 && cx == 0) || (kx == 2 && cx == W - 1)) continue;
      float4 u[4][4];  // [channel quad][row]: all loads of this column first
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
          u[j][rr] = hd_load_b<DBF>(ub + c_px[kx] + (((uint32_t)j * (DBF ? 8 : 16)) ^ c_sw[kx]) +
                                    (uint32_t)(rr * W) * (kHsC * (DBF ? 2 : 4)));
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const float* wt = &cw.w[(ky * 3 + kx) * kHsC + j * 4];
          acc0[j] = fmaf(u[j][ky].x, wt[0], acc0[j]);
          acc0[j] = fmaf(u[j][ky].y, wt[1], acc0[j]);
          acc0[j] = fmaf(u[j][ky].z, wt[2], acc0[j]);
          acc0[j] = fmaf(u[j][ky].w, wt[3], acc0[j]);
          acc1[j] = fmaf(u[j][ky + 1].x, wt[0], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].y, wt[1], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].z, wt[2], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].w, wt[3], acc1[j]);
        }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(smem_u32(&empty[st]));  // this warp is done with stage st
    float* yo = y + ((size_t)b * H + y0 + 2 * rp) * W + cx;
    yo[0] = ((acc0[0] + acc0[1]) + (acc0[2] + acc0[3])) + bv;
    yo[W] = ((acc1[0] + acc1[1]) + (acc1[2] + acc1[3])) + bv;
  }
}

// ---- column-tiled strip head (C0 = 16, W a multiple of 128 above 128) -----------------
// One CTA per SM walks a contiguous range of strips (R = 512 / TW rows x TW columns, TW =
// min(W, 128): wide maps are cut into column tiles; an image's ECA gate is computed once
// per CTA-image, halo rows/columns of neighbouring strips hit L2).  A producer warp
// bulk-copies, per staged row y0-1 .. y0+R, the row segment x0-1 .. x0+TW of d (NHWC fp32,
// in-image columns only) and of each skip-plane block (the plane's pad column / top margin
// supply the zero borders) into a 2-stage ring — lanes issue the copies in parallel — so
// strip i+1 is in flight while the 8 compute warps transform and convolve strip i.
// u = d * gate + skip is formed in place over d (zero outside the image), channel quad j of
// stage pixel p stored at quad slot j ^ ((p >> 1) & 3): the conv's float4 reads of 8
// consecutive pixels then hit 8 distinct 16-byte bank groups.  Each compute thread
// produces 2 output rows of one column.
struct HeadTiles {
  int R, SR, SW, dbytes, sblk, stage;  // rows, staged rows / columns, d / skip-block / stage bytes
  size_t smem;
};

__host__ __device__ constexpr HeadTiles head_tiles_geom(int TW) {
  HeadTiles g{};
  g.R = 2 * kHsCompute / TW;
  g.SR = g.R + 2;
  g.SW = TW + 2;
  g.dbytes = g.SR * g.SW * kHsC * 4;
  g.sblk = g.SR * g.SW * 16;
  g.stage = g.dbytes + 4 * g.sblk;
  g.smem = 2 * (size_t)g.stage + (9 * kHsC + kHsC + 16 * kHsC + kHsC) * 4 + 4 * 8;
  return g;
}

template <int TW, bool DBF = false>
__global__ void __launch_bounds__(kHsThreads, 1) head_tiles_kernel(
    const __grid_constant__ HeadConst cw, const float* __restrict__ bias, const float* __restrict__ gap, int items,
    const float* __restrict__ eca_w, int k, const float* __restrict__ d, PlBuf skip, float* __restrict__ y,
    int64_t B, int H, int W, int bf16) {
  using namespace ptx;
  extern __shared__ __align__(128) uint8_t hsm[];
  constexpr HeadTiles g = head_tiles_geom(TW);
  constexpr int R = g.R, SR = g.SR, SW = g.SW;
  float* ws = reinterpret_cast<float*>(hsm + 2 * (size_t)g.stage);  // [9][16]
  float* gate = ws + 9 * kHsC;                                       // [16]
  float* part = gate + kHsC;                                         // [16 groups][16]
  float* mean = part + 16 * kHsC;                                    // [16]
  uint64_t* full = reinterpret_cast<uint64_t*>(mean + kHsC);         // [2]
  uint64_t* empty = full + 2;                                        // [2]
  const int tid = threadIdx.x, warp = tid >> 5;
  const int L = W + 1;
  const int tpr = W / TW;         // column tiles per row band
  const int spi = (H / R) * tpr;  // strips per image
  const int64_t n_strips = B * spi;
  const int64_t s_begin = blockIdx.x * n_strips / gridDim.x;
  const int64_t s_end = (blockIdx.x + 1) * n_strips / gridDim.x;
  const int np = skip.np;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kHsCompute / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  grid_dep_wait();  // d, gap and skip come from the previous kernels

  if (warp == kHsCompute / 32) {
    // ===== producer warp: per staged row one copy of d and one per skip block; lane 0
    // posts the stage's byte count, the lanes issue the copies in parallel =====
    const int lane = tid & 31;
    const int nk = 1 + 2 * np;
    int i = 0;
    for (int64_t s = s_begin; s < s_end; ++s, ++i) {
      const int st = i & 1;
      mbar_wait(smem_u32(&empty[st]), ((i >> 1) & 1) ^ 1);
      const int64_t b = s / spi;
      const int rem = (int)(s - b * spi);
      const int y0 = (rem / tpr) * R, x0 = (rem - (rem / tpr) * tpr) * TW;
      const int r0 = y0 == 0 ? 1 : 0;            // first staged row inside the image
      const int r1 = y0 + R == H ? SR - 1 : SR;  // one past the last
      const int cl = x0 == 0 ? 0 : x0 - 1, cr = x0 + TW == W ? W : x0 + TW + 1;  // d columns
      const uint32_t bar = smem_u32(&full[st]);
      uint8_t* base = hsm + (size_t)st * g.stage;
      if (lane == 0)
        mbar_arrive_expect_tx(bar, (uint32_t)((r1 - r0) * ((cr - cl) * kHsC * (DBF ? 2 : 4) + np * 2 * SW * 16)));
      __syncwarp();
      for (int c = lane; c < (r1 - r0) * nk; c += 32) {
        const int r = r0 + c / nk, kk = c % nk, iy = y0 - 1 + r;
        if (kk == 0) {
          bulk_g2s(smem_u32(base + ((size_t)r * SW + (cl - (x0 - 1))) * kHsC * (DBF ? 2 : 4)),
                   reinterpret_cast<const uint8_t*>(d) + (((size_t)b * H + iy) * W + cl) * kHsC * (DBF ? 2 : 4),
                   (uint32_t)((cr - cl) * kHsC * (DBF ? 2 : 4)), bar);
        } else {
          const int blk = kk - 1;  // (pass, cg8)
          bulk_g2s(smem_u32(base + g.dbytes + (size_t)blk * g.sblk + (size_t)r * SW * 16),
                   skip.base + b * skip.img_stride +
                       ((int64_t)skip.block_index(0, blk >> 1, blk & 1) + skip.off + (int64_t)iy * L + x0 - 1) * 8,
                   (uint32_t)(SW * 16), bar);
        }
      }
    }
    return;
  }

  // ===== 8 compute warps =====
  const float bv = __ldg(bias);
  const int cx = tid % TW, rp = tid / TW;  // conv: column, row pair
  int64_t cur_b = -1;
  int i = 0;
  for (int64_t s = s_begin; s < s_end; ++s, ++i) {
    const int st = i & 1;
    const int64_t b = s / spi;
    const int rem = (int)(s - b * spi);
    const int y0 = (rem / tpr) * R, x0 = (rem - (rem / tpr) * tpr) * TW;
    if (b != cur_b && items == kGatesReady) {
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");  // previous image's gate readers
      if (tid < kHsC) gate[tid] = __ldg(gap + b * kHsC + tid);
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
      cur_b = b;
    } else if (b != cur_b) {
      // ECA gate of image b (model.py:128-135): kEcaGroups group sums in parallel, added
      // in group order (planes.cuh: the one reduction order of every gate)
      if (tid < kEcaGroups * kHsC) part[tid] = eca_group_sum(gap, items, kHsC, b, tid % kHsC, tid / kHsC);
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
      if (tid < kHsC) {
        float a = 0.f;
        for (int grp = 0; grp < kEcaGroups; ++grp) a += part[grp * kHsC + tid];
        mean[tid] = a / (float)(H * W);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
      if (tid < kHsC) gate[tid] = eca_gate_of(mean, kHsC, tid, eca_w, k);
      asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
      cur_b = b;
    }
    mbar_wait(smem_u32(&full[st]), (i >> 1) & 1);
    float* ubase = reinterpret_cast<float*>(hsm + (size_t)st * g.stage);
    const uint8_t* sbase = hsm + (size_t)st * g.stage + g.dbytes;
    // transform: one (stage pixel, channel quad) per thread step, NB steps per batch: all
    // loads of a batch, one __syncwarp (the 4 quads of a pixel are lanes of one warp and
    // are rewritten in place; steps touch disjoint pixels), then all stores.
    // Step `it` of the unrolled loop covers stage row it / 2, columns (it & 1) * 64 + tid / 4:
    // the row is a compile-time constant and every shared-memory address is a per-thread
    // byte offset plus an immediate (the kernel spent more cycles here than in the conv on
    // index arithmetic: divisions by SW, bounds checks); the two halo columns 128, 129 of
    // the SR rows (48 units) follow in one extra step of warps 0 and 1.
    static_assert(TW == 128 && SW == 130 && kHsCompute == 256, "transform step mapping");
    constexpr int VB = kHsC * (DBF ? 2 : 4), QB = DBF ? 8 : 16;  // bytes per stage pixel / value quad
    const int q = tid & 3, t4 = tid >> 2;
    const float4 g4 = *reinterpret_cast<const float4*>(gate + q * 4);
    const bool top = y0 == 0, bot = y0 + R == H, left = x0 == 0, right = x0 + TW == W;
    uint8_t* ub = reinterpret_cast<uint8_t*>(ubase);
    const uint32_t t_d = (uint32_t)t4 * VB + (uint32_t)q * QB;
    const uint32_t t_s = (uint32_t)(q >> 1) * g.sblk + (uint32_t)(q & 1) * 8 + (uint32_t)t4 * 16;
    // u = d * gate + skip (model.py:197-198) of one unit, zero outside the image
    auto unit = [&](float4 dvv, uint2 hvv, uint2 lvv, bool inside) {
      float4 uu = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inside) {
        float s4[4];
        s4[0] = __uint_as_float(hvv.x << 16);
        s4[1] = __uint_as_float(hvv.x & 0xFFFF0000u);
        s4[2] = __uint_as_float(hvv.y << 16);
        s4[3] = __uint_as_float(hvv.y & 0xFFFF0000u);
        if (np == 2) {
          s4[0] += __uint_as_float(lvv.x << 16);
          s4[1] += __uint_as_float(lvv.x & 0xFFFF0000u);
          s4[2] += __uint_as_float(lvv.y << 16);
          s4[3] += __uint_as_float(lvv.y & 0xFFFF0000u);
        }
        uu.x = gate_fma(dvv.x, g4.x, s4[0]);
        uu.y = gate_fma(dvv.y, g4.y, s4[1]);
        uu.z = gate_fma(dvv.z, g4.z, s4[2]);
        uu.w = gate_fma(dvv.w, g4.w, s4[3]);
        if (bf16) {
          uu.x = bf16_round(uu.x);
          uu.y = bf16_round(uu.y);
          uu.z = bf16_round(uu.z);
          uu.w = bf16_round(uu.w);
        }
      }
      return uu;
    };
    constexpr int NIT = 2 * SR, NB = 4;
    static_assert(NIT % NB == 0, "transform batches");
#pragma unroll
    for (int it0 = 0; it0 < NIT; it0 += NB) {
      float4 dv[NB];
      uint2 hv[NB], lv[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int it = it0 + j;
        const uint32_t pofs = (uint32_t)((it >> 1) * SW + (it & 1) * 64);  // compile-time
        dv[j] = hd_load_b<DBF>(ub + t_d + pofs * VB);
        // channels 4q..4q+3: cg8 block (q >> 1), bytes (q & 1) * 8 of the stage position
        hv[j] = *reinterpret_cast<const uint2*>(sbase + t_s + pofs * 16);
        lv[j] = np == 2 ? *reinterpret_cast<const uint2*>(sbase + t_s + pofs * 16 + 2 * g.sblk) : make_uint2(0u, 0u);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int it = it0 + j, r = it >> 1;
        const uint32_t pofs = (uint32_t)(r * SW + (it & 1) * 64);
        const bool inside = !(r == 0 && top) && !(r == SR - 1 && bot) && !((it & 1) == 0 && left && t4 == 0);
        // hs_swz(p) = (p >> 1) & 3 with p = r * 130 + column: (r + (column >> 1)) & 3
        const uint32_t sw = (uint32_t)((r + (t4 >> 1)) & 3);
        hd_store_b<DBF>(ub + (uint32_t)t4 * VB + pofs * VB + ((uint32_t)q ^ sw) * QB, unit(dv[j], hv[j], lv[j], inside));
      }
    }
    if (tid < 64) {  // the halo columns 128, 129: unit (row, column, quad) = (tid / 8, 128 + (tid / 4) % 2, tid % 4)
      const int r = min(tid >> 3, SR - 1), xs = 128 + (t4 & 1);
      const uint32_t pp = (uint32_t)(r * SW + xs);
      const bool act = tid < 8 * SR;
      const int iy = y0 - 1 + r;
      const bool inside = act && iy >= 0 && iy < H && !(xs == SW - 1 && right);
      const float4 dv1 = hd_load_b<DBF>(ub + pp * VB + (uint32_t)q * QB);
      const uint32_t so = (uint32_t)(q >> 1) * g.sblk + (uint32_t)(q & 1) * 8 + pp * 16;
      const uint2 hv1 = *reinterpret_cast<const uint2*>(sbase + so);
      const uint2 lv1 = np == 2 ? *reinterpret_cast<const uint2*>(sbase + so + 2 * g.sblk) : make_uint2(0u, 0u);
      __syncwarp();
      if (act) hd_store_b<DBF>(ub + pp * VB + ((uint32_t)q ^ (uint32_t)hs_swz((int)pp)) * QB, unit(dv1, hv1, lv1, inside));
    }
    fence_proxy_async();  // generic writes of this stage before its next async refill
    asm volatile("bar.sync 1, %0;" ::"n"(kHsCompute) : "memory");
    // conv3x3 (model.py:158,199): rows 2rp, 2rp+1 of the strip at column cx (stage column
    // cx + kx is image column x0 + cx + kx - 1; out-of-image pixels are zero in the stage)
    // 4 independent chains per output (channel quads j), summed at the end
    float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      float4 u[4][4];  // [channel quad][row]: all loads of this column first
      // stage pixel (2rp + rr) * SW + cx + kx: byte offset = per-thread base + rr * SW * VB,
      // swizzle (2rp + rr + ((cx + kx) >> 1)) & 3
      const uint32_t cb = (uint32_t)((2 * rp) * SW + cx + kx) * VB;
      const int s0 = 2 * rp + ((cx + kx) >> 1);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const uint32_t sw = (uint32_t)((s0 + rr) & 3) * QB;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          u[j][rr] = hd_load_b<DBF>(ub + cb + (uint32_t)(rr * SW) * VB + (((uint32_t)j * QB) ^ sw));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const float* wt = &cw.w[(ky * 3 + kx) * kHsC + j * 4];
          acc0[j] = fmaf(u[j][ky].x, wt[0], acc0[j]);
          acc0[j] = fmaf(u[j][ky].y, wt[1], acc0[j]);
          acc0[j] = fmaf(u[j][ky].z, wt[2], acc0[j]);
          acc0[j] = fmaf(u[j][ky].w, wt[3], acc0[j]);
          acc1[j] = fmaf(u[j][ky + 1].x, wt[0], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].y, wt[1], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].z, wt[2], acc1[j]);
          acc1[j] = fmaf(u[j][ky + 1].w, wt[3], acc1[j]);
        }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(smem_u32(&empty[st]));  // this warp is done with stage st
    float* yo = y + ((size_t)b * H + y0 + 2 * rp) * W + x0 + cx;
    yo[0] = ((acc0[0] + acc0[1]) + (acc0[2] + acc0[3])) + bv;
    yo[W] = ((acc1[0] + acc1[1]) + (acc1[2] + acc1[3])) + bv;
  }
}

bool head_strips_ok(int C0, int64_t B, int H, int W) {
  if (C0 != kHsC || B <= 0) return false;
  if (W == 32 || W == 64 || W == 128) {
    const HeadStrips g = head_strips_geom(W);
    return H % g.R == 0 && g.smem <= 227 * 1024;
  }
  const HeadTiles g = head_tiles_geom(128);  // wide maps: 128-column tiles
  return W % 128 == 0 && H % g.R == 0 && g.smem <= 227 * 1024;
}

template <typename K>
void set_smem(K kern) {
  ensure_dyn_smem(kern, 200 * 1024);
}

}  // namespace

bool stem_pp_only_ok(int C0, int F, int H, int W) {
  return C0 == kStemC && F >= 1 && F <= kStemMaxF && H % 4 == 0 && W % 2 == 0 && (W == 32 || W == 64 || W == 128) &&
         head_strips_ok(C0, 1, H, W);
}

void launch_stem_planes(const float* w, const float* bias, const Src& x, int F, int C0,
                        const PlBuf& pl, const PlBuf& pp, int64_t B, int H, int W, bool bf16,
                        cudaStream_t st, const float* canon_host) {
  STDA_CHECK(C0 % 16 == 0, "stem kernel needs stem_channels % 16 == 0");
  static const bool const_off = [] {
    const char* e = std::getenv("STDA_STEM");
    return e && std::string(e) == "rows";
  }();
  if (!const_off && canon_host && C0 == kStemC && F >= 1 && F <= kStemMaxF && x.xp == 1 && H % 2 == 0 &&
      W % 2 == 0 && W <= 1024) {
    StemConst cw{};
    for (int co = 0; co < kStemC; ++co) {
      for (int ci = 0; ci < F; ++ci)
        for (int t = 0; t < 9; ++t) cw.w[(ci * 9 + t) * kStemC + co] = canon_host[((size_t)co * F + ci) * 9 + t];
      cw.b[co] = canon_host[(size_t)kStemC * F * 9 + co];
    }
    static const int px = [] {  // env STDA_STEM_PX: pixels per thread (2, or 4: spills at 4 CTAs/SM)
      const char* e = std::getenv("STDA_STEM_PX");
      return e && std::atoi(e) == 4 ? 4 : 2;
    }();
    const int PXr = (H % (2 * px) == 0) ? px : 2;
    int R = PXr;
    while (R * 2 * W <= 256 * PXr && H % (R * 2) == 0) R *= 2;
    const size_t smem = (size_t)F * (R + 2) * W * 4;
    STDA_CHECK(smem <= 200 * 1024, "stem: rows do not fit shared memory");
    auto go = [&](auto fc) {
      constexpr int FF = decltype(fc)::value;
      const bool pl_out = pl.base != nullptr;
      const auto kern = !pl_out ? (bf16 ? stem_const_kernel<FF, 2, 1, false> : stem_const_kernel<FF, 2, 2, false>)
                        : bf16 ? (PXr == 4 ? stem_const_kernel<FF, 4, 1> : stem_const_kernel<FF, 2, 1>)
                               : (PXr == 4 ? stem_const_kernel<FF, 4, 2> : stem_const_kernel<FF, 2, 2>);
      STDA_CHECK(pl_out || PXr == 2, "stem: phase-planes-only output needs 2-pixel threads");
      ensure_dyn_smem(kern, 200 * 1024);
      for (int64_t b0 = 0; b0 < B; b0 += 65535) {
        dim3 grid(H / R, (unsigned)std::min<int64_t>(65535, B - b0));
        launch_pdl(kern, grid, dim3(kRowThreads), smem, st, "stem_const_kernel", cw, x, pl, pp, H, W, R, b0);
      }
    };
    switch (F) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 3: go(std::integral_constant<int, 3>{}); break;
      default: go(std::integral_constant<int, 4>{}); break;
    }
    return;
  }
  STDA_CHECK(pl.base != nullptr, "stem: phase-planes-only output needs the constant-bank stem");
  if (x.xp == 1 && H % 2 == 0 && W % 2 == 0 && W <= 1024) {
    // bulk-copy row-block path: R rows (even, dividing H) with R*W ~ 512 pixels
    // (256 threads x 2 vertically adjacent pixels)
    int R = 2;
    while (R * 2 * W <= 512 && H % (R * 2) == 0) R *= 2;
    const int np = pl.np, nblk = (C0 / 16) * np * 2, L = W + 1, Lp = W / 2 + 1;
    auto al = [](size_t v) { return (v + 127) / 128 * 128; };
    static const int direct = [] {
      const char* e = std::getenv("STDA_STEM_STORE");
      return e && std::string(e) == "bulk" ? 0 : 1;
    }();
    const size_t smem = al((size_t)F * (R + 2) * W * 4) + al((size_t)C0 * F * 9 * 4) +
                        (direct ? 0 : al((size_t)nblk * R * L * 16) + al((size_t)4 * nblk * (R / 2) * Lp * 16));
    STDA_CHECK(smem <= 200 * 1024, "stem: rows do not fit shared memory");
    set_smem(stem_rows_kernel);
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      dim3 grid(H / R, (unsigned)std::min<int64_t>(65535, B - b0));
      launch_pdl(stem_rows_kernel, grid, dim3(kRowThreads), smem, st, "stem_rows_kernel", w, bias, x, F, C0,
                 pl, pp, H, W, R, (int)bf16, b0, direct);
    }
    return;
  }
  const size_t smem = sizeof(float) * (F * kIH * kIW + F * 144);
  set_smem(stem_planes_kernel);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kTH), (unsigned)std::min<int64_t>(65535, B - b0));
    launch_pdl(stem_planes_kernel, grid, dim3(kThreads), smem, st, "stem_planes_kernel", w, bias, x, F, C0, pl,
               pp, H, W, (int)bf16, b0);
  }
}

bool head_bf16_ok(int C0, int64_t B, int H, int W, const PlBuf& skip) {
  static const bool strips_off = [] {
    const char* e = std::getenv("STDA_HEAD");
    return e && std::string(e) == "tiles";
  }();
  return !strips_off && head_strips_ok(C0, B, H, W) && (skip.planes == 1 || W <= 128);
}

void launch_head_fused(const float* w, const float* bias, const float* gap, int items,
                       const float* eca_w, int k, const float* d, const PlBuf& skip, int C0, float* y,
                       int64_t B, int H, int W, bool bf16, cudaStream_t st, const float* w_host, bool d_bf16) {
  STDA_CHECK(!d_bf16 || (w_host != nullptr && head_bf16_ok(C0, B, H, W, skip)), "head: bf16 d needs the strip head");
  STDA_CHECK(C0 % 8 == 0, "head kernel needs stem_channels % 8 == 0");
  static const bool strips_off = [] {
    const char* e = std::getenv("STDA_HEAD");
    return e && std::string(e) == "tiles";
  }();
  if (!strips_off && w_host != nullptr && head_strips_ok(C0, B, H, W)) {
    HeadConst hc{};
    for (int e = 0; e < 9 * kHsC; ++e) hc.w[e] = w_host[e];
    int dev = 0, sms = 148;
    STDA_CUDA(cudaGetDevice(&dev));
    STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    STDA_CHECK(skip.planes == 1 || W <= 128, "head: phase-plane skip needs the whole-width strips");
    if (W > 128) {  // column tiles
      const HeadTiles g = head_tiles_geom(128);
      const int64_t n_strips = B * (H / g.R) * (W / 128);
      const unsigned grid = (unsigned)std::min<int64_t>(n_strips, sms);
      const auto kern = d_bf16 ? head_tiles_kernel<128, true> : head_tiles_kernel<128, false>;
      ensure_dyn_smem(kern, 227 * 1024);
      launch_pdl(kern, dim3(grid), dim3(kHsThreads), g.smem, st, "head_tiles_kernel", hc, bias, gap, items, eca_w, k,
                 d, skip, y, B, H, W, (int)bf16);
      return;
    }
    const HeadStrips g = head_strips_geom(W);
    const int64_t n_strips = B * (H / g.R);
    const unsigned grid = (unsigned)std::min<int64_t>(n_strips, sms);
    auto go = [&](auto wc) {
      constexpr int WW = decltype(wc)::value;
      const auto kern = skip.planes == 4 ? (d_bf16 ? head_strips_kernel<WW, true, true> : head_strips_kernel<WW, true, false>)
                                         : (d_bf16 ? head_strips_kernel<WW, false, true> : head_strips_kernel<WW, false, false>);
      ensure_dyn_smem(kern, 227 * 1024);
      launch_pdl(kern, dim3(grid), dim3(kHsThreads), g.smem, st, "head_strips_kernel", hc, bias, gap, items, eca_w,
                 k, d, skip, y, B, H, (int)bf16);
    };
    if (W == 32) go(std::integral_constant<int, 32>{});
    else if (W == 64) go(std::integral_constant<int, 64>{});
    else go(std::integral_constant<int, 128>{});
    return;
  }
  STDA_CHECK(skip.planes == 1, "head: phase-plane skip needs the strip head");
  const size_t smem = sizeof(float) * ((size_t)(kHeadTH + 2) * kIW * (C0 + 4) + 9 * C0 + 2 * C0);
  STDA_CHECK(smem <= 200 * 1024, "head kernel: stem_channels too large for the smem tile");
  set_smem(head_fused_kernel);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    dim3 grid(cdiv(W, kTW), cdiv(H, kHeadTH), (unsigned)std::min<int64_t>(65535, B - b0));
    launch_pdl(head_fused_kernel, grid, dim3(kThreads), smem, st, "head_fused_kernel", w, bias, gap, items,
               eca_w, k, d, skip, C0, y, H, W, (int)bf16, b0);
  }
}

}  // namespace stda
