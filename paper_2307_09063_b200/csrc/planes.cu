// Operand-plane writers: the fused ECA gate + apply kernels (generic, row-block, persistent strips).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "planes.cuh"
#include "ptx.cuh"

namespace stda {
namespace {

constexpr int kGateThreads = 256;
constexpr int kPixPerCta = 128;

__global__ void __launch_bounds__(kGateThreads) gate_apply_kernel(
    const float* __restrict__ gap, int items, const float* __restrict__ eca_w, int k,
    const float* __restrict__ x, PlBuf skip, int has_skip, PlBuf out_pl, int has_pl, PlBuf out_pp,
    int has_pp, float* __restrict__ out_f32, int C, int H, int W) {
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
  __shared__ float mean[1024];
  __shared__ float gate[1024];
  __shared__ float part[kEcaGroups * kEcaParallelMaxC];
  const int64_t b = blockIdx.y;
  // gate for this image: fixed-order reduction of the producer's per-item partial sums
  if (items == kGatesReady) {
    for (int c = threadIdx.x; c < C; c += blockDim.x) gate[c] = __ldg(gap + b * C + c);
  } else {
    if (C <= kEcaParallelMaxC) {
      eca_means_block(gap, items, C, b, (float)(H * W), part, mean);
    } else {
      for (int c = threadIdx.x; c < C; c += blockDim.x) mean[c] = eca_channel_sum(gap, items, C, b, c) / (float)(H * W);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) gate[c] = eca_gate_of(mean, C, c, eca_w, k);
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
      for (int i = 0; i < 8; ++i)  // eca(x) = x * gate (+ skip, model.py:197-198)
        v[i] = has_skip ? gate_fma(v[i], gate[c8 * 8 + i], sk[j][i]) : gate_mul(v[i], gate[c8 * 8 + i]);
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

// Row-block gate + apply on the bulk-copy (TMA) engine: one CTA = R rows of one image.
// Inputs are contiguous row ranges — x rows (NHWC fp32) and, per (cg16, pass, cg8) block,
// the skip plane's positions [y0*L, (y0+R)*L) — bulk-loaded on an mbarrier; threads form
// v = x*gate (+ skip), split hi/lo into shared-memory images of the output plane rows
// (pad column included), and the row ranges go back with bulk stores.
__global__ void __launch_bounds__(kGateThreads) gate_apply_rows_kernel(
    const float* __restrict__ gap, int items, const float* __restrict__ eca_w, int k,
    const float* __restrict__ x, PlBuf skip, int has_skip, PlBuf out_pl, int has_pl, PlBuf out_pp,
    int has_pp, int C, int H, int W, int R) {
  grid_dep_wait();  // PDL: previous kernel complete (common.cuh)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ float gate[1024];
  __shared__ float mean[1024];
  __shared__ float part[kEcaGroups * kEcaParallelMaxC];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.y;
  const int y0 = blockIdx.x * R;
  const int G8 = C / 8;
  const int nblk = (C / 16) * out_pl.np * 2;  // (cg16, pass, cg8) blocks per plane
  const int L = W + 1, Lp = W / 2 + 1;
  // shared-memory carve-up (all 128-byte aligned)
  auto al = [](size_t v) { return (v + 127) / 128 * 128; };
  float* xs = reinterpret_cast<float*>(smem_raw);
  uint8_t* sk = smem_raw + al((size_t)R * W * C * 4);
  const size_t sk_blk = (size_t)R * L * 16;
  uint8_t* po = sk + (has_skip ? al(nblk * sk_blk) : 0);
  const size_t po_blk = (size_t)R * L * 16;
  uint8_t* pp = po + (has_pl ? al(nblk * po_blk) : 0);
  const size_t pp_blk = (size_t)(R / 2) * Lp * 16;

  if (tid == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t xb = (uint32_t)R * W * C * 4;
    const uint32_t sb = has_skip ? (uint32_t)(nblk * sk_blk) : 0u;
    ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), xb + sb);
    ptx::bulk_g2s(ptx::smem_u32(xs), x + ((size_t)b * H + y0) * W * C, xb, ptx::smem_u32(&bar));
    if (has_skip) {
      const uint16_t* img = skip.base + b * skip.img_stride;
      for (int kb = 0; kb < nblk; ++kb)
        ptx::bulk_g2s(ptx::smem_u32(sk + kb * sk_blk), img + ((size_t)kb * skip.Q + y0 * L + skip.off) * 8,
                      (uint32_t)sk_blk, ptx::smem_u32(&bar));
    }
  }
  // ECA gate of this image while the copies fly (fixed order: identical in every CTA)
  if (items == kGatesReady) {
    for (int c = tid; c < C; c += blockDim.x) gate[c] = __ldg(gap + b * C + c);
  } else {
    if (C <= kEcaParallelMaxC) {
      eca_means_block(gap, items, C, b, (float)(H * W), part, mean);
    } else {
      for (int c = tid; c < C; c += blockDim.x) mean[c] = eca_channel_sum(gap, items, C, b, c) / (float)(H * W);
    }
    __syncthreads();
    for (int c = tid; c < C; c += blockDim.x) gate[c] = eca_gate_of(mean, C, c, eca_w, k);
  }
  if (blockIdx.x == 0) {  // top / bottom margins of the output planes, once per image
    if (has_pl) pl_zero_margins(out_pl, b, tid, blockDim.x);
    if (has_pp) pl_zero_margins(out_pp, b, tid, blockDim.x);
  }
  __syncthreads();
  ptx::mbar_wait(ptx::smem_u32(&bar), 0);

  const int np = out_pl.np;
  const int n = R * W * G8;
  for (int u = tid; u < n; u += blockDim.x) {
    const int c8 = u % G8, pix = u / G8;
    const int r = pix / W, xx = pix - r * W;
    const float4 a0 = *reinterpret_cast<const float4*>(xs + (size_t)pix * C + c8 * 8);
    const float4 a1 = *reinterpret_cast<const float4*>(xs + (size_t)pix * C + c8 * 8 + 4);
    float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    if (!has_skip) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = gate_mul(v[i], gate[c8 * 8 + i]);  // eca(x) = x * gate
    } else {                                                               // + skip (model.py:197-198)
      const int kh = ((c8 >> 1) * np) * 2 + (c8 & 1);
      const uint4 h = *reinterpret_cast<const uint4*>(sk + kh * sk_blk + (size_t)(r * L + xx) * 16);
      const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&h);
      float s[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(hb[i]);
        s[2 * i] = f.x;
        s[2 * i + 1] = f.y;
      }
      if (np == 2) {
        const uint4 l = *reinterpret_cast<const uint4*>(sk + (kh + 2) * sk_blk + (size_t)(r * L + xx) * 16);
        const __nv_bfloat162* lb = reinterpret_cast<const __nv_bfloat162*>(&l);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(lb[i]);
          s[2 * i] += f.x;
          s[2 * i + 1] += f.y;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = gate_fma(v[i], gate[c8 * 8 + i], s[i]);
    }
    float hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hi[i] = bf16_round(v[i]);
      lo[i] = v[i] - hi[i];
    }
    const uint4 hv = make_uint4(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]), pack_bf16x2(hi[4], hi[5]),
                                pack_bf16x2(hi[6], hi[7]));
    const uint4 lv = make_uint4(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]), pack_bf16x2(lo[4], lo[5]),
                                pack_bf16x2(lo[6], lo[7]));
    const int kh = ((c8 >> 1) * np) * 2 + (c8 & 1);  // hi block of this 8-channel group
    if (has_pl) {
      *reinterpret_cast<uint4*>(po + kh * po_blk + (size_t)(r * L + xx) * 16) = hv;
      if (np == 2) *reinterpret_cast<uint4*>(po + (kh + 2) * po_blk + (size_t)(r * L + xx) * 16) = lv;
    }
    if (has_pp) {
      const int plane = ((y0 + r) & 1) * 2 + (xx & 1);
      uint8_t* ppl = pp + (size_t)plane * nblk * pp_blk;
      const size_t pos = (size_t)((r >> 1) * Lp + (xx >> 1)) * 16;
      *reinterpret_cast<uint4*>(ppl + kh * pp_blk + pos) = hv;
      if (np == 2) *reinterpret_cast<uint4*>(ppl + (kh + 2) * pp_blk + pos) = lv;
    }
  }
  // pad columns of the staged rows
  for (int u = tid; u < R * nblk; u += blockDim.x) {
    const int r = u / nblk, kb = u - r * nblk;
    if (has_pl) *reinterpret_cast<uint4*>(po + kb * po_blk + (size_t)(r * L + W) * 16) = make_uint4(0, 0, 0, 0);
    if (has_pp && (r & 1) == 0)
      for (int plane = 0; plane < 4; ++plane)
        *reinterpret_cast<uint4*>(pp + ((size_t)plane * nblk + kb) * pp_blk + (size_t)((r >> 1) * Lp + W / 2) * 16) =
            make_uint4(0, 0, 0, 0);
  }
  ptx::fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    if (has_pl) {
      uint16_t* img = out_pl.base + b * out_pl.img_stride;
      for (int kb = 0; kb < nblk; ++kb)
        ptx::bulk_s2g(img + ((size_t)kb * out_pl.Q + y0 * L + out_pl.off) * 8, ptx::smem_u32(po + kb * po_blk),
                      (uint32_t)po_blk);
    }
    if (has_pp) {
      for (int plane = 0; plane < 4; ++plane) {
        uint16_t* img = out_pp.base + b * out_pp.img_stride + (int64_t)plane * out_pp.plane_stride;
        for (int kb = 0; kb < nblk; ++kb)
          ptx::bulk_s2g(img + ((size_t)kb * out_pp.Q + (y0 / 2) * Lp + out_pp.off) * 8,
                        ptx::smem_u32(pp + ((size_t)plane * nblk + kb) * pp_blk), (uint32_t)pp_blk);
      }
    }
    ptx::bulk_commit();
    ptx::bulk_wait_read();
  }
}

}  // namespace

namespace {

// ---- persistent strip gate + apply ---------------------------------------------------
// One CTA per SM walks a contiguous range of strips (R rows of one image).  A producer
// warp bulk-copies each strip's rows of x (NHWC fp32: one contiguous range) and of the
// skip plane (one contiguous range per (cg16, pass, cg8) block, pad column included) into
// a kGsStages-deep ring; 8 compute warps form v = x * gate (+ skip), split hi/lo and store
// the output plane rows directly (PL, and PP phase planes when requested), pads included.
// The ECA gate is computed once per image per CTA by a parallel fixed-order reduction of
// the GAP partials (deterministic, independent of the CTA).
constexpr int kGsCompute = 512;  // 16 compute warps: the unit chains are latency-bound
constexpr int kGsThreads = kGsCompute + 32;
constexpr int kGsStages = 4;

// Compile-time channel count / passes / skip / phase-plane output: the unit loop has no
// runtime division and each thread keeps one 8-channel group (kGsCompute % (C / 8) == 0),
// so its plane block offsets are loop-invariant.
// XBF: x holds bf16 values (the bf16 variant's stage-2 outputs), else fp32
template <int C, int NP, bool SKIP, bool PP, bool WHOLE, bool XBF>
__global__ void __launch_bounds__(kGsThreads, 1) gate_strips_kernel(
    const float* __restrict__ gap, int items, const float* __restrict__ eca_w, int k,
    const void* __restrict__ x, PlBuf skip, PlBuf out_pl, PlBuf out_pp, int H, int W, int TW, uint32_t TW_mul,
    int R, int64_t B, uint32_t x_bytes, uint32_t stage_bytes) {
  constexpr int stages = kGsStages;
  constexpr int XB = XBF ? 2 : 4;  // bytes per x value
  using namespace ptx;
  constexpr int G8 = C / 8;
  constexpr int nblk = (C / 16) * NP * 2;
  static_assert(kGsCompute % G8 == 0, "one channel group per thread");
  extern __shared__ __align__(128) uint8_t gsm[];
  float* gate2 = reinterpret_cast<float*>(gsm + (size_t)stages * stage_bytes);  // [2][C]: current image, next image
  float* part = gate2 + 2 * C;                  // [2][kEcaGroups][C] group sums
  float* mean2 = part + 2 * kEcaGroups * C;     // [2][C]
  uint64_t* full = reinterpret_cast<uint64_t*>(mean2 + 2 * C);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = W + 1, Lp = W / 2 + 1;
  // a strip is R rows x TW columns; whole-width strips stage the skip rows with their pad
  // column (one contiguous range per block), column tiles stage TW positions per row
  constexpr bool whole = WHOLE;  // TW == W
  const int Ls = whole ? L : TW;
  const uint32_t sk_blk = (uint32_t)R * Ls * 16;
  const int tpr = WHOLE ? 1 : W / TW;  // column tiles per row band
  const int spi = (H / R) * tpr;
  const int64_t n_strips = B * spi;
  const int64_t s_begin = blockIdx.x * n_strips / gridDim.x;
  const int64_t s_end = (blockIdx.x + 1) * n_strips / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kGsCompute / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  grid_dep_wait();  // x, gap and skip come from the previous kernels

  if (warp == kGsCompute / 32) {
    // ===== producer warp: lane 0 posts the byte count, lanes issue one copy each =====
    // (whole-width strips: one range per tensor / block; column tiles: one per row)
    constexpr int nk = 1 + (SKIP ? nblk : 0);
    const int ncopy = whole ? nk : R * nk;
    int i = 0, st = 0;
    uint32_t ph = 0;
    for (int64_t s = s_begin; s < s_end; ++s, ++i) {
      mbar_wait(smem_u32(&empty[st]), ph ^ 1);
      const int64_t b = s / spi;
      const int rem = (int)(s - b * spi);
      const int y0 = (rem / tpr) * R, x0 = WHOLE ? 0 : (rem - (rem / tpr) * tpr) * TW;
      const uint32_t bar = smem_u32(&full[st]);
      uint8_t* base = gsm + (size_t)st * stage_bytes;
      if (lane == 0) mbar_arrive_expect_tx(bar, x_bytes + (SKIP ? nblk * sk_blk : 0u));
      __syncwarp();
      for (int c = lane; c < ncopy; c += 32) {
        const int r = whole ? 0 : c / nk, kk = whole ? c : c - r * nk;
        const int nr = whole ? R : 1;
        if (kk == 0)
          bulk_g2s(smem_u32(base + (size_t)r * TW * C * XB),
                   static_cast<const uint8_t*>(x) + ((((size_t)b * H + y0 + r) * W + x0) * C) * XB,
                   (uint32_t)nr * TW * C * XB, bar);
        else
          bulk_g2s(smem_u32(base + x_bytes + (size_t)(kk - 1) * sk_blk + (size_t)r * Ls * 16),
                   skip.base + b * skip.img_stride +
                       ((size_t)(kk - 1) * skip.Q + (size_t)(y0 + r) * L + x0 + skip.off) * 8,
                   (uint32_t)nr * Ls * 16, bar);
      }
      if (++st == stages) {
        st = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  // ===== 16 compute warps =====
  const int c8 = tid % G8, cg16 = c8 >> 1, cg8 = c8 & 1;
  const int kh = (cg16 * NP) * 2 + cg8;  // hi block of this 8-channel group (lo: kh + 2)
  const size_t pl_blk = ((size_t)kh * out_pl.Q + out_pl.off) * 8;
  const size_t pp_blk = PP ? ((size_t)kh * out_pp.Q + out_pp.off) * 8 : 0;
  const size_t pl_lo = (size_t)2 * out_pl.Q * 8, pp_lo = PP ? (size_t)2 * out_pp.Q * 8 : 0;
  int64_t cur_b = -1, pre_b = -1;  // image of gate slot 0 / of slot 1 (formed ahead)
  int st = 0;
  uint32_t ph = 0;
  float g8[8];
  for (int64_t s = s_begin; s < s_end; ++s) {
    const int64_t b = s / spi;
    const int rem = (int)(s - b * spi);
    const int y0 = (rem / tpr) * R, x0 = WHOLE ? 0 : (rem - (rem / tpr) * tpr) * TW;
    if (b != cur_b && b == pre_b) {
      // formed together with the previous image
#pragma unroll
      for (int j = 0; j < 8; ++j) g8[j] = gate2[C + c8 * 8 + j];
      cur_b = b;
    } else if (b != cur_b) {
      // ECA gates (model.py:128-135) of image b and — when this CTA's strips reach it — of
      // image b + 1 in the same pass (the second image's loads fly with the first's: the
      // CTAs whose strips span two images stop once instead of twice).  Per image: the
      // kEcaGroups group sums in parallel, then added in group order (planes.cuh: the one
      // reduction order of every gate).
      const int ni = b + 1 <= (s_end - 1) / spi ? 2 : 1;
      asm volatile("bar.sync 1, %0;" ::"n"(kGsCompute) : "memory");  // previous images' gate readers
      if (items == kGatesReady) {
        for (int u = tid; u < ni * C; u += kGsCompute) gate2[u] = __ldg(gap + b * C + u);
      } else {
        for (int u = tid; u < ni * kEcaGroups * C; u += kGsCompute) {
          const int im = u / (kEcaGroups * C), v = u - im * (kEcaGroups * C);
          part[u] = eca_group_sum(gap, items, C, b + im, v % C, v / C);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kGsCompute) : "memory");
        for (int u = tid; u < ni * C; u += kGsCompute) {
          const int im = u / C, c = u - im * C;
          float a = 0.f;
          for (int g = 0; g < kEcaGroups; ++g) a += part[im * (kEcaGroups * C) + g * C + c];
          mean2[u] = a / (float)(H * W);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kGsCompute) : "memory");
        for (int u = tid; u < ni * C; u += kGsCompute) {
          const int im = u / C, c = u - im * C;
          gate2[u] = eca_gate_of(mean2 + im * C, C, c, eca_w, k);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kGsCompute) : "memory");
#pragma unroll
      for (int j = 0; j < 8; ++j) g8[j] = gate2[c8 * 8 + j];
      cur_b = b;
      pre_b = ni == 2 ? b + 1 : -1;
    }
    if (y0 == 0 && x0 == 0) {  // top / bottom margins of the output planes, once per image
      pl_zero_margins(out_pl, b, tid, kGsCompute);
      if (PP) pl_zero_margins(out_pp, b, tid, kGsCompute);
    }
    mbar_wait(smem_u32(&full[st]), ph);
    const float* xs = reinterpret_cast<const float*>(gsm + (size_t)st * stage_bytes);
    const uint8_t* sk = gsm + (size_t)st * stage_bytes + x_bytes;
    uint16_t* opl = out_pl.base + b * out_pl.img_stride + pl_blk;
    uint16_t* opp = PP ? out_pp.base + b * out_pp.img_stride + pp_blk : nullptr;
#pragma unroll 2
    for (int pix = tid / G8; pix < R * TW; pix += kGsCompute / G8) {
      const int r = (int)__umulhi((uint32_t)pix, TW_mul), xl = pix - r * TW, xx = x0 + xl;
      float xv[8];
      if (XBF) {
        const uint4 h = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(xs) + (size_t)pix * C + c8 * 8);
        const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          xv[2 * j] = __uint_as_float(hw[j] << 16);
          xv[2 * j + 1] = __uint_as_float(hw[j] & 0xFFFF0000u);
        }
      } else {
        const float4 a0 = *reinterpret_cast<const float4*>(xs + (size_t)pix * C + c8 * 8);
        const float4 a1 = *reinterpret_cast<const float4*>(xs + (size_t)pix * C + c8 * 8 + 4);
        xv[0] = a0.x; xv[1] = a0.y; xv[2] = a0.z; xv[3] = a0.w;
        xv[4] = a1.x; xv[5] = a1.y; xv[6] = a1.z; xv[7] = a1.w;
      }
      float v[8];
      if (SKIP) {  // + skip (model.py:197-198), exact hi + lo of its plane
        const size_t so = (size_t)(r * Ls + xl) * 16;
        const uint4 h = *reinterpret_cast<const uint4*>(sk + (size_t)kh * sk_blk + so);
        const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
        float sk8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sk8[2 * j] = __uint_as_float(hw[j] << 16);
          sk8[2 * j + 1] = __uint_as_float(hw[j] & 0xFFFF0000u);
        }
        if (NP == 2) {
          const uint4 l = *reinterpret_cast<const uint4*>(sk + (size_t)(kh + 2) * sk_blk + so);
          const uint32_t lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            sk8[2 * j] += __uint_as_float(lw[j] << 16);
            sk8[2 * j + 1] += __uint_as_float(lw[j] & 0xFFFF0000u);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = gate_fma(xv[j], g8[j], sk8[j]);  // planes.cuh rounding order
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = gate_mul(xv[j], g8[j]);
      }
      const int oy = y0 + r;
      store8_split<NP>(opl + (size_t)(oy * L + xx) * 8, pl_lo, v);
      if (PP) {
        const int64_t pofs = (int64_t)((oy & 1) * 2 + (xx & 1)) * out_pp.plane_stride;
        store8_split<NP>(opp + pofs + (size_t)((oy >> 1) * Lp + (xx >> 1)) * 8, pp_lo, v);
      }
      if (xx >= W - 2) {  // pad columns of this thread's blocks (planes.cuh border contract)
        if (xx == W - 1) {
          pl_zero16(opl + (size_t)(oy * L + W) * 8);
          if (NP == 2) pl_zero16(opl + pl_lo + (size_t)(oy * L + W) * 8);
        }
        if (PP) {
          uint16_t* pz = opp + (int64_t)((oy & 1) * 2 + (xx & 1)) * out_pp.plane_stride +
                         (size_t)((oy >> 1) * Lp + W / 2) * 8;
          pl_zero16(pz);
          if (NP == 2) pl_zero16(pz + pp_lo);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[st]));  // this warp is done with stage st
    if (++st == stages) {
      st = 0;
      ph ^= 1u;
    }
  }
}

}  // namespace

namespace {
// gates[b][c] from per-item channel sums, one CTA per image: the kEcaGroups group sums in
// parallel, added in group order — the arithmetic of every in-kernel gate (planes.cuh)
__global__ void __launch_bounds__(256) eca_gates_kernel(const float* __restrict__ gap, int items,
                                                        const float* __restrict__ eca_w, int k,
                                                        float* __restrict__ gates, int C, int64_t hw) {
  grid_dep_wait();
  extern __shared__ float esm[];  // part [kEcaGroups][C], mean [C]
  float* part = esm;
  float* mean = esm + kEcaGroups * C;
  const int64_t b = blockIdx.x;
  for (int u = threadIdx.x; u < kEcaGroups * C; u += blockDim.x)
    part[u] = eca_group_sum(gap, items, C, b, u % C, u / C);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float a = 0.f;
    for (int g = 0; g < kEcaGroups; ++g) a += part[g * C + c];
    mean[c] = a / (float)hw;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) gates[b * C + c] = eca_gate_of(mean, C, c, eca_w, k);
}
}  // namespace

void launch_eca_gates(const float* gap, int items, const float* eca_w, int k, float* gates, int64_t B, int C,
                      int64_t hw, cudaStream_t st) {
  STDA_CHECK(B <= 0x7fffffff && C <= 4096, "eca gates: shape");
  if (B == 0) return;
  launch_pdl(eca_gates_kernel, dim3((unsigned)B), dim3(256), (size_t)(kEcaGroups + 1) * C * 4, st,
             "eca_gates_kernel", gap, items, eca_w, k, gates, C, hw);
}

namespace {
// the persistent strip plan of gate_apply (valid = the strip kernel runs)
struct GateStripPlan {
  bool valid = false;
  int TW = 0, R = 0;
  size_t stage_bytes = 0, smem = 0;
  unsigned grid = 0;
};
GateStripPlan gate_strip_plan(bool has_skip, const PlBuf* out_pl, bool f32_out, int64_t B, int C, int H, int W,
                              int xb) {
  GateStripPlan sp;
  static const bool strips_off = [] {
    const char* e = std::getenv("STDA_GATE");
    return e && std::string(e) == "rows";
  }();
  if (strips_off || f32_out || out_pl == nullptr || C % 16 != 0 || C > 128 || H % 2 || W % 2 || B <= 0) return sp;
  const int np = out_pl->np, nblk = (C / 16) * np * 2, L = W + 1;
  auto stage = [&](int r, int tw) {
    return (size_t)r * tw * C * xb + (has_skip ? (size_t)nblk * r * (tw == W ? L : tw) * 16 : 0);
  };
  static const size_t stage_cap = [] {  // env STDA_GATE_STAGE_KB (A/B timing), default 16
    const char* e = std::getenv("STDA_GATE_STAGE_KB");
    return (size_t)(e ? std::max(8, std::atoi(e)) : 16) * 1024;  // measured best of 16/32/48
  }();
  const size_t fixed = (size_t)2 * (kEcaGroups + 2) * C * 4 + 2 * kGsStages * 8;
  auto smem_of = [&](size_t sb) { return kGsStages * ((sb + 127) / 128 * 128) + fixed; };
  int TW = W;
  while (smem_of(stage(2, TW)) > 227 * 1024 && TW % 2 == 0 && TW / 2 >= 16) TW /= 2;
  int R = 2;
  while (R * 2 <= 16 && H % (R * 2) == 0 && stage(R * 2, TW) <= stage_cap) R *= 2;
  int dev = 0, sms = 148;
  STDA_CUDA(cudaGetDevice(&dev));
  STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t n_strips = B * (H / R) * (W / TW);
  sp.smem = smem_of(stage(R, TW));
  // measured: with fewer than ~4 strips per SM the per-CTA fill (first loads + gate)
  // dominates and the one-shot row-block kernel is faster.  bf16 inputs (xb == 2) only
  // the strip kernel reads, so for them the choice must not depend on the batch (the
  // bf16 storage decision, and with it the rounding, is per plan shape, not per B).
  sp.valid = H % R == 0 && sp.smem <= 227 * 1024 && (xb == 2 || n_strips >= 4 * (int64_t)sms);
  sp.TW = TW;
  sp.R = R;
  sp.stage_bytes = (stage(R, TW) + 127) / 128 * 128;
  sp.grid = (unsigned)std::min<int64_t>(n_strips, sms);
  return sp;
}
}  // namespace

bool gate_apply_bf16_ok(bool has_skip, const PlBuf* out_pl, int64_t B, int C, int H, int W) {
  return gate_strip_plan(has_skip, out_pl, false, B, C, H, W, 2).valid;
}

void launch_gate_apply(const float* gap, int items, const float* eca_w, int k, const float* x,
                       const PlBuf* skip, const PlBuf* out_pl, const PlBuf* out_pp, float* out_f32,
                       int64_t B, int C, int H, int W, cudaStream_t st, bool x_bf16) {
  STDA_CHECK(C % 8 == 0 && C <= 1024, "gate_apply: channel count");
  const GateStripPlan sp = gate_strip_plan(skip != nullptr, out_pl, out_f32 != nullptr, B, C, H, W, x_bf16 ? 2 : 4);
  STDA_CHECK(!x_bf16 || sp.valid, "gate_apply: bf16 input needs the strip kernel");
  if (sp.valid) {
    const int np = out_pl->np, TW = sp.TW, R = sp.R;
    const size_t stage_bytes = sp.stage_bytes, smem = sp.smem;
    {
      const unsigned grid = sp.grid;
      const uint32_t TW_mul = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)TW - 1) / (uint64_t)TW);
      STDA_CHECK((uint64_t)R * TW * TW < ((uint64_t)1 << 32), "gate strips: row index");
      auto go = [&](auto cc, auto npc, auto skc, auto ppc) {
        constexpr int CC = decltype(cc)::value, NPC = decltype(npc)::value;
        constexpr bool SKC = decltype(skc)::value, PPC = decltype(ppc)::value;
        auto kern = TW == W ? gate_strips_kernel<CC, NPC, SKC, PPC, true, false>
                            : gate_strips_kernel<CC, NPC, SKC, PPC, false, false>;
        if constexpr (NPC == 1) {  // bf16 inputs only in the bf16 variant (one pass)
          if (x_bf16)
            kern = TW == W ? gate_strips_kernel<CC, NPC, SKC, PPC, true, true>
                           : gate_strips_kernel<CC, NPC, SKC, PPC, false, true>;
        } else {
          STDA_CHECK(!x_bf16, "gate_apply: bf16 input with hi/lo planes");
        }
        ensure_dyn_smem(kern, 227 * 1024);
        launch_pdl(kern, dim3(grid), dim3(kGsThreads), smem, st, "gate_strips_kernel", gap, items, eca_w, k,
                   static_cast<const void*>(x), skip ? *skip : PlBuf{}, *out_pl, out_pp ? *out_pp : PlBuf{}, H,
                   W, TW, TW_mul, R, B, (uint32_t)((size_t)R * TW * C * (x_bf16 ? 2 : 4)),
                   (uint32_t)stage_bytes);
      };
      using std::integral_constant;
      auto g3 = [&](auto cc, auto npc) {
        if (skip && out_pp) go(cc, npc, integral_constant<bool, true>{}, integral_constant<bool, true>{});
        else if (skip) go(cc, npc, integral_constant<bool, true>{}, integral_constant<bool, false>{});
        else if (out_pp) go(cc, npc, integral_constant<bool, false>{}, integral_constant<bool, true>{});
        else go(cc, npc, integral_constant<bool, false>{}, integral_constant<bool, false>{});
      };
      auto g2 = [&](auto cc) {
        if (np == 2) g3(cc, integral_constant<int, 2>{});
        else g3(cc, integral_constant<int, 1>{});
      };
      switch (C) {
        case 16: g2(integral_constant<int, 16>{}); break;
        case 32: g2(integral_constant<int, 32>{}); break;
        case 64: g2(integral_constant<int, 64>{}); break;
        default: g2(integral_constant<int, 128>{}); break;
      }
      return;
    }
  }
  STDA_CHECK(B <= 65535, "gate_apply: batch too large for one launch");
  if (out_f32 == nullptr && out_pl != nullptr && C % 16 == 0 && H % 2 == 0 && W % 2 == 0) {
    // bulk-copy row-block path: R rows per CTA, shared memory sized for the buffers used
    const int np = out_pl->np, nblk = (C / 16) * np * 2, L = W + 1, Lp = W / 2 + 1;
    auto al = [](size_t v) { return (v + 127) / 128 * 128; };
    int R = 2;
    auto bytes = [&](int r) {
      return al((size_t)r * W * C * 4) + (skip ? al((size_t)nblk * r * L * 16) : 0) +
             al((size_t)nblk * r * L * 16) + (out_pp ? al((size_t)4 * nblk * (r / 2) * Lp * 16) : 0);
    };
    // (small batches: keep >= one CTA per SM before growing the row block)
    while (R * 2 <= 8 && H % (R * 2) == 0 && (size_t)R * 2 * W <= 512 && bytes(R * 2) <= 96 * 1024 &&
           (int64_t)(H / (R * 2)) * B >= 148)
      R *= 2;
    const size_t smem = bytes(R);
    STDA_CHECK(smem <= 200 * 1024, "gate_apply: rows do not fit shared memory");
    ensure_dyn_smem(gate_apply_rows_kernel, 200 * 1024);
    dim3 grid(H / R, (unsigned)B);
    launch_pdl(gate_apply_rows_kernel, grid, dim3(kGateThreads), smem, st, "gate_apply_rows_kernel", gap, items,
               eca_w, k, x, skip ? *skip : PlBuf{}, (int)(skip != nullptr), *out_pl, 1,
               out_pp ? *out_pp : PlBuf{}, (int)(out_pp != nullptr), C, H, W, R);
    return;
  }
  dim3 grid(cdiv(H * W, kPixPerCta), (unsigned)B);
  launch_pdl(gate_apply_kernel, grid, dim3(kGateThreads), 0, st, "gate_apply_kernel", gap, items, eca_w, k, x,
             skip ? *skip : PlBuf{}, (int)(skip != nullptr), out_pl ? *out_pl : PlBuf{}, (int)(out_pl != nullptr),
             out_pp ? *out_pp : PlBuf{}, (int)(out_pp != nullptr), out_f32, C, H, W);
}

}  // namespace stda
