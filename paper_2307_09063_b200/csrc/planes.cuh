// Operand planes: the HBM layout every tcgen05 convolution reads its A operand from.
//
// A tensor of C channels over an Hp x Wp grid is stored, per image, as the grid
// linearised with row stride L = Wp + 1 (the extra column is an always-zero pad), split
// into bf16 hi (+ lo) parts, in UMMA K-major core-matrix order:
//
//     elem(b, plane, cg16, pass, cg8, q, e) =
//         base[b*img_stride + plane*plane_stride + (((cg16*np + pass)*2 + cg8)*Q + q + off)*8 + e]
//
// q = y*L + x (x = Wp is the pad column), e = channel within the 8-channel group.
// Because channels of one 8-group are 16 contiguous bytes and positions are contiguous,
// the A tile of any 128-row M-tile and tap is ONE contiguous byte range per (pass, cg8):
// the producer is a handful of cp.async.bulk copies, no conversion.
//   planes = 1 ("PL"): the grid itself (stride-1 convs, transposed convs, skips);
//   planes = 4 ("PP"): phase planes (py, px) of a 2Hp x 2Wp tensor, plane = py*2 + px,
//                      (y, x) <-> source pixel (2y+py, 2x+px) (stride-2 conv inputs).
// Borders that taps can reach — rows -1 and Hp (with margins) and the pad column — are
// kept zero by the kernels that write the plane (pads of the rows they write, margins once
// per image); positions past row Hp are only ever read into discarded (junk) output rows.
#pragma once

#include "common.cuh"

namespace stda {

struct PlBuf {
  uint16_t* base = nullptr;
  int planes = 1;
  int Hp = 0, Wp = 0, L = 0;
  int C = 0;   // multiple of 16
  int np = 2;  // 2: hi + lo (fp32 contract), 1: bf16
  int Q = 0;   // positions per (cg16, pass, cg8) block
  int off = 0; // position q is stored at index q + off
  int64_t plane_stride = 0, img_stride = 0;  // in bf16 elements

  __host__ __device__ size_t block_index(int cg16, int pass, int cg8) const {
    return (size_t)((cg16 * np + pass) * 2 + cg8) * Q;
  }
};

// Margins: taps reach q >= -L-1 (kept >= -off), tiles reach q < Hp*L + 4*128 + L + 1.
inline PlBuf make_plbuf(int planes, int Hp, int Wp, int C, int np) {
  PlBuf p;
  p.planes = planes;
  p.Hp = Hp;
  p.Wp = Wp;
  p.L = Wp + 1;
  p.C = C;
  p.np = np;
  p.off = p.L + 8;
  p.Q = (p.off + Hp * p.L + 4 * 128 + p.L + 16 + 7) / 8 * 8;
  p.plane_stride = (int64_t)(C / 16) * np * 2 * p.Q * 8;
  p.img_stride = p.plane_stride * planes;
  return p;
}

inline size_t plbuf_bytes(const PlBuf& p, int64_t B) { return (size_t)B * p.img_stride * 2; }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Write 8 channels (one cg8) of position (b, plane, q): hi and, when np == 2, lo.
__device__ __forceinline__ void pl_store8(const PlBuf& p, int64_t b, int plane, int c8, int q,
                                          const float (&v)[8]) {
  const int cg16 = c8 >> 1, cg8 = c8 & 1;
  uint16_t* img = p.base + b * p.img_stride + (int64_t)plane * p.plane_stride;
  float hi[8], lo[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    hi[i] = bf16_round(v[i]);
    lo[i] = v[i] - hi[i];
  }
  uint16_t* dh = img + (p.block_index(cg16, 0, cg8) + q + p.off) * 8;
  *reinterpret_cast<uint4*>(dh) = make_uint4(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]),
                                             pack_bf16x2(hi[4], hi[5]), pack_bf16x2(hi[6], hi[7]));
  if (p.np == 2) {
    uint16_t* dl = img + (p.block_index(cg16, 1, cg8) + q + p.off) * 8;
    *reinterpret_cast<uint4*>(dl) = make_uint4(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]),
                                               pack_bf16x2(lo[4], lo[5]), pack_bf16x2(lo[6], lo[7]));
  }
}

// pl_store8 with the pass count known at compile time and the block address precomputed:
// 8 channels -> bf16 hi at hi[0..7] (+ lo = v - hi at hi[lo_delta ..]), same bits as pl_store8
template <int NP>
__device__ __forceinline__ void store8_split(uint16_t* hi, size_t lo_delta, const float (&v)[8]) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __nv_bfloat162 hb = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    h[j] = *reinterpret_cast<const uint32_t*>(&hb);
    if (NP == 2) {
      const float2 hf = __bfloat1622float2(hb);
      l[j] = pack_bf16x2(v[2 * j] - hf.x, v[2 * j + 1] - hf.y);
    }
  }
  *reinterpret_cast<uint4*>(hi) = make_uint4(h[0], h[1], h[2], h[3]);
  if (NP == 2) *reinterpret_cast<uint4*>(hi + lo_delta) = make_uint4(l[0], l[1], l[2], l[3]);
}

// Read back 8 channels as fp32 (hi + lo).
__device__ __forceinline__ void pl_load8(const PlBuf& p, int64_t b, int plane, int c8, int q,
                                         float (&v)[8]) {
  const int cg16 = c8 >> 1, cg8 = c8 & 1;
  const uint16_t* img = p.base + b * p.img_stride + (int64_t)plane * p.plane_stride;
  const uint4 h = __ldg(reinterpret_cast<const uint4*>(img + (p.block_index(cg16, 0, cg8) + q + p.off) * 8));
  const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&h);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(hb[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
  if (p.np == 2) {
    const uint4 l = __ldg(reinterpret_cast<const uint4*>(img + (p.block_index(cg16, 1, cg8) + q + p.off) * 8));
    const __nv_bfloat162* lb = reinterpret_cast<const __nv_bfloat162*>(&l);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(lb[i]);
      v[2 * i] += f.x;
      v[2 * i + 1] += f.y;
    }
  }
}

// Border maintenance by the writers themselves (no separate zeroing pass):
// the pad column of a row is zeroed by whichever thread writes that row's last column,
// the top / bottom margins of an image by one CTA (or warp group) per image.
__device__ __forceinline__ void pl_zero16(uint16_t* p) {
  *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0);
}
// zero position q of every (cg16, pass, cg8) block of (b, plane)
__device__ __forceinline__ void pl_zero_pos(const PlBuf& p, int64_t b, int plane, int q) {
  uint16_t* img = p.base + b * p.img_stride + (int64_t)plane * p.plane_stride;
  const int nblk = (p.C / 16) * p.np * 2;
  for (int k = 0; k < nblk; ++k) pl_zero16(img + ((size_t)k * p.Q + q + p.off) * 8);
}
// top margin [-L-8, 0) and bottom margin [Hp*L, Hp*L+L+8) of all planes/blocks of image b,
// split over `nthr` cooperating threads
__device__ __forceinline__ void pl_zero_margins(const PlBuf& p, int64_t b, int tid, int nthr) {
  const int margin = p.L + 8;
  const int nblk = p.planes * (p.C / 16) * p.np * 2;
  uint16_t* img = p.base + b * p.img_stride;  // blocks of one image are contiguous
  for (int u = tid; u < nblk * 2 * margin; u += nthr) {
    const int k = u / (2 * margin), r = u - k * 2 * margin;
    const int q = r < margin ? -margin + r : p.Hp * p.L + (r - margin);
    pl_zero16(img + ((size_t)k * p.Q + q + p.off) * 8);
  }
}

// ---- ECA channel means (model.py:128-135) from per-item channel sums -------------------
// ONE reduction order for every kernel that forms a gate, whatever its thread count: the
// items of a channel are summed in kEcaGroups interleaved groups (t = g, g + kEcaGroups,
// ...), each in increasing t, and the group sums are added in increasing g.  A thread that
// loops over the groups itself performs exactly the same float operations as the parallel
// form below, so the gates — and every output — are bitwise independent of which gate
// kernel ran (and so of the batch size).
constexpr int kEcaGroups = 8;

// Gate source of the gate / head kernels: `gap` holds per-item channel sums (items > 0)
// from which the kernel forms the gate itself, or, with items == kGatesReady, the finished
// gates [B][C] (launch_eca_gates, same arithmetic: used when an image has so many items
// that every CTA re-reducing them would dominate, i.e. large maps).
constexpr int kGatesReady = -1;
inline bool precompute_gates(int items, int C) { return (int64_t)items * C >= 4096; }
void launch_eca_gates(const float* gap, int items, const float* eca_w, int k, float* gates, int64_t B, int C,
                      int64_t hw, cudaStream_t st);

__device__ __forceinline__ float eca_group_sum(const float* gap, int items, int C, int64_t b, int c, int g) {
  // loads batched 8 at a time ahead of the adds (one L2 round trip per 8 items instead of
  // one per item); the adds keep the order t = g, g + 8, ...
  const float* src = gap + ((size_t)b * items + g) * C + c;
  const size_t step = (size_t)kEcaGroups * C;
  const int n = items > g ? (items - g + kEcaGroups - 1) / kEcaGroups : 0;
  float a = 0.f;
  for (int t0 = 0; t0 < n; t0 += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = t0 + u < n ? __ldg(src + (size_t)(t0 + u) * step) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t0 + u < n) a += v[u];
  }
  return a;
}
// sequential form: the channel sum of channel c
__device__ __forceinline__ float eca_channel_sum(const float* gap, int items, int C, int64_t b, int c) {
  float s = 0.f;
  for (int g = 0; g < kEcaGroups; ++g) s += eca_group_sum(gap, items, C, b, c, g);
  return s;
}
// block-parallel form of eca_channel_sum for every channel of image b: thread u forms the
// group sum (c = u % C, g = u / C) — one batch of loads in flight per thread instead of
// kEcaGroups dependent round trips — then the groups are added in increasing g: the same
// float operations as eca_channel_sum, so the same bits.  mean[c] = sum / hw.
// part: kEcaGroups * C floats of shared memory; every thread of the block calls this.
constexpr int kEcaParallelMaxC = 128;
__device__ __forceinline__ void eca_means_block(const float* gap, int items, int C, int64_t b, float hw,
                                                float* part, float* mean) {
  for (int u = threadIdx.x; u < kEcaGroups * C; u += blockDim.x)
    part[u] = eca_group_sum(gap, items, C, b, u % C, u / C);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < kEcaGroups; ++g) s += part[g * C + c];
    mean[c] = s / hw;
  }
}
// eca(x) (+ skip) (model.py:95-98, 197-198) in ONE rounding order for every kernel that
// applies a gate: skip = hi + lo of its operand plane (exact in fp32), then one fused
// multiply-add; without a skip one multiply.  Explicit intrinsics: no kernel may differ
// by compiler contraction (batch invariance across gate-kernel choices).
__device__ __forceinline__ float gate_mul(float x, float g) { return __fmul_rn(x, g); }
__device__ __forceinline__ float gate_fma(float x, float g, float skip) { return __fmaf_rn(x, g, skip); }

// gate[c] = sigmoid(sum_j w[j] * mean[c + j - k/2]), zero-padded 1-D conv over channels
__device__ __forceinline__ float eca_gate_of(const float* mean, int C, int c, const float* eca_w, int k) {
  float z = 0.f;
  for (int j = 0; j < k; ++j) {
    const int cc = c + j - k / 2;
    if (cc >= 0 && cc < C) z = fmaf(__ldg(eca_w + j), mean[cc], z);
  }
  return 1.f / (1.f + expf(-z));
}

// ECA gate for image b computed from GAP partials, then applied:
//   v = x * g (+ skip)   x: NHWC fp32 [B][H][W][C]; skip: PL over H x W (or null)
// written to any of: PL over H x W, PP over (H/2 x W/2) planes, NHWC fp32.
void launch_gate_apply(const float* gap, int items, const float* eca_w, int k, const float* x,
                       const PlBuf* skip, const PlBuf* out_pl, const PlBuf* out_pp, float* out_f32,
                       int64_t B, int C, int H, int W, cudaStream_t st, bool x_bf16 = false);
// x_bf16 (the bf16 variant's stage-2 outputs stored as bf16) is taken by the strip kernel only
bool gate_apply_bf16_ok(bool has_skip, const PlBuf* out_pl, int64_t B, int C, int H, int W);

}  // namespace stda
