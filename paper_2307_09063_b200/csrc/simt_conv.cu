// Generic FP32-SIMT direct convolution (see simt_conv.cuh).
//
// CTA = 256 threads = 8 warps, output tile 16 rows x 32 columns of one triplet and
// `COB` output channels.  Each thread owns 2 output pixels x COB channels (x2 for the
// dual-accumulator stages); weights are warp-uniform smem broadcasts (float4), input
// halo tiles are staged per chunk of CICH input channels with the source transform
// (ECA gate, skip add) applied on the way in.
#include <algorithm>
#include <vector>

#include "simt_conv.cuh"

namespace stda {

namespace {

constexpr int kThreads = 256;
constexpr int kTileH = 16;
constexpr int kTileW = 32;

template <int MODE>
struct Geo;
template <>
struct Geo<CONV3_S1> {  // input rows oy0-1..oy0+16, cols ox0-1..ox0+32
  static constexpr int IH = 18, IW = 34, IWP = 34;
};
template <>
struct Geo<CONV3_S2> {  // input rows 2oy0-1..2oy0+31, cols 2ox0-1..2ox0+63 (even|odd planes)
  static constexpr int IH = 33, IW = 65, IWP = 65;
};
template <>
struct Geo<CONVT4_S2> {  // input rows m0-1..m0+8, cols n0-1..n0+16
  static constexpr int IH = 10, IW = 18, IWP = 18;
};

__host__ __device__ constexpr int tapsz_of(int mode, int cob) {
  return mode == CONVT4_S2 ? 4 * (4 * cob + 4) : 9 * cob;
}

struct Args {
  Src in0, in1;
  const float* w0;
  const float* b0;
  const float* w1;
  const float* b1;
  float* out;
  float* gap;
  OutLayout ol;
  int64_t b_base;
  int Cin, Cout, Hi, Wi, Ho, Wo;
  int relu0, bf16;
  int tiles_x, ntiles;
};

__device__ __forceinline__ float src_value(const Src& s, int64_t b, int c, int64_t pix) {
  float v = __ldg(s.x + b * s.xb + (int64_t)c * s.xc + pix * s.xp);
  if (s.gx) v = v * __ldg(s.gx + b * s.C + c);
  if (s.s) {
    float u = __ldg(s.s + b * s.sb + (int64_t)c * s.sc + pix * s.sp);
    if (s.gs) u = u * __ldg(s.gs + b * s.C + c);
    v = v + u;
  }
  return v;
}

template <int MODE, int CICH>
__device__ __forceinline__ void stage_tile(float* tile, const Src& s, int64_t b, int ci0, int Cin,
                                           int Hi, int Wi, int iy0, int ix0, bool bf16) {
  using G = Geo<MODE>;
  constexpr int PER_CH = G::IH * G::IW;
  // NCHW sources: x fastest (coalesced rows); NHWC sources: channel fastest (coalesced
  // pixels).  Both visit every (ci, r, c) of the tile exactly once.
  const bool chan_fast = s.xc == 1;
  for (int e = threadIdx.x; e < CICH * PER_CH; e += kThreads) {
    int ci, rem;
    if (chan_fast) {
      rem = e / CICH;
      ci = e - rem * CICH;
    } else {
      ci = e / PER_CH;
      rem = e - ci * PER_CH;
    }
    const int r = rem / G::IW;
    const int c = rem - r * G::IW;
    const int iy = iy0 + r, ix = ix0 + c;
    float v = 0.f;
    if (ci0 + ci < Cin && iy >= 0 && iy < Hi && ix >= 0 && ix < Wi) {
      v = src_value(s, b, ci0 + ci, (int64_t)iy * Wi + ix);
      if (bf16) v = bf16_round(v);
    }
    int col = c;
    if (MODE == CONV3_S2) col = (c & 1) ? 33 + (c >> 1) : (c >> 1);
    tile[ci * G::IH * G::IWP + r * G::IWP + col] = v;
  }
}

template <int TAPSZ, int CICH>
__device__ __forceinline__ void stage_weights(float* wsm, const float* w, int blk, int ci0, int Cin) {
  const int n_valid = min(CICH, Cin - ci0) * TAPSZ;
  const float* src = w + ((int64_t)blk * Cin + ci0) * TAPSZ;
  for (int e = threadIdx.x; e < CICH * TAPSZ; e += kThreads) wsm[e] = e < n_valid ? __ldg(src + e) : 0.f;
}

template <int COB>
__device__ __forceinline__ void fma_cob(float (&acc)[COB], float v, const float* w) {
  if constexpr (COB % 4 == 0) {
#pragma unroll
    for (int q = 0; q < COB / 4; ++q) {
      const float4 w4 = reinterpret_cast<const float4*>(w)[q];
      acc[4 * q + 0] = fmaf(v, w4.x, acc[4 * q + 0]);
      acc[4 * q + 1] = fmaf(v, w4.y, acc[4 * q + 1]);
      acc[4 * q + 2] = fmaf(v, w4.z, acc[4 * q + 2]);
      acc[4 * q + 3] = fmaf(v, w4.w, acc[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < COB; ++q) acc[q] = fmaf(v, w[q], acc[q]);
  }
}

// acc[r][co] += sum over CICH channels and taps, for this thread's 2 pixels.
template <int MODE, int COB, int CICH>
__device__ __forceinline__ void compute_chunk(float (&acc)[2][COB], const float* tile,
                                              const float* wsm) {
  using G = Geo<MODE>;
  constexpr int TAPSZ = tapsz_of(MODE, COB);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int ci = 0; ci < CICH; ++ci) {
    const float* t = tile + ci * G::IH * G::IWP;
    const float* wc = wsm + ci * TAPSZ;
    if constexpr (MODE == CONV3_S1) {
      float v[4][3];
      const float* tp = t + (2 * warp) * G::IWP + lane;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[r][c] = tp[r * G::IWP + c];
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float* w = wc + (ky * 3 + kx) * COB;
          fma_cob<COB>(acc[0], v[ky][kx], w);
          fma_cob<COB>(acc[1], v[ky + 1][kx], w);
        }
    } else if constexpr (MODE == CONV3_S2) {
      float v[5][3];
      const float* tp = t + (4 * warp) * G::IWP;
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        v[r][0] = tp[r * G::IWP + lane];
        v[r][1] = tp[r * G::IWP + 33 + lane];
        v[r][2] = tp[r * G::IWP + lane + 1];
      }
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float* w = wc + (ky * 3 + kx) * COB;
          fma_cob<COB>(acc[0], v[ky][kx], w);
          fma_cob<COB>(acc[1], v[ky + 2][kx], w);
        }
    } else {
      const int py = warp & 1, j = warp >> 1;
      const int nl = lane >> 1, px = lane & 1;
      float v[3][2];
#pragma unroll
      for (int rr = 0; rr < 3; ++rr)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) v[rr][bb] = t[(2 * j + py + rr) * G::IWP + nl + px + bb];
      const float* wp = wc + (py * 2 + px) * (4 * COB + 4);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          const float* w = wp + (a * 2 + bb) * COB;
          fma_cob<COB>(acc[0], v[a][bb], w);
          fma_cob<COB>(acc[1], v[a + 1][bb], w);
        }
    }
  }
}

template <int MODE, bool DUAL, int COB, int CICH>
__global__ void __launch_bounds__(kThreads, 2) conv_simt_kernel(Args a) {
  using G = Geo<MODE>;
  constexpr int TAPSZ = tapsz_of(MODE, COB);
  constexpr int TILE_FLOATS = CICH * G::IH * G::IWP;
  constexpr int W_FLOATS = CICH * TAPSZ;
  extern __shared__ __align__(16) float smem[];
  float* w0s = smem;
  float* w1s = w0s + W_FLOATS;
  float* t0s = w1s + (DUAL ? W_FLOATS : 0);
  float* t1s = t0s + TILE_FLOATS;
  float* red = t1s + (DUAL ? TILE_FLOATS : 0);

  const int tile = blockIdx.x;
  const int blk = blockIdx.y;
  const int64_t b = a.b_base + blockIdx.z;
  const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
  const int oy0 = ty * kTileH, ox0 = tx * kTileW;
  int iy0, ix0;
  if (MODE == CONV3_S1) {
    iy0 = oy0 - 1; ix0 = ox0 - 1;
  } else if (MODE == CONV3_S2) {
    iy0 = 2 * oy0 - 1; ix0 = 2 * ox0 - 1;
  } else {
    iy0 = oy0 / 2 - 1; ix0 = ox0 / 2 - 1;
  }

  float acc0[2][COB], acc1[2][COB];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int q = 0; q < COB; ++q) acc0[r][q] = acc1[r][q] = 0.f;

  for (int ci0 = 0; ci0 < a.Cin; ci0 += CICH) {
    __syncthreads();
    stage_weights<TAPSZ, CICH>(w0s, a.w0, blk, ci0, a.Cin);
    stage_tile<MODE, CICH>(t0s, a.in0, b, ci0, a.Cin, a.Hi, a.Wi, iy0, ix0, a.bf16);
    if constexpr (DUAL) {
      stage_weights<TAPSZ, CICH>(w1s, a.w1, blk, ci0, a.Cin);
      stage_tile<MODE, CICH>(t1s, a.in1, b, ci0, a.Cin, a.Hi, a.Wi, iy0, ix0, a.bf16);
    }
    __syncthreads();
    compute_chunk<MODE, COB, CICH>(acc0, t0s, w0s);
    if constexpr (DUAL) compute_chunk<MODE, COB, CICH>(acc1, t1s, w1s);
  }

  // epilogue: bias, relu, dual add, store, per-tile channel sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int oy[2];
  if (MODE == CONVT4_S2) {
    const int py = warp & 1, j = warp >> 1;
    oy[0] = 2 * (oy0 / 2 + 2 * j) + py;
    oy[1] = oy[0] + 2;
  } else {
    oy[0] = oy0 + 2 * warp;
    oy[1] = oy[0] + 1;
  }
  const int ox = ox0 + lane;
  float gsum[COB];
  // NHWC output with a full channel block per pixel: contiguous float4 stores
  const bool vec_store = COB % 4 == 0 && a.ol.oc == 1 && (blk + 1) * COB <= a.Cout;
#pragma unroll
  for (int q = 0; q < COB; ++q) {
    const int co = blk * COB + q;
    gsum[q] = 0.f;
    if (co >= a.Cout) continue;
    const float bias0 = __ldg(a.b0 + co);
    const float bias1 = DUAL ? __ldg(a.b1 + co) : 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float v = acc0[r][q] + bias0;
      if (a.relu0) v = fmaxf(v, 0.f);
      if (DUAL) v = v + (acc1[r][q] + bias1);
      acc0[r][q] = v;
      if (oy[r] < a.Ho && ox < a.Wo) {
        if (!vec_store) a.out[b * a.ol.ob + co * a.ol.oc + ((int64_t)oy[r] * a.Wo + ox) * a.ol.op] = v;
        gsum[q] += v;
      }
    }
  }
  if (vec_store) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (oy[r] >= a.Ho || ox >= a.Wo) continue;
      float* op = a.out + b * a.ol.ob + blk * COB + ((int64_t)oy[r] * a.Wo + ox) * a.ol.op;
#pragma unroll
      for (int q = 0; q < COB; q += 4)
        *reinterpret_cast<float4*>(op + q) =
            make_float4(acc0[r][q], acc0[r][q + 1], acc0[r][q + 2], acc0[r][q + 3]);
    }
  }
  if (a.gap) {
#pragma unroll
    for (int q = 0; q < COB; ++q) {
      float s = gsum[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp * COB + q] = s;
    }
    __syncthreads();
    if (threadIdx.x < COB) {
      const int co = blk * COB + threadIdx.x;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) s += red[w * COB + threadIdx.x];
      if (co < a.Cout) a.gap[(b * a.ntiles + tile) * a.Cout + co] = s;
    }
  }
}

template <int MODE, bool DUAL, int COB, int CICH>
void launch_impl(Args a, int64_t B, int nblk, cudaStream_t st) {
  using G = Geo<MODE>;
  constexpr int TAPSZ = tapsz_of(MODE, COB);
  const size_t smem = sizeof(float) * ((DUAL ? 2 : 1) * (CICH * TAPSZ + CICH * G::IH * G::IWP) +
                                       (kThreads / 32) * COB);
  auto kern = conv_simt_kernel<MODE, DUAL, COB, CICH>;
  ensure_dyn_smem(kern, (int)smem);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    a.b_base = b0;
    dim3 grid(a.ntiles, nblk, (unsigned)std::min<int64_t>(65535, B - b0));
    kern<<<grid, kThreads, smem, st>>>(a);
    check_launch("conv_simt_kernel");
  }
}

template <int MODE, bool DUAL, int CICH>
void dispatch_cob(int cob, Args a, int64_t B, int nblk, cudaStream_t st) {
  switch (cob) {
    case 1: return launch_impl<MODE, DUAL, 1, CICH>(a, B, nblk, st);
    case 4: return launch_impl<MODE, DUAL, 4, CICH>(a, B, nblk, st);
    case 8: return launch_impl<MODE, DUAL, 8, CICH>(a, B, nblk, st);
    default: return launch_impl<MODE, DUAL, 16, CICH>(a, B, nblk, st);
  }
}

// ---- ECA helpers ---------------------------------------------------------------
// `gap` and `gates` may alias (stda_eca reduces the channel sums in place: every sum is
// read into shared memory before the __syncthreads that precedes the first gate store),
// so neither is declared __restrict__.
__global__ void gate_kernel(const float* gap, int ntiles, const float* __restrict__ w,
                            int k, float* gates, int C, int hw) {
  extern __shared__ float mean[];
  const int64_t b = blockIdx.x;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int t = 0; t < ntiles; ++t) s += gap[(b * ntiles + t) * C + c];
    mean[c] = s / (float)hw;
  }
  __syncthreads();
  const int h = k / 2;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float z = 0.f;
    for (int j = 0; j < k; ++j) {
      const int cc = c + j - h;
      if (cc >= 0 && cc < C) z = fmaf(__ldg(w + j), mean[cc], z);
    }
    gates[b * C + c] = 1.f / (1.f + expf(-z));
  }
}

__global__ void channel_sum_kernel(const float* __restrict__ x, float* __restrict__ gap, int hw) {
  const int64_t bc = blockIdx.x;
  const float* p = x + bc * hw;
  float s = 0.f;
  for (int i = threadIdx.x; i < hw; i += blockDim.x) s += p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    gap[bc] = t;
  }
}

__global__ void scale_kernel(const float* __restrict__ x, const float* __restrict__ g,
                             float* __restrict__ y, int64_t n, int hw) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * g[i / hw];
}

}  // namespace

int simt_cob_for(int cout) {
  if (cout <= 1) return 1;
  if (cout <= 4) return 4;
  if (cout <= 8) return 8;
  return 16;
}

int simt_tapsz(int mode, int cob) { return tapsz_of(mode, cob); }

int conv_out_h(int mode, int hi) {
  return mode == CONV3_S1 ? hi : (mode == CONV3_S2 ? hi / 2 : 2 * hi);
}

int conv_tiles(int mode, int ho, int wo) { return cdiv(ho, kTileH) * cdiv(wo, kTileW); }

void simt_pack(int mode, int cin, int cout, const float* w, const float* bias, bool bf16,
               float* w_out, float* b_out) {
  const int cob = simt_cob_for(cout);
  const int nblk = cdiv(cout, cob);
  const int tapsz = tapsz_of(mode, cob);
  auto rnd = [bf16](float v) {
    return bf16 ? __bfloat162float(__float2bfloat16_rn(v)) : v;
  };
  std::fill(w_out, w_out + (size_t)nblk * cin * tapsz, 0.f);
  std::fill(b_out, b_out + (size_t)nblk * cob, 0.f);
  for (int co = 0; co < cout; ++co) {
    const int blk = co / cob, q = co % cob;
    b_out[co] = bias[co];
    for (int ci = 0; ci < cin; ++ci) {
      float* dst = w_out + ((size_t)blk * cin + ci) * tapsz;
      if (mode == CONVT4_S2) {
        // canonical [co][ci][py][px][a][b]
        const float* src = w + ((size_t)co * cin + ci) * 16;
        for (int ph = 0; ph < 4; ++ph)
          for (int t = 0; t < 4; ++t) dst[ph * (4 * cob + 4) + t * cob + q] = rnd(src[ph * 4 + t]);
      } else {
        // canonical [co][ci][ky][kx]
        const float* src = w + ((size_t)co * cin + ci) * 9;
        for (int t = 0; t < 9; ++t) dst[t * cob + q] = rnd(src[t]);
      }
    }
  }
}

void launch_conv(const ConvLayer& L0, const ConvLayer* L1, const Src& in0, const Src* in1,
                 float* out, float* gap, int64_t B, int hi, int wi, bool relu0, bool bf16,
                 cudaStream_t st, const OutLayout* out_layout) {
  Args a{};
  a.in0 = in0;
  if (in1) a.in1 = *in1;
  a.w0 = L0.w;
  a.b0 = L0.b;
  a.w1 = L1 ? L1->w : nullptr;
  a.b1 = L1 ? L1->b : nullptr;
  a.out = out;
  a.gap = gap;
  a.Cin = L0.cin;
  a.Cout = L0.cout;
  a.Hi = hi;
  a.Wi = wi;
  a.Ho = conv_out_h(L0.mode, hi);
  a.Wo = conv_out_h(L0.mode, wi);
  a.relu0 = relu0;
  a.bf16 = bf16;
  a.ol = out_layout ? *out_layout : OutLayout::nchw(L0.cout, a.Ho, a.Wo);
  a.tiles_x = cdiv(a.Wo, kTileW);
  a.ntiles = conv_tiles(L0.mode, a.Ho, a.Wo);
  const int nblk = cdiv(L0.cout, L0.cob);
  const bool dual = L1 != nullptr;
  STDA_CHECK(!dual || (L1->cin == L0.cin && L1->cout == L0.cout && L1->mode == L0.mode),
             "dual conv layers disagree");
  switch (L0.mode) {
    case CONV3_S1:
      STDA_CHECK(!dual, "dual stride-1 conv not supported");
      if (L0.cin <= 4)
        return dispatch_cob<CONV3_S1, false, 4>(L0.cob, a, B, nblk, st);
      return dispatch_cob<CONV3_S1, false, 8>(L0.cob, a, B, nblk, st);
    case CONV3_S2:
      STDA_CHECK(dual, "stride-2 conv is always dual");
      return dispatch_cob<CONV3_S2, true, 4>(L0.cob, a, B, nblk, st);
    case CONVT4_S2:
      STDA_CHECK(dual, "transposed conv is always dual");
      return dispatch_cob<CONVT4_S2, true, 8>(L0.cob, a, B, nblk, st);
  }
  throw Error{"unknown conv mode"};
}

void launch_gate(const float* gap, int ntiles, const float* w, int k, float* gates, int64_t B, int C,
                 int hw, cudaStream_t st) {
  const int threads = std::min(1024, std::max(32, cdiv(C, 32) * 32));
  gate_kernel<<<(unsigned)B, threads, C * sizeof(float), st>>>(gap, ntiles, w, k, gates, C, hw);
  check_launch("gate_kernel");
}

void launch_channel_sum(const float* x, float* gap, int64_t B, int C, int hw, cudaStream_t st) {
  channel_sum_kernel<<<(unsigned)(B * C), 256, 0, st>>>(x, gap, hw);
  check_launch("channel_sum_kernel");
}

void launch_scale(const float* x, const float* gates, float* y, int64_t B, int C, int hw,
                  cudaStream_t st) {
  const int64_t n = B * C * (int64_t)hw;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(148 * 16, (n + 255) / 256));
  scale_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, gates, y, n, hw);
  check_launch("scale_kernel");
}

}  // namespace stda
