// GPU-side seeded RD-map synthesiser (BASELINE.json generator).
//
// A frame is the normalised log-magnitude of
//     z[h][w] = sigma_row[h] * (n_re + j n_im)  +  sum_targets A e^{j phi}  at the target bin
// with h = Doppler bin, w = range bin (the reference's network orientation, data.py:95):
//   * receiver noise: complex Gaussian, sigma = 1 (rdlab signal_model.py:263-266 convention);
//   * point targets: 1-5 (scene 0) or 10-20 (scene 1) per sequence, amplitude
//     20log10(A) ~ U[10,30] dB, position p0 + f*v (v in {-1,0,1}^2, wrapped), random
//     phase per frame — closed form, so any frame is generable independently
//     (like rdlab dataset.py:228-241 targets_at_frame);
//   * interference stripes: 1-3 (scene 0) or 1-5 (scene 1) per frame, each a band of
//     U{1..8} Doppler rows across all range bins with sigma raised by 10^(P/20),
//     P ~ U[5,20] dB;
//   * 20*log10(|z| + 1e-12) (rd_pipeline.py:22-23,103-108), then per-frame min-max to
//     [0,1] (rdlab normalize is affine, rd_pipeline.py:121-154).
// Randomness is counter-based Philox4x32-10 keyed by (seed, scene), counter
// (purpose, sequence, frame, element), mirroring rdlab's seeded_rng
// (signal_model.py:25-38): results depend only on (seed, scene, seq, frame, H, W).
#include <algorithm>

#include "common.cuh"

namespace stda {
namespace {

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ float u01(uint32_t v) {  // (0, 1)
  return ((v >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

enum Purpose : uint32_t { kSeq = 1, kFrame = 2, kNoise = 3 };

struct Key {
  uint32_t k0, k1;
};

__device__ __forceinline__ U4 draw(Key k, uint32_t purpose, int64_t seq, int64_t frame, uint32_t elem) {
  // counter = (purpose | element<<2, seq lo, seq hi, frame)
  const U4 c{purpose | (elem << 2), (uint32_t)seq, (uint32_t)((uint64_t)seq >> 32), (uint32_t)frame};
  return philox(c, k.k0, k.k1);
}

constexpr int kMaxTargets = 20;
constexpr int kThreads = 512;

__global__ void __launch_bounds__(kThreads) synth_kernel(Key key, int scene, int64_t seq0,
                                                          int64_t seq_step, int64_t frame0,
                                                          int frames_per_seq_out, int frame_order,
                                                          int H, int W, float* __restrict__ out) {
  // blockIdx.x enumerates output frames: o = i_seq * frames_per_seq_out + i_frame
  const int64_t o = blockIdx.x;
  const int64_t i_seq = o / frames_per_seq_out;
  const int i_fr = (int)(o - i_seq * frames_per_seq_out);
  const int64_t seq = seq0 + i_seq * seq_step;
  // frame_order 0: frame = frame0 + i_fr; 1 (triplet channels): frame = F-1-i_fr
  const int64_t frame = frame_order == 0 ? frame0 + i_fr : (int64_t)(frames_per_seq_out - 1 - i_fr);

  __shared__ int t_h[kMaxTargets], t_w[kMaxTargets];
  __shared__ float t_re[kMaxTargets], t_im[kMaxTargets];
  __shared__ int n_t;
  __shared__ float red_min[kThreads / 32], red_max[kThreads / 32];
  extern __shared__ float sigma_row[];  // [H]

  if (threadIdx.x == 0) {
    const U4 r = draw(key, kSeq, seq, 0, 0);
    n_t = scene == 0 ? 1 + (int)(u01(r.x) * 5.f) : 10 + (int)(u01(r.x) * 11.f);
    n_t = min(n_t, kMaxTargets);
  }
  for (int h = threadIdx.x; h < H; h += blockDim.x) sigma_row[h] = 1.f;
  __syncthreads();
  if (threadIdx.x < n_t) {
    const int k = threadIdx.x;
    const U4 p = draw(key, kSeq, seq, 0, 1 + k);          // sequence-level target draw
    const int h0 = (int)(u01(p.x) * H), w0 = (int)(u01(p.y) * W);
    const int vh = (int)(p.z % 3u) - 1, vw = (int)((p.z / 3u) % 3u) - 1;
    const float amp_db = 10.f + 20.f * u01(p.w);
    const U4 q = draw(key, kFrame, seq, frame, 64 + k);   // per-frame phase
    const float phi = 6.283185307179586f * u01(q.x);
    const float amp = exp10f(amp_db / 20.f);
    int64_t hh = (h0 + (int64_t)vh * frame) % H, ww = (w0 + (int64_t)vw * frame) % W;
    if (hh < 0) hh += H;
    if (ww < 0) ww += W;
    t_h[k] = (int)hh;
    t_w[k] = (int)ww;
    float s, c;
    sincosf(phi, &s, &c);
    t_re[k] = amp * c;
    t_im[k] = amp * s;
  }
  if (threadIdx.x == 0) {
    const U4 r = draw(key, kFrame, seq, frame, 0);
    const int n_s = scene == 0 ? 1 + (int)(u01(r.x) * 3.f) : 1 + (int)(u01(r.x) * 5.f);
    for (int s = 0; s < n_s; ++s) {
      const U4 d = draw(key, kFrame, seq, frame, 1 + s);
      const int h0 = (int)(u01(d.x) * H);
      const int width = 1 + (int)(u01(d.y) * 8.f);
      const float sig = exp10f((5.f + 15.f * u01(d.z)) / 20.f);
      for (int i = 0; i < width; ++i) {
        const int h = (h0 + i) % H;
        sigma_row[h] = fmaxf(sigma_row[h], sig);
      }
    }
  }
  __syncthreads();

  float* dst = out + o * (int64_t)H * W;
  const int n = H * W;
  float vmin = 3.4e38f, vmax = -3.4e38f;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int h = e / W, w = e - h * W;
    const U4 r = draw(key, kNoise, seq, frame, (uint32_t)e);
    const float rad = sqrtf(-2.f * logf(u01(r.x)));
    float s, c;
    sincosf(6.283185307179586f * u01(r.y), &s, &c);
    const float sg = sigma_row[h];
    float re = sg * rad * c, im = sg * rad * s;
    for (int k = 0; k < n_t; ++k)
      if (t_h[k] == h && t_w[k] == w) {
        re += t_re[k];
        im += t_im[k];
      }
    const float db = 20.f * log10f(sqrtf(re * re + im * im) + 1e-12f);
    dst[e] = db;
    vmin = fminf(vmin, db);
    vmax = fmaxf(vmax, db);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, off));
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, off));
  }
  if ((threadIdx.x & 31) == 0) {
    red_min[threadIdx.x >> 5] = vmin;
    red_max[threadIdx.x >> 5] = vmax;
  }
  __syncthreads();
  vmin = red_min[0];
  vmax = red_max[0];
  for (int i = 1; i < kThreads / 32; ++i) {
    vmin = fminf(vmin, red_min[i]);
    vmax = fmaxf(vmax, red_max[i]);
  }
  // division (not a reciprocal multiply) so the brightest bin maps to exactly 1
  const float range = vmax - vmin;
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    dst[e] = range > 0.f ? (dst[e] - vmin) / range : 0.f;
}

Key make_key(uint64_t seed, int scene) {
  return Key{(uint32_t)seed ^ 0x5354DA00u, (uint32_t)(seed >> 32) ^ (uint32_t)(scene * 0x9E3779B9u)};
}

}  // namespace

void launch_synth(uint64_t seed, int scene, int64_t seq0, int64_t seq_step, int64_t frame0,
                  int frames_per_seq, int frame_order, int64_t n_out, int H, int W, float* out,
                  cudaStream_t st) {
  STDA_CHECK(scene == 0 || scene == 1, "scene must be 0 (default) or 1 (dense)");
  STDA_CHECK(H > 0 && W > 0, "bad map size");
  const Key key = make_key(seed, scene);
  STDA_CHECK(n_out < (1ll << 31) && (int64_t)H * W < (1ll << 30), "synth request too large");
  if (n_out == 0) return;
  synth_kernel<<<(unsigned)n_out, kThreads, H * sizeof(float), st>>>(key, scene, seq0, seq_step, frame0,
                                                                     frames_per_seq, frame_order, H, W, out);
  check_launch("synth_kernel");
}

}  // namespace stda
