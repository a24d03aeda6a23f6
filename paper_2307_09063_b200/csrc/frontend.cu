// GPU range-Doppler front end: beat frames -> normalised RD maps, the
// step before the denoiser.  One CTA per frame, everything in shared memory, float64
// arithmetic (the reference chain is numpy float64):
//   range_doppler_map  (reference rdlab/rd_pipeline.py:82-95)  P-point DFT over fast time
//                      (axis 0, zero-padded), Q-point DFT over slow time (axis 1), no
//                      window or scaling, Doppler axis fftshift-ed (zero Doppler at Q/2)
//   to_db              (rd_pipeline.py:105-111)  20 log10(|v| + 1e-12)
//   clutter_filter     (rdlab/dataset.py:184-211)  cells of range rows {0, 1} and Doppler
//                      columns {Q/2-1, Q/2, Q/2+1} above the map median are set to it
//                      (median of an even count = mean of the two middle values)
//   normalize          (rd_pipeline.py:135-159)  standardise then min-max into [0, 1]
//                      with given statistics, or the map's own (single-frame mode); a
//                      degenerate record gives 0.5 everywhere
// Output float32, either range x Doppler [P][Q] (the dataset's orientation) or
// Doppler x range [Q][P] (the network's h x w, a frame stream for stda_forward_window).
#include <cuda_runtime.h>

#include "common.cuh"

namespace stda {
namespace {

constexpr int kFeThreads = 512;
constexpr double kDbEps = 1e-12;

struct Cplx {
  double re, im;
};

__device__ __forceinline__ int bitrev(int v, int bits) { return (int)(__brev((unsigned)v) >> (32 - bits)); }

// in-place radix-2 DIT FFT of `count` sequences of length n = 2^bits, element i of
// sequence s at x[s * sstride + i * istride]; tw[k] = exp(-2 pi i k / n), k < n/2
__device__ void fft_batch(Cplx* x, const Cplx* tw, int n, int bits, int count, int istride, int sstride) {
  const int tid = threadIdx.x;
  for (int u = tid; u < n * count; u += kFeThreads) {  // bit-reversal permutation
    const int s = u / n, i = u - s * n, r = bitrev(i, bits);
    if (i < r) {
      Cplx* a = x + (size_t)s * sstride + (size_t)i * istride;
      Cplx* b = x + (size_t)s * sstride + (size_t)r * istride;
      const Cplx t = *a;
      *a = *b;
      *b = t;
    }
  }
  __syncthreads();
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    for (int u = tid; u < (n >> 1) * count; u += kFeThreads) {
      const int s = u / (n >> 1), bf = u - s * (n >> 1);
      const int g = bf / half, j = bf - g * half;
      const Cplx w = tw[j * (n / len)];  // exp(-2 pi i j / len)
      const double cs = w.re, sn = w.im;
      Cplx* a = x + (size_t)s * sstride + (size_t)(g * len + j) * istride;
      Cplx* b = a + (size_t)half * istride;
      const Cplx bv = *b, av = *a;
      const Cplx t = {cs * bv.re - sn * bv.im, cs * bv.im + sn * bv.re};
      *b = {av.re - t.re, av.im - t.im};
      *a = {av.re + t.re, av.im + t.im};
    }
    __syncthreads();
  }
}

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < kFeThreads / 32; ++i) s += red[i];  // fixed order
  return s;
}

__device__ double block_reduce_minmax(double v, double* red, bool want_max) {
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = want_max ? fmax(v, u) : fmin(v, u);
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < kFeThreads / 32; ++i) s = want_max ? fmax(s, red[i]) : fmin(s, red[i]);
  return s;
}

__global__ void __launch_bounds__(kFeThreads, 1) rd_frontend_kernel(const float2* __restrict__ beat, int N, int M,
                                                                     int P, int pbits, int Q, int qbits,
                                                                     const double* __restrict__ stats, int clutter,
                                                                     int layout, float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char fsm[];
  Cplx* X = reinterpret_cast<Cplx*>(fsm);                          // [P][Q]
  double* D = reinterpret_cast<double*>(fsm + (size_t)P * Q * 16);  // [P][Q] dB map
  Cplx* twP = reinterpret_cast<Cplx*>(fsm + (size_t)P * Q * 24);   // [P/2]
  Cplx* twQ = twP + P / 2;                                          // [Q/2]
  __shared__ double red[kFeThreads / 32];
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long sel[2];
  const int tid = threadIdx.x;
  const int64_t f = blockIdx.x;
  const int PQ = P * Q;
  for (int k = tid; k < P / 2 + Q / 2; k += kFeThreads) {  // twiddles exp(-2 pi i k / n)
    const int n = k < P / 2 ? P : Q, kk = k < P / 2 ? k : k - P / 2;
    double sn, cs;
    sincospi(-2.0 * (double)kk / (double)n, &sn, &cs);
    twP[k] = {cs, sn};
  }
  const float2* src = beat + f * (int64_t)N * M;
  for (int e = tid; e < PQ; e += kFeThreads) {  // zero-padded P x Q staging
    const int p = e / Q, q = e - p * Q;
    const float2 v = (p < N && q < M) ? src[(int64_t)p * M + q] : make_float2(0.f, 0.f);
    X[e] = {(double)v.x, (double)v.y};
  }
  __syncthreads();
  fft_batch(X, twP, P, pbits, Q, Q, 1);  // fast time: axis 0 of every column
  fft_batch(X, twQ, Q, qbits, P, 1, Q);  // slow time: axis 1 of every row
  for (int e = tid; e < PQ; e += kFeThreads) {  // fftshift over Doppler + dB
    const int p = e / Q, q = e - p * Q;
    const Cplx v = X[p * Q + ((q + Q / 2) & (Q - 1))];
    D[e] = 20.0 * log10(hypot(v.re, v.im) + kDbEps);
  }
  __syncthreads();
  if (clutter) {
    // median = mean of the two middle values of the sorted map (numpy, even count):
    // exact MSB-first radix select over order-preserving 64-bit keys, 8 passes of 8 bits
    auto key_of = [](double v) {
      const unsigned long long u = (unsigned long long)__double_as_longlong(v);
      return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    };
    auto val_of = [](unsigned long long k) {
      return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
    };
    const int k1 = PQ / 2 - 1;
    unsigned long long prefix = 0, mask = 0;
    int rank = k1;  // rank of the wanted key among the keys matching `prefix`
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += kFeThreads) hist[i] = 0;
      __syncthreads();
      for (int e = tid; e < PQ; e += kFeThreads) {
        // warp-aggregated: the leading digits of dB values barely vary, so per-element
        // atomics would serialise on one or two bins
        const unsigned long long k = key_of(D[e]);
        const int d = (k & mask) == prefix ? (int)((k >> shift) & 255) : 256;
        const unsigned same = __match_any_sync(__activemask(), d);
        if (d < 256 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&hist[d], (unsigned)__popc(same));
      }
      __syncthreads();
      if (tid < 32) {  // warp 0: find the digit holding `rank` (lane l owns bins 8l .. 8l+7)
        unsigned int c[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) tot += (c[i] = hist[tid * 8 + i]);
        unsigned int incl = tot;
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += t;
        }
        const unsigned int excl = incl - tot;
        const bool mine = excl <= (unsigned)rank && (unsigned)rank < incl;
        if (mine) {
          unsigned int cum = excl;
          int d = 0;
          while (cum + c[d] <= (unsigned)rank) cum += c[d++];
          sel[0] = ((unsigned long long)(tid * 8 + d) << 32) | (rank - cum);
        }
      }
      __syncthreads();
      const unsigned long long r = sel[0];
      prefix |= (r >> 32) << shift;
      mask |= 255ull << shift;
      rank = (int)(r & 0xFFFFFFFFu);
      __syncthreads();
    }
    const double v1 = val_of(prefix);
    // the next order statistic: v1 again if more than k1 + 1 keys are <= it, else the
    // smallest key above it
    unsigned int le = 0;
    unsigned long long above = ~0ull;
    for (int e = tid; e < PQ; e += kFeThreads) {
      const unsigned long long k = key_of(D[e]);
      if (k <= prefix) ++le;
      else above = k < above ? k : above;
    }
    for (int o = 16; o > 0; o >>= 1) {
      le += __shfl_xor_sync(0xffffffffu, le, o);
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, above, o);
      above = t < above ? t : above;
    }
    if (tid == 0) {
      sel[0] = 0;
      sel[1] = ~0ull;
    }
    __syncthreads();
    if ((tid & 31) == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&sel[0]), (unsigned long long)le);
      atomicMin(&sel[1], above);
    }
    __syncthreads();
    const double v2 = sel[0] > (unsigned long long)(k1 + 1) ? v1 : val_of(sel[1]);
    const double median = (v1 + v2) / 2.0;
    __syncthreads();
    for (int e = tid; e < PQ; e += kFeThreads) {
      const int p = e / Q, q = e - p * Q;
      const bool region = p <= 1 || (q >= Q / 2 - 1 && q <= Q / 2 + 1);
      if (region && D[e] > median) D[e] = median;
    }
    __syncthreads();
  }
  // normalize
  double mean, stdv, zmin, zmax;
  bool degenerate;
  if (stats != nullptr) {
    mean = stats[0];
    stdv = stats[1];
    zmin = stats[2];
    zmax = stats[3];
    degenerate = stats[4] != 0.0;
  } else {  // single-frame statistics (map_stats, rd_pipeline.py:114-125)
    double s = 0.0;
    for (int e = tid; e < PQ; e += kFeThreads) s += D[e];
    mean = block_sum(s, red) / (double)PQ;
    double s2 = 0.0;
    for (int e = tid; e < PQ; e += kFeThreads) s2 += (D[e] - mean) * (D[e] - mean);
    stdv = sqrt(block_sum(s2, red) / (double)PQ);
    degenerate = stdv == 0.0;
    double lo = 1e308, hi = -1e308;
    if (!degenerate)
      for (int e = tid; e < PQ; e += kFeThreads) {
        const double z = (D[e] - mean) / stdv;
        lo = fmin(lo, z);
        hi = fmax(hi, z);
      }
    zmin = block_reduce_minmax(lo, red, false);
    zmax = block_reduce_minmax(hi, red, true);
    degenerate = degenerate || zmax == zmin;
  }
  float* dst = out + f * (int64_t)PQ;
  for (int e = tid; e < PQ; e += kFeThreads) {
    const int p = e / Q, q = e - p * Q;
    double v = 0.5;
    if (!degenerate) {
      const double z = (D[e] - mean) / stdv;
      v = (z - zmin) / (zmax - zmin);
      v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
    if (layout == 0)
      dst[e] = (float)v;  // [P][Q] range x Doppler
    else
      dst[(int64_t)q * P + p] = (float)v;  // [Q][P] Doppler x range (network h x w)
  }
}

}  // namespace

size_t rd_frontend_smem(int P, int Q) { return (size_t)P * Q * 24 + (size_t)(P + Q) * 8; }

void launch_rd_frontend(const float2* beat, int64_t n, int N, int M, int P, int Q, const double* stats,
                        bool clutter, int layout, float* out, cudaStream_t st) {
  auto log2i = [](int v) {
    int b = 0;
    while ((1 << b) < v) ++b;
    return (1 << b) == v ? b : -1;
  };
  const int pb = log2i(P), qb = log2i(Q);
  STDA_CHECK(pb >= 1 && qb >= 2, "rd front end: P and Q must be powers of two (Q >= 4)");
  STDA_CHECK(N >= 1 && M >= 1 && N <= P && M <= Q, "rd front end: beat frame larger than the FFT");
  constexpr int kMaxDyn = 220 * 1024;  // + the kernel's static reduction scratch
  STDA_CHECK(rd_frontend_smem(P, Q) <= (size_t)kMaxDyn, "rd front end: P x Q too large for one CTA");
  STDA_CHECK(layout == 0 || layout == 1, "rd front end: layout");
  ensure_dyn_smem(rd_frontend_kernel, kMaxDyn);
  for (int64_t f0 = 0; f0 < n; f0 += 65535) {
    const unsigned nf = (unsigned)std::min<int64_t>(65535, n - f0);
    rd_frontend_kernel<<<nf, kFeThreads, rd_frontend_smem(P, Q), st>>>(
        beat + f0 * (int64_t)N * M, N, M, P, pb, Q, qb, stats, clutter ? 1 : 0, layout, out + f0 * (int64_t)P * Q);
    check_launch("rd_frontend_kernel");
  }
}

}  // namespace stda
