// GPU scoring of denoised maps: the step after the denoiser.  One CTA
// per sample, float64 (the reference is numpy float64), for the "denoised" method of
// reference rdlab/evaluation.py:160-201:
//   objects / noise  object_noise_cells (rdlab/detection_metrics.py:205-230): CA-CFAR at
//                    pfa_obj on |clean|, object cells = hits dilated by `margin` (Chebyshev,
//                    toroidal), noise cells = complement of a second dilation
//   test map         db_to_linear_magnitude (rd_pipeline.py:114-121) of the denoised dB map:
//                    max(10^(db/20) - 1e-12, 0)
//   sinr             (detection_metrics.py:233-245) 10 log10(mean |test|^2 over objects /
//                    mean |test|^2 over noise)
//   evm              (:248-259) mean |clean - test| / |clean| over objects
//   detections       ca_cfar (:119-153) on the test map at pfa_det: the hit mask, for the
//                    host-side DBSCAN clustering and AP (which stay on the host)
// ca_cfar: power = |v|^2, the 16-cell cross-shaped training window (guard g, training t
// per axis, toroidal) summed in the reference's offset order (axis 0 then 1, k = g/2+1 ..
// g/2+t/2, sign + then -), hit = power > alpha * sum / n: the same float64 operations, so
// the hit decisions are identical to the reference's.
#include <cuda_runtime.h>

#include "common.cuh"

namespace stda {
namespace {

constexpr int kScThreads = 512;

struct CfarOffsets {
  int n;
  int dp[64], dq[64];
};

__device__ void cfar(const double* mag, unsigned char* hit, int P, int Q, const CfarOffsets& off, double alpha) {
  for (int e = threadIdx.x; e < P * Q; e += kScThreads) {
    const int p = e / Q, q = e - p * Q;
    double acc = 0.0;
    for (int i = 0; i < off.n; ++i) {  // np.roll(power, (dp, dq)): acc[p] += power[p - dp]
      const int pp = (p - off.dp[i] + P) % P, qq = (q - off.dq[i] + Q) % Q;
      const double m = mag[pp * Q + qq];
      acc += m * m;
    }
    const double pw = mag[e] * mag[e];
    hit[e] = pw > alpha * (acc / (double)off.n) ? 1 : 0;
  }
}

__device__ void dilate(const unsigned char* in, unsigned char* out, int P, int Q, int margin) {
  for (int e = threadIdx.x; e < P * Q; e += kScThreads) {
    const int p = e / Q, q = e - p * Q;
    unsigned char v = 0;
    for (int dp = -margin; dp <= margin && !v; ++dp)
      for (int dq = -margin; dq <= margin; ++dq)
        if (in[((p - dp + P) % P) * Q + (q - dq + Q) % Q]) {
          v = 1;
          break;
        }
    out[e] = v;
  }
}

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < kScThreads / 32; ++i) s += red[i];
  return s;
}

// clean: complex64 [n][P][Q] (kind 0) or float32 magnitudes (kind 1); test_db: float32 dB
// maps [n][P][Q].  out: per sample {sinr_db, evm, n_object, n_noise, status} (status 0 ok,
// 1 no object cells, 2 clean map zero at an object cell, 3 empty noise set).
__global__ void __launch_bounds__(kScThreads, 1) score_kernel(const void* __restrict__ clean, int clean_kind,
                                                              const float* __restrict__ test_db, int P, int Q,
                                                              CfarOffsets off, double alpha_obj, double alpha_det,
                                                              int margin, double* __restrict__ out,
                                                              unsigned char* __restrict__ det_hits) {
  extern __shared__ __align__(16) unsigned char ssm[];
  const int PQ = P * Q;
  double* mc = reinterpret_cast<double*>(ssm);  // |clean|
  double* mt = mc + PQ;                          // test, linear magnitude
  unsigned char* m0 = reinterpret_cast<unsigned char*>(mt + PQ);
  unsigned char* m1 = m0 + PQ;
  unsigned char* m2 = m1 + PQ;
  __shared__ double red[kScThreads / 32];
  const int64_t s = blockIdx.x;
  for (int e = threadIdx.x; e < PQ; e += kScThreads) {
    if (clean_kind == 0) {
      const float2 v = static_cast<const float2*>(clean)[s * PQ + e];
      mc[e] = hypot((double)v.x, (double)v.y);
    } else {
      mc[e] = fabs((double)static_cast<const float*>(clean)[s * PQ + e]);
    }
    const double lin = pow(10.0, (double)test_db[s * PQ + e] / 20.0) - 1e-12;
    mt[e] = lin > 0.0 ? lin : 0.0;
  }
  __syncthreads();
  cfar(mt, m0, P, Q, off, alpha_det);  // detections on the test map
  __syncthreads();
  for (int e = threadIdx.x; e < PQ; e += kScThreads) det_hits[s * PQ + e] = m0[e];
  cfar(mc, m1, P, Q, off, alpha_obj);  // object extraction on the clean map
  __syncthreads();
  double nhit = 0.0;
  for (int e = threadIdx.x; e < PQ; e += kScThreads) nhit += m1[e];
  nhit = block_sum(nhit, red);
  dilate(m1, m0, P, Q, margin);  // m0: object cells
  __syncthreads();
  dilate(m0, m2, P, Q, margin);  // m2: excluded (noise = !m2)
  __syncthreads();
  double o_pow = 0.0, o_n = 0.0, n_pow = 0.0, n_n = 0.0, ev = 0.0, zero_ref = 0.0;
  for (int e = threadIdx.x; e < PQ; e += kScThreads) {
    const double t2 = mt[e] * mt[e];
    if (m0[e]) {
      o_pow += t2;
      o_n += 1.0;
      if (mc[e] == 0.0) zero_ref += 1.0;
      else ev += fabs(mc[e] - mt[e]) / mc[e];
    }
    if (!m2[e]) {
      n_pow += t2;
      n_n += 1.0;
    }
  }
  o_pow = block_sum(o_pow, red);
  o_n = block_sum(o_n, red);
  n_pow = block_sum(n_pow, red);
  n_n = block_sum(n_n, red);
  ev = block_sum(ev, red);
  zero_ref = block_sum(zero_ref, red);
  if (threadIdx.x == 0) {
    double* o = out + s * 5;
    const double status = nhit == 0.0 ? 1.0 : zero_ref > 0.0 ? 2.0 : n_n == 0.0 ? 3.0 : 0.0;
    o[0] = status == 0.0 ? 10.0 * log10((o_pow / o_n) / (n_pow / n_n)) : nan("");
    o[1] = status == 0.0 ? ev / o_n : nan("");
    o[2] = o_n;
    o[3] = n_n;
    o[4] = status;
  }
}

CfarOffsets make_offsets(int g0, int g1, int t0, int t1) {
  CfarOffsets off{};
  const int g[2] = {g0, g1}, t[2] = {t0, t1};
  for (int axis = 0; axis < 2; ++axis)
    for (int k = g[axis] / 2 + 1; k <= g[axis] / 2 + t[axis] / 2; ++k)
      for (int sign : {1, -1}) {
        STDA_CHECK(off.n < 64, "CFAR window too large");
        off.dp[off.n] = axis == 0 ? sign * k : 0;
        off.dq[off.n] = axis == 1 ? sign * k : 0;
        ++off.n;
      }
  return off;
}

}  // namespace

void launch_score(const void* clean, int clean_kind, const float* test_db, int64_t n, int P, int Q, int guard0,
                  int guard1, int train0, int train1, double alpha_obj, double alpha_det, int margin, double* out,
                  unsigned char* det_hits, cudaStream_t st) {
  STDA_CHECK(guard0 >= 1 && guard1 >= 1 && guard0 % 2 == 0 && guard1 % 2 == 0 && train0 >= 1 && train1 >= 1 &&
                 train0 % 2 == 0 && train1 % 2 == 0,
             "CFAR guard/training counts must be even and >= 1");
  STDA_CHECK(2 * (guard0 / 2 + train0 / 2) + 1 <= P && 2 * (guard1 / 2 + train1 / 2) + 1 <= Q,
             "CFAR window exceeds the map");
  STDA_CHECK(margin >= 0 && clean_kind >= 0 && clean_kind <= 1, "scoring: bad arguments");
  const size_t smem = (size_t)P * Q * (16 + 3);
  STDA_CHECK(smem <= 200 * 1024, "scoring: map too large for one CTA");
  ensure_dyn_smem(score_kernel, 200 * 1024);
  const CfarOffsets off = make_offsets(guard0, guard1, train0, train1);
  for (int64_t s0 = 0; s0 < n; s0 += 65535) {
    const unsigned ns = (unsigned)std::min<int64_t>(65535, n - s0);
    const size_t esz = clean_kind == 0 ? 8 : 4;
    score_kernel<<<ns, kScThreads, smem, st>>>(static_cast<const char*>(clean) + s0 * P * Q * esz, clean_kind,
                                               test_db + s0 * P * Q, P, Q, off, alpha_obj, alpha_det, margin,
                                               out + s0 * 5, det_hits + s0 * P * Q);
    check_launch("score_kernel");
  }
}

}  // namespace stda
