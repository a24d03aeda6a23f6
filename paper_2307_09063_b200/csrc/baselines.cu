// The paper's baselines behind the same forward boundary (reference
// stda/model.py:202-258), fp32 on the GPU:
//   BaselineMlp  frame t flattened -> Linear(HW,160) -> ReLU -> Linear(160,160) -> ReLU ->
//                Linear(160,HW)  (`linear_kernel`: tiled SIMT GEMM, bias + ReLU fused)
//   BaselineCae  frame t -> Conv3x3(1,32)+ReLU -> MaxPool2 -> Conv3x3(32,64)+ReLU -> MaxPool2
//                -> ConvT4x4s2(64,32)+ReLU -> ConvT4x4s2(32,1)  (the engine's SIMT conv /
//                4-phase ConvT kernels + `maxpool2_kernel`)
#include <cmath>

#include "common.cuh"
#include "simt_conv.cuh"

namespace stda {
namespace {

constexpr int kLT = 64, kLK = 16, kLThreads = 256;  // 64 x 64 output tile, 4 x 4 per thread

// Y[m][n] = act(sum_k X[m*xs + k] * Wt[n][k] + b[n]); X rows with stride xs (frame-t view)
// Split-K: slice blockIdx.z covers k in [z*kslice, (z+1)*kslice) and, when `partial` is set,
// writes its raw sums to partial[z][m][n] (reduced by linear_reduce_kernel in slice order).
__global__ void __launch_bounds__(kLThreads) linear_kernel(const float* __restrict__ X, int64_t xs,
                                                           const float* __restrict__ Wt, const float* __restrict__ b,
                                                           float* __restrict__ Y, int M, int N, int K, int relu,
                                                           int kslice, float* __restrict__ partial) {
  grid_dep_wait();
  __shared__ float xt[kLK][kLT + 4], wt[kLK][kLT + 4];
  const int m0 = blockIdx.y * kLT, n0 = blockIdx.x * kLT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int kb = blockIdx.z * kslice, ke = min(K, kb + kslice);
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += kLK) {
    for (int e = threadIdx.x; e < kLT * kLK; e += kLThreads) {
      const int r = e / kLK, kk = e - r * kLK;
      const int m = m0 + r, n = n0 + r, k = k0 + kk;
      xt[kk][r] = (m < M && k < ke) ? X[(int64_t)m * xs + k] : 0.f;
      wt[kk][r] = (n < N && k < ke) ? Wt[(int64_t)n * K + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kLK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = xt[kk][ty * 4 + i];
        w[i] = wt[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      if (partial) {
        partial[((int64_t)blockIdx.z * M + m) * N + n] = acc[i][j];
        continue;
      }
      float v = acc[i][j] + b[n];
      if (relu) v = fmaxf(v, 0.f);
      Y[(int64_t)m * N + n] = v;
    }
  }
}

__global__ void linear_reduce_kernel(const float* __restrict__ partial, int S, const float* __restrict__ b,
                                     float* __restrict__ Y, int M, int N, int relu) {
  grid_dep_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  float v = 0.f;
  for (int z = 0; z < S; ++z) v += partial[(int64_t)z * M * N + i];  // fixed slice order
  v += b[i % N];
  Y[i] = relu ? fmaxf(v, 0.f) : v;
}

// NCHW 2x2 max pool, stride 2, floor mode, NaN-propagating (torch max_pool2d)
__global__ void maxpool2_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t planes, int H, int W) {
  grid_dep_wait();
  const int Ho = H / 2, Wo = W / 2;
  const int64_t n = planes * Ho * Wo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pl = i / ((int64_t)Ho * Wo);
    const int r = (int)(i - pl * Ho * Wo);
    const int oy = r / Wo, ox = r - oy * Wo;
    const float* p = x + pl * H * W + (int64_t)(2 * oy) * W + 2 * ox;
    float m = p[0];
    for (const float v : {p[1], p[W], p[W + 1]}) m = (v > m || isnan(v)) ? v : m;
    y[i] = m;
  }
}

}  // namespace

// K slices of a layer: a function of K only (not of the batch), so every output is summed in
// the same order whatever the batch size.
int linear_splits(int K) { return K >= 2048 ? K / 256 : 1; }

void launch_linear(const float* X, int64_t xs, const float* Wt, const float* b, float* Y, int M, int N, int K,
                   bool relu, float* partial, cudaStream_t st) {
  STDA_CHECK(M >= 0 && N > 0 && K > 0, "linear: bad shape");
  if (M == 0) return;
  STDA_CHECK(cdiv(M, kLT) <= 65535, "linear: batch too large for one launch");
  const int S = linear_splits(K), kslice = cdiv(K, S);
  STDA_CHECK(S == 1 || partial != nullptr, "linear: split-K needs a partial buffer");
  launch_pdl(linear_kernel, dim3(cdiv(N, kLT), cdiv(M, kLT), S), dim3(kLThreads), 0, st, "linear_kernel", X, xs,
             Wt, b, Y, M, N, K, relu ? 1 : 0, kslice, S > 1 ? partial : nullptr);
  if (S > 1)
    launch_pdl(linear_reduce_kernel, dim3(cdiv(M * N, 256)), dim3(256), 0, st, "linear_reduce_kernel",
               (const float*)partial, S, b, Y, M, N, relu ? 1 : 0);
}

void launch_maxpool2(const float* x, float* y, int64_t planes, int H, int W, cudaStream_t st) {
  const int64_t n = planes * (H / 2) * (W / 2);
  if (n == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv((int)std::min<int64_t>(n, 1 << 30), 256), 148 * 16);
  launch_pdl(maxpool2_kernel, dim3(grid), dim3(256), 0, st, "maxpool2_kernel", x, y, planes, H, W);
}

}  // namespace stda
