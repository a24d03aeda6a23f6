// Batched-inference epilogue (reference denoise.py:40-42, data.py:34-36):
//   out[b][x][h] = denormalize(clip(y[b][0][h][x], 0, 1))
//   denormalize(v) = (v * (z_max - z_min) + z_min) * std + mean
// i.e. the network output map (h = Doppler, x = range) is clipped, mapped back to dB with the
// dataset's normalisation statistics and transposed to the generator's range x Doppler
// orientation, in one pass over HBM.  The arithmetic is float32 with every multiply and add
// rounded separately (no FMA contraction), as numpy evaluates the reference's expression on
// a float32 array with Python-float operands: the result is bitwise identical.
#include "common.cuh"

namespace stda {
namespace {

constexpr int kTile = 32, kRows = 8;

__global__ void __launch_bounds__(kTile* kRows) denoise_epilogue_kernel(const float* __restrict__ y,
                                                                       float* __restrict__ out, int H, int W,
                                                                       float scale, float z_min, float stdv,
                                                                       float mean) {
  grid_dep_wait();
  __shared__ float tile[kTile][kTile + 1];
  const int64_t b = blockIdx.z;
  const int h0 = blockIdx.y * kTile, x0 = blockIdx.x * kTile;
  const float* src = y + b * (int64_t)H * W;
  float* dst = out + b * (int64_t)H * W;
  for (int r = threadIdx.y; r < kTile; r += kRows) {
    const int h = h0 + r, x = x0 + threadIdx.x;
    if (h < H && x < W) {
      float v = src[(int64_t)h * W + x];
      v = v < 0.f ? 0.f : (v > 1.f ? 1.f : v);  // np.clip (NaN stays NaN)
      const float z = __fadd_rn(__fmul_rn(v, scale), z_min);
      tile[r][threadIdx.x] = __fadd_rn(__fmul_rn(z, stdv), mean);
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < kTile; r += kRows) {
    const int x = x0 + r, h = h0 + threadIdx.x;
    if (x < W && h < H) dst[(int64_t)x * H + h] = tile[threadIdx.x][r];
  }
}

}  // namespace

void launch_denoise_epilogue(const float* y, float* out, int64_t B, int H, int W, float scale, float z_min,
                             float stdv, float mean, cudaStream_t st) {
  STDA_CHECK(B >= 0 && H > 0 && W > 0, "denoise epilogue: bad shape");
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    const unsigned nb = (unsigned)std::min<int64_t>(65535, B - b0);
    launch_pdl(denoise_epilogue_kernel, dim3(cdiv(W, kTile), cdiv(H, kTile), nb), dim3(kTile, kRows), 0, st,
               "denoise_epilogue_kernel", y + b0 * (int64_t)H * W, out + b0 * (int64_t)H * W, H, W, scale, z_min,
               stdv, mean);
  }
}

}  // namespace stda
