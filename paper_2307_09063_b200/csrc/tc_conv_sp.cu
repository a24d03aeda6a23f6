// tcgen05 conv instantiations: CONVT4_SP, the shifted-phase transposed conv (tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_sp(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  // fp32: 3-MMA (default) or concat, N = 16 (the dual 2 x 4 phase accumulators fit two TMEM
  // slots); bf16: one pass, N = 16 or 32
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_k<NN, CONVT4_SP, true, PM, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, CONVT4_SP, true, PM, 2>(p, grid, smem, st);
      default: return launch_k<NN, CONVT4_SP, true, PM, 4>(p, grid, smem, st);
    }
  };
  using std::integral_constant;
  if (npm == kNpmBf16) {
    STDA_CHECK(n == 16 || n == 32, "shifted-phase ConvT (bf16): N = 16 or 32");
    if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmBf16>{});
    return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmBf16>{});
  }
  STDA_CHECK(n == 16, "shifted-phase ConvT: N = 16");
  if (npm == kNpm3) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpm3>{});
  STDA_CHECK(npm == kNpmConcat, "shifted-phase ConvT: precision scheme");
  return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmConcat>{});
}

void dispatch_sph(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat || npm == kNpm3, "shifted half-phase ConvT: fp32 schemes only");
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_k<NN, CONVT4_SPH, true, PM, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, CONVT4_SPH, true, PM, 2>(p, grid, smem, st);
      default: return launch_k<NN, CONVT4_SPH, true, PM, 4>(p, grid, smem, st);
    }
  };
  STDA_CHECK(n == 16 || n == 32, "shifted half-phase ConvT: N = 16 or 32");
  using std::integral_constant;
  if (npm == kNpm3) {
    if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpm3>{});
    return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpm3>{});
  }
  if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmConcat>{});
  return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmConcat>{});
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
