// tcgen05 conv instantiations: CONVT4_SP, the shifted-phase transposed conv (tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_sp(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat, "shifted-phase ConvT: fp32 hi/lo concat only");
  // (the dual 2 x 4 concatenated phase accumulators fit two TMEM slots only for N = 16)
  STDA_CHECK(n == 16, "shifted-phase ConvT: N = 16");
  auto by_g = [&](auto n_c) {
    constexpr int NN = decltype(n_c)::value;
    switch (G) {
      case 1: return launch_k<NN, CONVT4_SP, true, kNpmConcat, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, CONVT4_SP, true, kNpmConcat, 2>(p, grid, smem, st);
      default: return launch_k<NN, CONVT4_SP, true, kNpmConcat, 4>(p, grid, smem, st);
    }
  };
  return by_g(std::integral_constant<int, 16>{});
}

void dispatch_sph(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat, "shifted half-phase ConvT: fp32 hi/lo concat only");
  auto by_g = [&](auto n_c) {
    constexpr int NN = decltype(n_c)::value;
    switch (G) {
      case 1: return launch_k<NN, CONVT4_SPH, true, kNpmConcat, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, CONVT4_SPH, true, kNpmConcat, 2>(p, grid, smem, st);
      default: return launch_k<NN, CONVT4_SPH, true, kNpmConcat, 4>(p, grid, smem, st);
    }
  };
  STDA_CHECK(n == 16 || n == 32, "shifted half-phase ConvT: N = 16 or 32");
  if (n == 16) return by_g(std::integral_constant<int, 16>{});
  return by_g(std::integral_constant<int, 32>{});
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
