// tcgen05 conv instantiations: CONV3_S1P, the phase-plane stride-1 conv (see tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_s1p(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  // four phase accumulators per tile: the widest shift group stacks 4 tiles of N (bf16) or
  // 2N (fp32 hi/lo concat) columns, <= 256
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_k<NN, CONV3_S1P, false, PM, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, CONV3_S1P, false, PM, 2>(p, grid, smem, st);
      default: return launch_k<NN, CONV3_S1P, false, PM, 4>(p, grid, smem, st);
    }
  };
  using std::integral_constant;
  STDA_CHECK(npm == kNpmConcat || npm == kNpmBf16 || npm == kNpm3, "phase-plane conv: precision scheme");
  if (npm == kNpm3) {
    STDA_CHECK(n == 16 || n == 32, "phase-plane conv: 3-MMA N");
    if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpm3>{});
    return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpm3>{});
  }
  if (npm == kNpmConcat) {
    STDA_CHECK(n == 16 || n == 32, "phase-plane conv: fp32 needs cout <= 32");
    if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmConcat>{});
    return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmConcat>{});
  }
  switch (n) {
    case 16: return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmBf16>{});
    case 32: return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmBf16>{});
    default: return by_g(integral_constant<int, 64>{}, integral_constant<int, kNpmBf16>{});
  }
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
