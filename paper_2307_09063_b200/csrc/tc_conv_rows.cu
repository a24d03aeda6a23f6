// tcgen05 conv instantiations: CONV3_ROWS, the row-band stride-1 conv (see tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_rows(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  // three stacked tap blocks per MMA: 3 * N (bf16) or 3 * 2N (fp32 concat) <= 256 columns
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 2: return launch_k<NN, CONV3_ROWS, false, PM, 2>(p, grid, smem, st);
      case 4: return launch_k<NN, CONV3_ROWS, false, PM, 4>(p, grid, smem, st);
      default: return launch_k<NN, CONV3_ROWS, false, PM, 8>(p, grid, smem, st);
    }
  };
  using std::integral_constant;
  if (npm == kNpmConcat) {
    STDA_CHECK(n == 16 || n == 32, "row-band conv: fp32 needs cout <= 32");
    if (n == 16) return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmConcat>{});
    return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmConcat>{});
  }
  STDA_CHECK(npm == kNpmBf16, "row-band conv: precision scheme");
  switch (n) {
    case 16: return by_g(integral_constant<int, 16>{}, integral_constant<int, kNpmBf16>{});
    case 32: return by_g(integral_constant<int, 32>{}, integral_constant<int, kNpmBf16>{});
    default: return by_g(integral_constant<int, 64>{}, integral_constant<int, kNpmBf16>{});
  }
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
