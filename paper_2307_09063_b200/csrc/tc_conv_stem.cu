// tcgen05 conv instantiations: the fused stem + first encoder stride-1 conv (STEM kernels,
// tc_kernel.cuh stem role): C0 = 16 output channels, fp32 hi/lo concat or bf16.
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_stem(int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat || npm == kNpmBf16, "fused stem: precision scheme");
  auto by_g = [&](auto npm_c) {
    constexpr int PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_stem_k<16, PM, 1>(p, grid, smem, st);
      case 2: return launch_stem_k<16, PM, 2>(p, grid, smem, st);
      default: return launch_stem_k<16, PM, 4>(p, grid, smem, st);
    }
  };
  if (npm == kNpmConcat) return by_g(std::integral_constant<int, kNpmConcat>{});
  return by_g(std::integral_constant<int, kNpmBf16>{});
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
