// tcgen05 conv instantiations: the fused stem + first encoder stride-1 conv (STEM kernels,
// tc_kernel.cuh stem role): C0 = 16 output channels, fp32 hi/lo concat or bf16.
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_stem(int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat || npm == kNpmBf16, "fused stem: precision scheme");
  // G = 4 (W <= 128 keeps >= 6 full items per CTA at the C2 batch) or 2 / 1 for small batches
  auto by_g = [&](auto npm_c, auto f_c) {
    constexpr int PM = decltype(npm_c)::value, FF = decltype(f_c)::value;
    switch (G) {
      case 1: return launch_stem_k<16, PM, 1, FF>(p, grid, smem, st);
      case 2: return launch_stem_k<16, PM, 2, FF>(p, grid, smem, st);
      default: return launch_stem_k<16, PM, 4, FF>(p, grid, smem, st);
    }
  };
  auto by_f = [&](auto npm_c) {
    switch (p.sF) {
      case 1: return by_g(npm_c, std::integral_constant<int, 1>{});
      case 2: return by_g(npm_c, std::integral_constant<int, 2>{});
      case 3: return by_g(npm_c, std::integral_constant<int, 3>{});
      default: return by_g(npm_c, std::integral_constant<int, 4>{});
    }
  };
  if (npm == kNpmConcat) return by_f(std::integral_constant<int, kNpmConcat>{});
  return by_f(std::integral_constant<int, kNpmBf16>{});
}

// the tensor-core stem (CONV_STEMT): 16 channels, F frames, G = 1 / 2 (4 phase
// accumulators of 2 x 16 columns per tile leave two TMEM slots at G = 2)
void dispatch_stemt(int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat || npm == kNpmBf16, "tensor-core stem: precision scheme");
  auto by_g = [&](auto npm_c, auto f_c) {
    constexpr int PM = decltype(npm_c)::value, FF = decltype(f_c)::value;
    if (G == 1) return launch_stemt_k<PM, 1, FF>(p, grid, smem, st);
    return launch_stemt_k<PM, 2, FF>(p, grid, smem, st);
  };
  auto by_f = [&](auto npm_c) {
    switch (p.sF) {
      case 1: return by_g(npm_c, std::integral_constant<int, 1>{});
      case 2: return by_g(npm_c, std::integral_constant<int, 2>{});
      case 3: return by_g(npm_c, std::integral_constant<int, 3>{});
      default: return by_g(npm_c, std::integral_constant<int, 4>{});
    }
  };
  if (npm == kNpmConcat) return by_f(std::integral_constant<int, kNpmConcat>{});
  return by_f(std::integral_constant<int, kNpmBf16>{});
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
