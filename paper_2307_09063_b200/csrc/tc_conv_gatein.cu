// tcgen05 conv instantiations: the gate-on-load stride-1 conv (STEM = kGateIn): builder
// warps form the A stages from the previous block's NHWC output x ECA gate (+ skip).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

template <int N, int NPM, int G>
void launch_gatein_k(const Params& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = tc_conv_kernel<N, CONV3_S1, false, NPM, G, 1, kGateIn>;
  ensure_dyn_smem(kern, kMaxSmem);
  launch_pdl(kern, dim3(grid), dim3(threads_of(CONV3_S1, kGateIn)), smem, st, "tc_conv_kernel<gatein>", p);
}

void dispatch_gatein(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  STDA_CHECK(npm == kNpmConcat || npm == kNpmBf16, "gate-in conv: precision scheme");
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_gatein_k<NN, PM, 1>(p, grid, smem, st);
      case 2: return launch_gatein_k<NN, PM, 2>(p, grid, smem, st);
      default: return launch_gatein_k<NN, PM, 4>(p, grid, smem, st);
    }
  };
  using std::integral_constant;
  auto by_n = [&](auto npm_c) {
    switch (n) {
      case 16: return by_g(integral_constant<int, 16>{}, npm_c);
      case 32: return by_g(integral_constant<int, 32>{}, npm_c);
      default: return by_g(integral_constant<int, 64>{}, npm_c);
    }
  };
  if (npm == kNpmConcat) return by_n(integral_constant<int, kNpmConcat>{});
  return by_n(integral_constant<int, kNpmBf16>{});
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
