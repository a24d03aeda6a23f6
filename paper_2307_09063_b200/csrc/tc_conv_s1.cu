// tcgen05 conv instantiations: CONV3_S1 (see tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_s1(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  dispatch_mode<CONV3_S1, false>(n, npm, G, p, grid, smem, st);
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
