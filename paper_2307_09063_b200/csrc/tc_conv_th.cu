// tcgen05 conv instantiations: CONVT4_HALF (see tc_kernel.cuh).
#include "tc_kernel.cuh"

namespace stda {
namespace tc {
namespace detail {

void dispatch_th(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  dispatch_mode<CONVT4_HALF, true>(n, npm, G, p, grid, smem, st);
}

}  // namespace detail
}  // namespace tc
}  // namespace stda
