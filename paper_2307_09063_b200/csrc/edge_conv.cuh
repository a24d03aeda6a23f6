// Stem / head kernels of the tensor-core path (see edge_conv.cu).
#pragma once

#include "common.cuh"
#include "simt_conv.cuh"

namespace stda {

// x: F input frames (Src strides; NCHW or sliding window) -> s: NHWC [B][H][W][C0], relu.
// w: SIMT layout with cob = 16 ([C0/16][F][9][16]), bias [C0].
void launch_stem_nhwc(const float* w, const float* bias, const Src& x, int F, int C0, float* s,
                      int64_t B, int H, int W, bool bf16, cudaStream_t st);

// y[b][h][w] = bias + conv3x3(d*g + s*gs) over C0 NHWC channels; w [9][C0].
void launch_head_nhwc(const float* w, const float* bias, const float* d, const float* g,
                      const float* s, const float* gs, int C0, float* y, int64_t B, int H, int W,
                      bool bf16, cudaStream_t st);

}  // namespace stda
