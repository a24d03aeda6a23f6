// Stem / head kernels of the tensor-core path (see edge_conv.cu).
#pragma once

#include "common.cuh"
#include "planes.cuh"
#include "simt_conv.cuh"

namespace stda {

// x: F input frames (Src strides; NCHW or sliding window) -> relu(conv3x3) written as
// operand planes pl (PL over H x W) and pp (PP over H/2 x W/2).
// pl.base == nullptr: phase planes only (see stem_pp_only_ok).
// w: SIMT layout with cob = 16 ([C0/16][F][9][16]), bias [C0].
// canon_host (optional): host copy of the canonical weights [C0][F][3][3] + bias [C0];
// with C0 = 16 and F <= 4 it selects the constant-bank stem kernel.
// The stem may write its phase planes only (pl.base == nullptr): enc0.s1 then reads the
// phase planes (CONV3_S1P) and the strip head reads its skip from them.  True when both
// kernels cover the shape (C0 = 16, F <= 4, W in {32, 64, 128}).
bool stem_pp_only_ok(int C0, int F, int H, int W);

void launch_stem_planes(const float* w, const float* bias, const Src& x, int F, int C0,
                        const PlBuf& pl, const PlBuf& pp, int64_t B, int H, int W, bool bf16,
                        cudaStream_t st, const float* canon_host = nullptr);

// y[b][h][w] = bias + conv3x3(d * gate + skip) over C0 channels, gate = ECA of d computed
// from its per-item channel sums gap [B][items][C0]; d NHWC fp32, skip a PL plane.
// w [9][C0].
// w_host (optional): host copy of w ([9][C0]); the strip head then takes the weights from
// the kernel-parameter bank instead of shared memory.
void launch_head_fused(const float* w, const float* bias, const float* gap, int items,
                       const float* eca_w, int k, const float* d, const PlBuf& skip, int C0, float* y,
                       int64_t B, int H, int W, bool bf16, cudaStream_t st, const float* w_host = nullptr,
                       bool d_bf16 = false);
// d_bf16 (the bf16 variant's last stage-2 output stored as bf16): strip / tile heads only
bool head_bf16_ok(int C0, int64_t B, int H, int W, const PlBuf& skip);

}  // namespace stda
