// tcgen05 implicit-GEMM convolution (sm_100a): the tensor-core path of the engine.
//
// GEMM view.  M = output positions, N = output channels (16/32/64), K = taps x Cin.
// Positions are the image linearised with row stride L = plane_width + 1: the extra
// column is an always-zero pad, so a 3x3 tap (dy, dx) is a constant shift dy*L + dx of
// the A rows and every tap of every M-tile is a plain UMMA shared-memory descriptor
// offset — no im2col copies.  The pad positions are computed and discarded (W/(W+1)
// efficiency).  Three geometries share one kernel:
//   S1  3x3 stride 1      A = input grid,             1 plane, 9 taps
//   S2  3x3 stride 2      A = 4 input phase planes,   tap (dy,dx) -> plane (py,px), shift
//                         (oy,ox) in {-1,0}^2 (deinterleaved while staging)
//   T   ConvT 4x4 s2 p1   A = input grid, 4 output phases = 4 accumulators, each a 2x2
//                         sub-pixel kernel (taps with shifts in {-1,0,1})
// Stage-2 blocks are dual: a second source (the block input) with its own weights feeds
// separate TMEM accumulators; the epilogue forms relu(acc0 + b0) + (acc1 + b1).
//
// fp32 parity: activations and weights are split into bf16 hi + lo parts and each
// product is formed as hi*hi + lo*hi + hi*lo (3 MMAs, fp32 accumulation in TMEM).
//
// Roles (416 threads): warps 0-7 stage A (fp32 NHWC global -> gate/skip transform ->
// bf16 hi/lo core-matrix layout in smem) and thread 0 bulk-copies the packed weights
// (cp.async.bulk + mbarrier tx); warp 12 allocates TMEM and one lane issues every
// tcgen05.mma; warps 8-11 drain TMEM (tcgen05.ld) into bias/relu/dual epilogues, NHWC
// stores and per-item channel sums for ECA.  mbarrier pipelines: smem stages
// (full/empty) and TMEM accumulator slots (full/empty).  Persistent CTAs.
#pragma once

#include <vector>

#include "common.cuh"
#include "simt_conv.cuh"

namespace stda {
namespace tc {

constexpr int kMaxChunks = 16;
constexpr int kMaxTaps = 16;
constexpr int kMaxPlanes = 4;

// NHWC fp32 logical input: value = x*gx[b][c] + s*gs[b][c] (s, gx, gs optional).
struct TcSrc {
  const float* x = nullptr;
  const float* gx = nullptr;
  const float* s = nullptr;
  const float* gs = nullptr;
};

// Per plane: the taps that read it (position shift = dy*L + dx).
struct PlaneTaps {
  int8_t n;
  int8_t acc[kMaxTaps];
  int8_t dy[kMaxTaps];
  int8_t dx[kMaxTaps];
  int16_t lo, hi;  // min / max shift over the taps, in positions (needs L; set by tc_plan)
};

struct TcLayerDesc {
  int mode;        // CONV3_S1 / CONV3_S2 / CONVT4_S2
  int n_src;       // 1 or 2
  int cin, cout;   // cin % 16 == 0; cout in {16, 32, 64}
  int n_planes;    // 1 (S1, T) or 4 (S2)
  int n_acc_src;   // accumulators per source: 1 (S1, S2) or 4 (T)
  int npass;       // 3 (fp32 parity) or 1 (bf16)
  PlaneTaps planes[kMaxPlanes];
  // packed weights: chunk c = plane*(cin/16) + cgroup; inside a chunk for src, tap,
  // weight pass (hi[, lo]): [kgrp 2][n cout][8] bf16.  chunk_off = byte offsets.
  const uint16_t* w = nullptr;
  int64_t chunk_off[kMaxChunks + 1];
  const float* bias0 = nullptr;
  const float* bias1 = nullptr;
};

// Host: canonical fp32 weights (see include/stda_b200.h) -> descriptor + packed bf16.
void tc_pack_layer(TcLayerDesc& d, int mode, int cin, int cout, const float* w0, const float* w1,
                   bool bf16, std::vector<uint16_t>& packed);

struct TcGeometry {
  int B, H, W;            // input tensor (NHWC, cin channels)
  int Hp, Wp, L;          // A plane size and linear stride
  int Ho, Wo;             // output tensor
  int G;                  // M-tiles of 128 positions per work item
  int stages, slots;      // smem pipeline depth, TMEM accumulator slots
  int items_per_image;
  int tmem_cols;
  int P_max;              // staged positions per plane
  uint32_t a_stage_bytes, b_stage_bytes;
  size_t smem_bytes;
};

bool tc_supported(int mode, int cin, int cout);
TcGeometry tc_plan(TcLayerDesc& d, int B, int H, int W);

// out: NHWC fp32 [B][Ho][Wo][cout]; gap (optional): [B][items_per_image][cout].
void tc_launch(const TcLayerDesc& d, const TcGeometry& g, const TcSrc& src0, const TcSrc* src1,
               float* out, float* gap, bool relu0, cudaStream_t st);

}  // namespace tc
}  // namespace stda
