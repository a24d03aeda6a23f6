// tcgen05 implicit-GEMM convolution (sm_100a): the tensor-core path of the engine.
//
// GEMM view.  M = output positions, N = output channels (16/32/64), K = taps x Cin.
// Positions are the image linearised with row stride L = plane_width + 1 (planes.cuh):
// the extra column is an always-zero pad, so a 3x3 tap (dy, dx) is a constant shift
// dy*L + dx of the A rows and every tap of every M-tile is a plain UMMA shared-memory
// descriptor offset — no im2col.  Pad positions are computed and discarded.
//   S1  3x3 stride 1      A = input plane (PL),                   9 taps
//   S2  3x3 stride 2      A = 4 phase planes of the input (PP),   tap (dy,dx) -> plane
//                         (py,px) + shift (oy,ox) in {-1,0}^2
//   T   ConvT 4x4 s2 p1   A = input plane (PL), 4 output phases = 4 TMEM accumulators,
//                         each a 2x2 sub-pixel kernel (shifts in {-1,0,1})
//   ROWS 3x3 stride 1 over planes of width 128k: row bands, one A read per (input row, dx)
//                         for three dy taps (tc_kernel.cuh kRowsSL)
// Stage-2 blocks are dual: the block input (second source, own weights) feeds separate
// accumulators; the epilogue forms relu(acc0 + b0) + (acc1 + b1).
//
// fp32 parity: operands are bf16 hi + lo planes (activations) and hi/lo packed weights;
// each product is hi*hi + lo*hi + hi*lo (3 MMAs, fp32 accumulation in TMEM).
//
// Data movement: the operand planes already hold bf16 hi/lo core matrices in HBM, so the
// producer is ONE thread issuing cp.async.bulk copies (A: one contiguous range per
// source/pass/8-channel group; B: one packed weight chunk) completing on an mbarrier
// transaction count.  Roles (352 threads): warp 0 = bulk-copy producer (lane l issues copy
// l); warp 1 = TMEM allocator + single-thread tcgen05.mma issuer; warps 2-9 = epilogue
// (warp % 4 = TMEM lane quarter): tcgen05.ld -> bias/relu/dual -> operand-plane (hi/lo) or
// NHWC fp32 stores + per-item channel sums for ECA; warp 10 = second producer on the
// launches that take it (every other ring stage, tc_kernel.cuh kProd2).  smem stage ring (full/empty) and TMEM
// accumulator slots (full/empty); persistent CTAs.
#pragma once

#include <vector>

#include "common.cuh"
#include "planes.cuh"
#include "simt_conv.cuh"

namespace stda {
namespace tc {

constexpr int kMaxChunks = 16;
constexpr int kMaxTaps = 16;
constexpr int kMaxPlanes = 4;

// Per plane: the taps that read it (position shift = dy*L + dx).
struct PlaneTaps {
  int8_t n;
  int8_t acc[kMaxTaps];
  int8_t dy[kMaxTaps];
  int8_t dx[kMaxTaps];
  int16_t lo, hi;  // min / max shift over the taps, in positions (set by tc_plan)
};

struct TcLayerDesc {
  int mode;        // CONV3_S1 / CONV3_S2 / CONVT4_S2
  int n_src;       // 1 or 2
  int cin, cout;   // cin % 16 == 0; cout in {16, 32, 64}
  int n_planes;    // 1 (S1, T) or 4 (S2)
  int n_acc_src;   // accumulators per source: 1 (S1, S2) or 4 (T)
  int npass;       // 3 (fp32 parity) or 1 (bf16)
  int concat;      // B = [B_hi | B_lo] along N (2 MMAs per tap instead of 3)
  PlaneTaps planes[kMaxPlanes];
  // packed weights: chunk c = plane*(cin/16) + cgroup; inside a chunk for src, tap,
  // weight pass (hi[, lo]): [kgrp 2][n cout][8] bf16.  chunk_off = byte offsets.
  const uint16_t* w = nullptr;
  int64_t chunk_off[kMaxChunks + 1];
  // CONVT4_HALF: the weights are two blocks, py = 0 then py = 1, each chunk-ordered
  // (chunk_off are offsets inside one block); a CTA of an even grid only ever sees items
  // of one py (items alternate py), so it loads / keeps one block
  int64_t half_bytes = 0;
  const float* bias0 = nullptr;
  const float* bias1 = nullptr;
  // the same biases by value: the kernel reads them from its parameter (constant) bank
  float bias0_c[64] = {};
  float bias1_c[64] = {};
};

// Host: canonical fp32 weights (see include/stda_b200.h) -> descriptor + packed bf16.
// plane_w = width of the input plane (stride-1 layers over widths that are multiples of 128
// may be packed for the row-band kernel, CONV3_ROWS; transposed convs over planes >= 256
// wide run as half-phase items); 0 = unknown.
void tc_pack_layer(TcLayerDesc& d, int mode, int cin, int cout, const float* w0, const float* w1,
                   bool bf16, std::vector<uint16_t>& packed, int plane_w = 0);

struct TcGeometry {
  int B, H, W;            // input grid
  int Hp, Wp, L;          // A plane size and linear stride
  int Ho, Wo;             // output grid
  int G;                  // M-tiles of 128 positions per work item
  int stages, slots;      // smem pipeline depth, TMEM accumulator slots
  int items_per_image;
  int tail = 0;           // partial items per image, scheduled last (tc_kernel.cuh item_coords)
  int tmem_cols;
  int P_max;              // staged positions per plane
  uint32_t a_stage_bytes, b_stage_bytes;
  int cps;                // K chunks per ring stage (one barrier round trip per cps chunks)
  uint32_t chunk_a_bytes, chunk_b_bytes;
  bool resident;          // packed weights stay in smem for the whole launch
  int gx_nst = 0;         // gate-in plans: x ring stages
  uint32_t w_total;       // packed weight bytes
  size_t smem_bytes;
};

bool tc_supported(int mode, int cin, int cout);
bool s1p_enabled();  // encoder stride-1 convs as CONV3_S1P over phase planes (env STDA_TC_S1P)
// extra_smem: bytes a kernel variant needs besides the rings / weights (the fused stem's
// frame-row ring); resident_only: weights must stay resident
TcGeometry tc_plan(TcLayerDesc& d, int B, int H, int W, size_t extra_smem = 0, bool resident_only = false);



// Output of one launch: either operand planes (PL over the output grid, or PP phase
// planes of it) or NHWC fp32 with per-item channel sums gap [B][items_per_image][cout].
struct TcOut {
  int mode = 0;  // 0 = NHWC fp32 (+gap), 1 = PL, 2 = PP
  int cp = 0;    // mode 0: chunk-planar fp32 [B][C/16][Ho*Wo][16] instead of NHWC (gate-in input)
  int bf = 0;    // mode 0: the NHWC / chunk-planar values stored as bf16 (bf16 variant)
  float* f32 = nullptr;
  float* gap = nullptr;
  PlBuf pl;
};

// rev: process the images last to first.  A stage-2 conv reads the stage-1 output written
// just before it; running stage 1 in reverse image order makes the stage-1 output it wrote
// last (still in L2) the first thing stage 2 reads.
void tc_launch(const TcLayerDesc& d, const TcGeometry& g, const PlBuf& src0, const PlBuf* src1,
               const TcOut& out, bool relu0, cudaStream_t st, bool rev = false);

// ---- fused stem + first encoder stride-1 conv --------------------------------------------
// The stem (F frames -> 16 channels, relu(conv3x3), model.py:141-144) computed by extra
// warps of the enc0.s1 tcgen05 kernel directly into its A stages; the stem output is
// still written once as operand planes (PP for enc0.s2's residual, PL for the head).
struct TcStem {
  Src x;                          // frames (NCHW or stream windows), x.xp == 1
  int F = 3;
  PlBuf s_pl, s_pp;               // stem output planes
  bool has_pl = true;
  const float* canon = nullptr;   // host: canonical stem weights [16][F][3][3] + bias [16]
};
// true when the fused kernel covers this layer / input (C0 = 16, F <= 4, plain S1 layer,
// W % 4 == 0, W <= 128: the position tiles' halo recompute stays <= 1.5x); env
// STDA_STEM_FUSED=1 enables it (off by default: the stem warps' frame reads compete with
// the MMA operand fetch for shared-memory bandwidth; measured 200 us vs 76 us unfused at C2)
bool tc_stem_fusable(const TcLayerDesc& d1, const TcStem& s, int H, int W);
TcGeometry tc_plan_stem(TcLayerDesc& d1, int B, int H, int W, int F);
void tc_launch_stem(const TcLayerDesc& d1, const TcGeometry& g, const TcStem& s, const TcOut& out,
                    cudaStream_t st, bool rev);

// ---- tensor-core stem (CONV_STEMT) ---------------------------------------------------------
// The stem as a tcgen05 GEMM (simt_conv.cuh CONV_STEMT): im2col warps build each
// position's F x 4 x 4 frame window (bf16 hi/lo) from frame rows staged by bulk copies;
// the epilogue writes the stem output's phase planes (PP).  Layer: make_tc(CONV_STEMT,
// 16 * F, 16, canonical stem weights [16][F][3][3], bias).  Opt-in: env STDA_STEM_TC=1.
bool tc_stemt_ok(const TcStem& s, int H, int W);
TcGeometry tc_plan_stemt(TcLayerDesc& d, int B, int H, int W, int F);
void tc_launch_stemt(const TcLayerDesc& d, const TcGeometry& g, const TcStem& s, const TcOut& out,
                     cudaStream_t st);

// ---- gate-on-load stride-1 conv -------------------------------------------------------------
// The ECA gate (and skip add) of the previous block applied while the A stages of the next
// stride-1 conv are formed (tc_kernel.cuh gate-in role): x = that block's NHWC fp32 output,
// gates = its ECA gates [B][C] (eca_gates_kernel), optional skip planes (PL); the gated
// tensor is also written as PL (+ PP) operand planes for its other consumers — bitwise the
// planes gate_apply writes.  Opt-in (env STDA_GATEIN=1): slower than the gate kernels at C2.
struct TcGateIn {
  const float* x = nullptr;  // chunk-planar fp32 [B][C/16][H*W][16] (TcOut::cp of its producer)
  const float* gates = nullptr;
  PlBuf skip;    // base null: no skip
  PlBuf out_pl;  // the gated tensor as PL
  PlBuf out_pp;  // ... and PP (base null: none)
};
bool gatein_enabled();
bool tc_gatein_ok(const TcLayerDesc& d, const TcGateIn& gi, int H, int W);
TcGeometry tc_plan_gatein(TcLayerDesc& d, int B, int H, int W, const TcGateIn& gi);
bool tc_gatein_fits(const TcLayerDesc& d, int B, int H, int W, const TcGateIn& gi);
void tc_launch_gatein(const TcLayerDesc& d, const TcGeometry& g, const TcGateIn& gi, const TcOut& out,
                      cudaStream_t st, bool rev);

// Debug: record a clock64 timeline of CTA 0 (see tc_kernel.cuh trace_at) into dev_buf
// during the launch_index-th following tc_launch.
void tc_debug_trace(void* dev_buf, int launch_index);

}  // namespace tc
}  // namespace stda
