// Generic FP32-SIMT convolution kernels: the engine's any-config path.
//
// One templated direct-convolution kernel covers every conv-type op of the folded
// network (reference model.py): 3x3 stride-1 (stem, reparameterised stage 1, head),
// 3x3 stride-2 dual-accumulator (encoder stage 2: relu(down(mixed)) + residual(x)),
// and 4-phase sub-pixel ConvTranspose 4x4/s2 dual-accumulator (decoder stage 2).
// Inputs are "sources": x*gate_x + skip*gate_skip evaluated while staging the halo
// tile into shared memory, so ECA scaling and skip adds never round-trip HBM.
#pragma once

#include "common.cuh"

namespace stda {

// CONVT4_HALF: tensor-core only — ConvT 4x4/s2 with one output-row parity py per work item
// CONV3_S1P: tensor-core only — 3x3 stride 1 over a phase-plane (PP) input, the four
//            output phases of a 2x2 pixel block as four accumulators (tc_kernel.cuh)
// CONV_STEMT: tensor-core only — the stem (F frames -> 16 channels, 3x3) as one GEMM per
//            half-resolution position: K = the F x 4 x 4 frame window of the position's 2x2
//            pixel block (one 16-value chunk per frame), N = 4 phases x 16 channels
// CONVT4_SP: tensor-core only — ConvT 4x4/s2 with each output phase's tile origin shifted
//            so that all four phases read the same four A windows (tc_kernel.cuh)
enum ConvMode : int { CONV3_S1 = 0, CONV3_S2 = 1, CONVT4_S2 = 2, CONVT4_HALF = 3, CONV3_ROWS = 4,
                      CONV3_S1P = 5, CONV_STEMT = 6, CONVT4_SP = 7, CONVT4_SPH = 8 };

// A logical input tensor [B][C][H][W]: value = x*gx[b][c] (+ s*gs[b][c]).
// Element (b, c, pixel p = y*W + x) of x lives at x[b*xb + c*xc + p*xp] (NCHW: xp = 1,
// NHWC: xc = 1, xp = C); the optional skip tensor s has its own strides.
struct Src {
  const float* x = nullptr;
  int64_t xb = 0, xc = 0, xp = 1;
  const float* gx = nullptr;
  const float* s = nullptr;
  int64_t sb = 0, sc = 0, sp = 1;
  const float* gs = nullptr;
  int C = 0;
};

inline Src plain_src(const float* x, int C, int H, int W) {
  Src s;
  s.x = x;
  s.C = C;
  s.xc = (int64_t)H * W;
  s.xb = (int64_t)C * H * W;
  s.xp = 1;
  return s;
}

inline Src nhwc_src(const float* x, int C, int H, int W) {
  Src s;
  s.x = x;
  s.C = C;
  s.xc = 1;
  s.xp = C;
  s.xb = (int64_t)C * H * W;
  return s;
}

// Output addressing of a SIMT conv: out[b*ob + c*oc + (y*Wo + x)*op].
struct OutLayout {
  int64_t ob = 0, oc = 0, op = 1;
  static OutLayout nchw(int C, int H, int W) {
    return OutLayout{(int64_t)C * H * W, (int64_t)H * W, 1};
  }
  static OutLayout nhwc(int C, int H, int W) { return OutLayout{(int64_t)C * H * W, 1, C}; }
};

// Device weights of one conv layer in the SIMT layout:
//   w[blk][ci][tapsz], blk = output-channel block of `cob` channels,
//   conv modes: tapsz = 9*cob ([tap][co]); CONVT4_S2: tapsz = 4*(4*cob+4)
//   ([py*2+px][(a*2+b)*cob + co], +4 floats padding per phase against bank conflicts).
//   b[nblk*cob] (zero-padded).
struct ConvLayer {
  int mode = 0, cin = 0, cout = 0, cob = 0, tapsz = 0;
  float* w = nullptr;
  float* b = nullptr;
};

int simt_cob_for(int cout);
int simt_tapsz(int mode, int cob);
// host: canonical weights -> SIMT layout (vectors sized nblk*cin*tapsz and nblk*cob)
void simt_pack(int mode, int cin, int cout, const float* w_canon, const float* b_canon, bool bf16,
               float* w_out, float* b_out);

int conv_out_h(int mode, int hi);
int conv_tiles(int mode, int ho, int wo);

// Launch one conv layer.  L1/in1 non-null => dual: out = relu(acc0+b0) + (acc1+b1).
// relu0 applies relu to the first accumulator.  gap != null => per-tile channel sums
// [B][tiles][cout] of the final output (deterministic, fixed order).
void launch_conv(const ConvLayer& L0, const ConvLayer* L1, const Src& in0, const Src* in1,
                 float* out, float* gap, int64_t B, int hi, int wi, bool relu0, bool bf16,
                 cudaStream_t st, const OutLayout* out_layout = nullptr);

// gates[b][c] = sigmoid(conv1d_k(sum_t gap[b][t][c] / hw)), zero-padded conv1d.
void launch_gate(const float* gap, int ntiles, const float* w, int k, float* gates, int64_t B, int C,
                 int hw, cudaStream_t st);
// gap[b][c] = sum over the whole [h][w] map of x (ntiles = 1 for launch_gate)
void launch_channel_sum(const float* x, float* gap, int64_t B, int C, int hw, cudaStream_t st);
// y = x * gates[b][c]
void launch_scale(const float* x, const float* gates, float* y, int64_t B, int C, int hw,
                  cudaStream_t st);

}  // namespace stda
