/*
 * stda_b200.h — C ABI of the B200-native Radar-STDA inference engine.
 *
 * Replaces the reference's eval-mode forward path:
 *   StdaNet.forward                /root/reference/pkg/stda/src/stda/model.py:185-199
 *   MobileEncoderBlock.forward     model.py:49-53
 *   MobileDecoderBlock.forward     model.py:77-79
 *   EcaBlock.channel_weights/forward model.py:91-98
 *   StdaNet(StdaConfig) + load_state_dict (weights in)  model.py:140-159, train.py:186-193
 *   denoise_dataset batch loop (host buffers in/out)    denoise.py:39-44
 * The reference has no FFI: it is a Python/torch module.  The Python host package
 * `paper_2307_09063_b200` binds this ABI with ctypes.
 *
 * Conventions
 *   - Plain C types only; no torch or C++ types cross the boundary.
 *   - Every int-returning function returns 0 on success, nonzero on failure, and
 *     never throws; stda_last_error() returns a thread-local message for the last
 *     failure on the calling thread.
 *   - Device pointers (x, y, frames, workspace) are caller-owned CUDA global memory
 *     on the plan's device; `stream` is a cudaStream_t passed as void*.
 *   - All work is stream-ordered; no host synchronisation inside, except
 *     stda_forward_host (host buffers), which returns when y_host is written.
 *   - Plans are immutable after create: concurrent calls on distinct workspaces /
 *     streams are safe.
 *
 * Tensors (float32, contiguous, NCHW):
 *   x [B][input_frames][H][W], channel c = frame t-c (newest first, model.py:21-27)
 *   y [B][1][H][W]
 *
 * Folded weight blob (float32; produced on the host by fold.py, exact eval-mode
 * folding of BatchNorm / branch reparameterisation / transposed-conv phases):
 *   stem   W[c0][F][3][3] b[c0]
 *   enc i  (c = c0<<i):            s1 W[c][c][3][3] b[c]; dn W[2c][c][3][3] b[2c];
 *                                  rs W[2c][c][3][3] b[2c]; eca w[k]
 *   dec j  (c2 = c0<<(S-j), c=c2/2): s1 W[c2][c2][3][3] b[c2];
 *                                  up W[c][c2][py][px][a][b] b[c]; rs (same) b[c]; eca w[k]
 *   head   W[1][c0][3][3] b[1]
 * with transposed-conv phases: out[2m+py][2n+px] = sum W[..][py][px][a][b] * in[m+py+a-1][n+px+b-1].
 */
#ifndef STDA_B200_H
#define STDA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STDA_ABI_VERSION 1

#define STDA_PRECISION_FP32 0 /* fp32 parity contract: max|dy|/max|y| <= 1e-4 */
#define STDA_PRECISION_BF16 1 /* bf16 operands, fp32 accumulation: <= 3e-2 */

#define STDA_SCENE_DEFAULT 0 /* 1-5 targets, 1-3 stripes per frame (BASELINE configs 1-4) */
#define STDA_SCENE_DENSE 1   /* 10-20 targets, 1-5 stripes per frame (BASELINE config 5) */

typedef struct stda_plan stda_plan;

/* Mirrors StdaConfig (model.py:101-128) plus the engine precision knob. */
typedef struct {
  int32_t input_frames;
  int32_t stem_channels;
  int32_t stages;
  int32_t eca_kernel;
  int32_t map_height;
  int32_t map_width;
  int32_t precision;
} stda_config;

int stda_abi_version(void);
const char* stda_last_error(void);

/* ---- whole-network plan (replaces StdaNet construction + load_state_dict + eval) ---- */
size_t stda_blob_floats(const stda_config* cfg);
int stda_plan_create(const stda_config* cfg, const float* folded_host_blob, size_t n_floats,
                     int device, stda_plan** out);
void stda_plan_destroy(stda_plan* plan);
/* profiled launch slots of one stda_forward call (stda_forward_profiled / stda_launch_names) */
int stda_launches_per_forward(const stda_plan* plan);
/* kernels launched by one stda_forward call (slots + the separate ECA gate kernels of
   large maps, which are timed inside the slot of the gate they feed) */
int stda_kernels_per_forward(const stda_plan* plan);

/* ---- StdaNet.forward (model.py:185-199) on device buffers ---- */
size_t stda_workspace_bytes(const stda_plan* plan, int64_t batch);
int stda_forward(const stda_plan* plan, const float* x, float* y, int64_t batch, void* workspace,
                 size_t workspace_bytes, void* stream);

/* Same as stda_forward, but records an event after every launch, synchronises, and
 * writes each launch's device time (ms) to ms_per_launch[0 .. launches_per_forward).
 * Measurement aid for bench.py's roofline (names via stda_launch_names). */
int stda_forward_profiled(const stda_plan* plan, const float* x, float* y, int64_t batch,
                          void* workspace, size_t workspace_bytes, void* stream,
                          float* ms_per_launch, int32_t n);
/* Measurement aid (bench.py roofline): one stda_forward (every intermediate in place), then
 * launch slot `slot` alone `reps` times back to back; *ms_per_launch = the average device
 * time per launch (CUDA events around the repeats).  Tensor-core plans only. */
int stda_forward_launch_repeat(const stda_plan* plan, const float* x, float* y, int64_t batch,
                               void* workspace, size_t workspace_bytes, void* stream, int32_t slot,
                               int32_t reps, float* ms_per_launch);
/* ';'-separated launch names in stda_forward order (thread-local storage). */
const char* stda_launch_names(const stda_plan* plan);

/* Stride-1 sliding window over a frame sequence frames[T][H][W]: y[t-(F-1)] is the
 * forward of (frame t, t-1, ..., t-F+1) for t = F-1 .. T-1; bitwise identical to
 * stacking those triplets and calling stda_forward. */
int stda_forward_window(const stda_plan* plan, const float* frames, int64_t n_frames, float* y,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---- host-buffer entry (the end-to-end path): pinned host x in, host y out.
 * Chunks of `chunk` triplets are pipelined H2D / forward / D2H on internal streams
 * ordered after `stream`; returns after y_host is complete.  stda_host_chunk suggests a
 * chunk for a batch: 1/16 of its input bytes, clamped to [16, 128] MB. ---- */
int64_t stda_host_chunk(const stda_plan* plan, int64_t batch);
size_t stda_host_workspace_bytes(const stda_plan* plan, int64_t chunk);
int stda_forward_host(const stda_plan* plan, const float* x_host, float* y_host, int64_t batch,
                      int64_t chunk, void* workspace, size_t workspace_bytes, void* stream);

/* ---- block-level entries (MobileEncoderBlock / MobileDecoderBlock / EcaBlock) ----
 * kind 0 = encoder block (C -> 2C, H,W -> H/2,W/2), blob = [s1 W b, dn W b, rs W b];
 * kind 1 = decoder block (C -> C/2, H,W -> 2H,2W),  blob = [s1 W b, up W b, rs W b]. */
int stda_block_plan_create(int32_t kind, int32_t channels, const float* folded_host_blob,
                           size_t n_floats, int device, stda_plan** out);
size_t stda_block_workspace_bytes(const stda_plan* block, int64_t batch, int32_t h, int32_t w);
int stda_block_forward(const stda_plan* block, const float* x, float* y, int64_t batch, int32_t h,
                       int32_t w, void* workspace, size_t workspace_bytes, void* stream);
/* gates[B][C] = sigmoid(conv1d_k(mean_hw(x))); if y != NULL also y = x * gate. */
int stda_eca(const float* w_dev, int32_t k, const float* x, float* gates, float* y, int64_t batch,
             int32_t channels, int32_t h, int32_t w, void* stream);

/* ---- GPU-side seeded RD-map synthesiser (BASELINE.json configs; counter-based Philox) ----
 * frame f of sequence s depends only on (seed, scene, s, f, H, W).
 * synth_frames: out[i] = frame (first_frame + i) of sequence `seq`, [n][H][W].
 * synth_triplets: x[b][c] = frame (F-1-c) of sequence (first_seq + b), [B][F][H][W]. */
int stda_synth_frames(uint64_t seed, int32_t scene, int64_t seq, int64_t first_frame,
                      int64_t n_frames, int32_t h, int32_t w, float* out, void* stream);
int stda_synth_triplets(uint64_t seed, int32_t scene, int64_t first_seq, int64_t batch,
                        int32_t frames, int32_t h, int32_t w, float* x, void* stream);

/* ---- batched-inference epilogue (replaces the per-sample numpy tail of reference
 * denoise.py:40-42 and NormStats.denormalize, data.py:34-36) ----
 * out[b][x][h] = (clip(y[b][0][h][x], 0, 1) * scale + z_min) * std + mean, float32 with every
 * product and sum rounded separately; scale = float32(z_max - z_min) computed in double.
 * y [batch][1][h][w] (network orientation h = Doppler, w = range) -> out [batch][w][h]
 * (the dataset's range x Doppler orientation).  Device pointers, stream-ordered. */
int stda_denoise_epilogue(const float* y, float* out, int64_t batch, int32_t h, int32_t w, float scale,
                          float z_min, float std_, float mean, void* stream);

/* ---- range-Doppler front end (the step before the denoiser; reference
 * rdlab/rd_pipeline.py:82-159 range_doppler_map -> to_db -> normalize and
 * rdlab/dataset.py:184-211 clutter_filter), float64 inside ----
 * beat: n frames of N x M complex64 (fast time x slow time, re/im interleaved), N <= P,
 * M <= Q (zero padded); P, Q powers of two with P*Q*24 bytes <= 227 KB (64 x 128 default).
 * stats: device pointer to 5 doubles {mean, std, z_min, z_max, degenerate} (the dataset's
 * normalisation record) or NULL for single-frame statistics.  clutter: apply the median
 * clutter filter.  layout 0: out [n][P][Q] range x Doppler; 1: out [n][Q][P] Doppler x range
 * (the network's h x w: a frame stream for stda_forward_window). */
int stda_rd_frontend(const void* beat, int64_t n, int32_t N, int32_t M, int32_t P, int32_t Q,
                     const double* stats, int32_t clutter, int32_t layout, float* out, void* stream);

/* ---- scoring of denoised maps (the step after the denoiser; reference
 * rdlab/evaluation.py:160-201 method "denoised", rdlab/detection_metrics.py:119-259) ----
 * clean: n maps P x Q, complex64 (clean_kind 0: the clean RD map) or float32 magnitudes
 * (kind 1); test_db: n float32 dB maps P x Q (the denoiser's output, range x Doppler).
 * CA-CFAR cross window guard (g0, g1) / training (t0, t1) cells per axis (even), threshold
 * factors alpha_obj (object extraction on |clean|) and alpha_det (detections on the
 * linearised test map), object dilation `margin`.  out: n x {sinr_db, evm, n_object,
 * n_noise, status} doubles (status 0 ok, 1 no object cells, 2 clean map zero at an object
 * cell, 3 empty noise set; sinr/evm NaN unless 0); det_hits: n x P x Q bytes (test-map
 * CFAR hits, for host-side clustering).  Device pointers, float64 inside. */
/* ---- the paper's baselines behind the same forward boundary (reference
 * stda/model.py:202-258), fp32 ----
 * kind 0 = BaselineMlp (blob: torch Linear layout W1 [hidden][h*w], b1 [hidden],
 *          W2 [hidden][hidden], b2, W3 [h*w][hidden], b3 [h*w]);
 * kind 1 = BaselineCae (blob: conv1 w [32][1][3][3] b [32], conv2 w [64][32][3][3] b [64],
 *          convT1 4-phase canonical [32][64][2][2][2][2] b [32] (as the network's ConvT),
 *          convT2 [1][32][2][2][2][2] b [1]); h, w divisible by 4.
 * forward: x [batch][x_channels][h][w] (channel 0 = frame t is used) -> y [batch][1][h][w]. */
int stda_baseline_plan_create(int32_t kind, int32_t h, int32_t w, int32_t hidden, const float* blob,
                              size_t n_floats, int device, stda_plan** out);
size_t stda_baseline_workspace_bytes(const stda_plan* plan, int64_t batch);
int stda_baseline_forward(const stda_plan* plan, const float* x, int32_t x_channels, float* y, int64_t batch,
                          void* workspace, size_t ws_bytes, void* stream);

int stda_score(const void* clean, int32_t clean_kind, const float* test_db, int64_t n, int32_t P, int32_t Q,
               int32_t guard0, int32_t guard1, int32_t train0, int32_t train1, double alpha_obj, double alpha_det,
               int32_t margin, double* out, unsigned char* det_hits, void* stream);

/* ---- debug (no reference counterpart) ----
 * Arm a one-shot clock64 timeline of CTA 0 (+ %globaltimer start/end of every CTA) for the
 * launch_index-th following tensor-core conv launch; dev_buf holds 6 x 8192 uint64 (layout
 * in csrc/tc_kernel.cuh, trace_at / trace_cta). */
int stda_debug_trace(void* dev_buf, int32_t launch_index);

#ifdef __cplusplus
}
#endif
#endif /* STDA_B200_H */
