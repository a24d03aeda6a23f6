// tcgen05 implicit-GEMM convolution: device code (internal header of tc_conv_*.cu).
//
// The kernel is specialised at compile time on (N, geometry, dual, precision scheme, G):
// tap tables are constexpr and the per-chunk MMA stream is fully unrolled, so each
// tcgen05.mma costs a few uniform adds to issue (tools/mma_bench.cu: an M=128 SS-mode
// MMA executes in 39-48 cycles for N = 16..64, i.e. (A + B bytes) / 128 B/clk).
// Instantiations are split by geometry over tc_conv_s1.cu / _s2.cu / _t.cu.
#pragma once

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "tc_conv.cuh"

namespace stda {
namespace tc {
namespace detail {

constexpr int kProdWarp = 0;   // lane 0: cp.async.bulk producer
constexpr int kMmaWarp = 1;    // TMEM allocator + tcgen05.mma issuer
constexpr int kEpiWarp0 = 2;   // warps 2..9: epilogue (warp % 4 = TMEM lane quarter)
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
// fused stem (STEM kernels, stem + first encoder stride-1 conv): warps 10.. compute the
// stem straight into the A stages (tc_kernel.cuh stem role); warp 0 stages the frame rows
constexpr int kStemWarp0 = kEpiWarp0 + kEpiWarps;
constexpr int kStemWarps = 8;
constexpr int kStemThreads = kStemWarps * 32;
constexpr int kThreadsStem = kThreads + kStemThreads;
constexpr int kStemC = 16, kStemMaxF = 4;
// the tensor-core stem (CONV_STEMT) needs only 4 im2col warps: fewer threads leave the
// epilogue warps the registers for batched TMEM loads
constexpr int kStemtThreads = 128;
// gate-on-load stride-1 conv (STEM template value kGateIn, MODE CONV3_S1): 6 builder warps
// form the A stages from the previous block's NHWC fp32 output x gate (+ skip), and write the
// gated tensor's operand planes as a side output (tc_kernel.cuh gate-in role)
constexpr int kGateIn = 8;
constexpr int kGateInThreads = 192;
__host__ __device__ constexpr int stem_threads(int mode, int stem = 0) {
  return stem == kGateIn ? kGateInThreads : mode == CONV_STEMT ? kStemtThreads : kStemThreads;
}
// epilogue warps: 8.  A build with -DSTDA_EPI16_SP=1 gives the shifted-phase transposed
// conv 16 (its epilogue binds once the MMA stream is 4 windows per chunk); measured slower
// at C2 (dec1.s2 48.4 vs 41.1 us: 113 registers per thread, spills), so off.
#ifndef STDA_EPI16_SP
#define STDA_EPI16_SP 0
#endif
constexpr int kEpiWarpsMax = STDA_EPI16_SP ? 16 : kEpiWarps;
__host__ __device__ constexpr int epi_warps(int mode) { return mode == CONVT4_SP && STDA_EPI16_SP ? 16 : kEpiWarps; }
// Kernels without STEM warps run a second producer warp (the warp after the epilogue warps):
// the two take alternate ring stages.  One warp needs ~1000 cycles to post a stage of the
// stride-2 convs (wait, byte count, address arithmetic, one bulk copy per lane) against
// ~800-1200 cycles of MMA issue per stage, and the MMA warp waited on it
// (profiles/r2_cta_trace_v2.txt: enc1.s2 MMA wait-full 604 cycles per chunk).
constexpr int kProd2 = 1;
__host__ __device__ constexpr int threads_of(int mode, int stem) {
  return stem ? kThreads + stem_threads(mode, stem) : (kEpiWarp0 + epi_warps(mode) + kProd2) * 32;
}
constexpr int kMaxSmem = 227 * 1024;
constexpr int kMaxStages = 6;  // smem ring depth cap
constexpr int kMaxSlots = 4;   // TMEM accumulator slots cap

// precision schemes
constexpr int kNpmBf16 = 0;    // one pass: A_hi x B_hi
constexpr int kNpm3 = 1;       // hi*hi + lo*hi + hi*lo, three MMAs of width N
constexpr int kNpmConcat = 2;  // A_hi x [B_hi | B_lo] (width 2N) + A_lo x B_hi (width N)

struct Params {
  TcLayerDesc d;
  PlBuf src[2];
  TcOut out;
  int H, W, C;            // input grid
  int Hp, Wp, L, Ho, Wo;
  uint32_t L_mul;          // ceil(2^32 / L): q / L == umulhi(q, L_mul) for q * L < 2^32
  int G, stages, slots, items_per_image, total_items;
  int tail;  // partial items per image (the last 1, HALF 2) scheduled after all full ones
  int rev;   // walk the images last to first (L2 reuse of the previous launch's output)
  int P_max;
  uint32_t a_stage_bytes, b_stage_bytes, slot_cols;
  int cps;                          // K chunks per ring stage (1 or 2)
  uint32_t chunk_a_bytes, chunk_b_bytes;  // one chunk's A (all sources) / staged weights
  int resident;       // all packed weights loaded once into smem (else one chunk per stage)
  uint32_t w_total;   // packed weight bytes of the layer
  uint32_t tmem_cols;
  int relu0;
  unsigned long long* trace;  // debug timeline of CTA 0 (null in normal runs)
  int early_trigger;          // griddepcontrol.launch_dependents at kernel start
  int prod2;                  // the second producer warp takes every other ring stage (else it idles)
  int dbg;                    // debug ablations (env STDA_TC_DBG; 0 in normal runs):
                              // 1 no epilogue stores, 2 no TMEM loads, 4 no A copies after
                              // the first fill, 8 epilogue only releases the slot
  // ---- fused stem (STEM kernels only) ----
  // frames: element (b, ci, y, x) at sx[b*sxb + ci*sxc + y*W + x] (NCHW or stream windows)
  const float* sx;
  int64_t sxb, sxc;
  int sF;                     // input frames (<= kStemMaxF)
  int stem_xrows;             // frame rows staged per item (x ring stage = sF * rows * W floats)
  uint32_t stem_xstage;       // bytes per x ring stage
  PlBuf s_pl, s_pp;           // stem output written as operand planes (enc0.s2 / head read them)
  int s_has_pl;
  // relu(conv3x3(frames)) weights [ci][ky][kx][co] (co pairs = 8-byte units) and bias, read
  // from the parameter bank by every FFMA2 (uniform across the warp)
  alignas(16) float stem_w[kStemMaxF * 9 * kStemC];
  alignas(16) float stem_b[kStemC];
  // ---- gate-on-load (STEM == kGateIn) ----
  const float* gx;      // the block input before its ECA gate: NHWC fp32 [B][H][W][C]
  const float* gates;   // ECA gates [B][C] (eca_gates_kernel)
  PlBuf gskip;          // optional skip added after the gate (base null: none), PL planes
  PlBuf gpl, gpp;       // side outputs: the gated tensor as PL (always) and PP (base null: none)
  uint32_t gx_skip_off; // x ring stage: skip ranges after the rows (bytes)
  int gx_nst;           // x ring stages (2..4)
};

// ---- debug timeline (stda_debug_trace): clock64 stamps of CTA 0, one region per role ---
// region 0: producer  [k*2 + {empty acquired, chunk issued}]
// region 1: MMA warp  [k*2 + {full acquired, chunk issued}]
// region 2: MMA warp  [ic]  TMEM slot acquired
// region 3: epilogue  [ic*2 + {TMEM full acquired, slot released}]
// region 4: [0] kernel start, [1] kernel end
constexpr int kTraceRegion = 8192;
__device__ __forceinline__ void trace_at(unsigned long long* tr, int region, int idx) {
  if (tr != nullptr && blockIdx.x == 0 && idx < kTraceRegion)
    tr[region * kTraceRegion + idx] = clock64();
}
// region 5: every CTA, [2*cta + {0 start, 1 end}] in %globaltimer ns (comparable across SMs)
__device__ __forceinline__ void trace_cta(unsigned long long* tr, int which) {
  if (tr == nullptr || 2 * (int)blockIdx.x + 1 >= kTraceRegion) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  tr[5 * kTraceRegion + 2 * blockIdx.x + which] = t;
}
// region 5 from 512: every CTA, [512 + 32*cta + ic] = %globaltimer when the epilogue
// released item ic's accumulators (ic < 31); [512 + 32*cta + 31] = first MMA stage acquired
__device__ __forceinline__ void trace_cta_item(unsigned long long* tr, int idx) {
  if (tr == nullptr || idx > 31 || 512 + 32 * (int)blockIdx.x + 31 >= kTraceRegion) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  tr[5 * kTraceRegion + 512 + 32 * blockIdx.x + idx] = t;
}

// Work item n -> (image, item of the image).  The last `tail` items of an image cover a
// partial tile group; they are numbered after every full item, so the final round of the
// strided persistent schedule is made of the cheap partial items instead of full ones (the
// image-major numbering left e.g. 40 full enc0.s1 items for a 15th round on 40 CTAs).
// Parity of `it` equals parity of n when tail is even (HALF: items alternate py).
__device__ __forceinline__ void item_coords(int n, const Params& p, int& b, int& it) {
  const int full = p.items_per_image - p.tail;
  const int nf = (p.total_items / p.items_per_image) * full;
  if (n < nf) {
    b = n / full;
    it = n - b * full;
  } else {
    const int r = n - nf;
    b = r / p.tail;
    it = full + (r - b * p.tail);
  }
  if (p.rev) b = p.total_items / p.items_per_image - 1 - b;
}

// ---- compile-time tap tables (must match plane_taps() on the host) ----------------
// S1:  t = ky*3+kx, shift (ky-1, kx-1)
// S2:  plane (py,px) = (dy != 0, dx != 0); shift (dy == -1 ? -1 : 0, dx == -1 ? -1 : 0),
//      taps of a plane in (ky, kx) order
// T:   t = ph*4 + a*2 + b, accumulator ph, shift (py + a - 1, px + b - 1)
// HALF (ConvT, one output-row parity py per work item): t = px*4 + a*2 + b, accumulator px,
//      shift (a - 1, px + b - 1) relative to the item's origin shifted down by py rows
__host__ __device__ constexpr int ntaps(int mode, int pl) {
  return mode == CONVT4_SP || mode == CONVT4_SPH ? 4
         : mode == CONV3_S1 || mode == CONV3_ROWS ? 9
         : mode == CONVT4_S2   ? 16
         : mode == CONVT4_HALF ? 8
                               : (pl == 0 ? 1 : pl == 3 ? 4 : 2);
}
__host__ __device__ constexpr int tap_dy(int mode, int pl, int t) {
  return mode == CONVT4_SP || mode == CONVT4_SPH ? t >> 1
         : mode == CONV3_S1 || mode == CONV3_ROWS ? t / 3 - 1
         : mode == CONVT4_S2   ? (t / 4 >> 1) + ((t >> 1) & 1) - 1
         : mode == CONVT4_HALF ? ((t >> 1) & 1) - 1
         : pl == 2             ? (t == 0 ? -1 : 0)
         : pl == 3             ? (t < 2 ? -1 : 0)
                               : 0;
}
__host__ __device__ constexpr int tap_dx(int mode, int pl, int t) {
  return mode == CONVT4_SP || mode == CONVT4_SPH ? t & 1
         : mode == CONV3_S1 || mode == CONV3_ROWS ? t % 3 - 1
         : mode == CONVT4_S2   ? ((t / 4) & 1) + (t & 1) - 1
         : mode == CONVT4_HALF ? (t >> 2) + (t & 1) - 1
         : pl == 1             ? (t == 0 ? -1 : 0)
         : pl == 3             ? ((t & 1) == 0 ? -1 : 0)
                               : 0;
}
__host__ __device__ constexpr int tap_acc(int mode, int t) {
  return mode == CONVT4_S2 || mode == CONVT4_HALF ? t / 4 : 0;
}
// first tap touching its accumulator (in chunk 0 = plane 0, channel group 0)
__host__ __device__ constexpr bool tap_first(int mode, int t) {
  return mode == CONVT4_S2 || mode == CONVT4_HALF ? (t & 3) == 0 : t == 0;
}
// accumulators per source
__host__ __device__ constexpr int nacc_src(int mode) {
  return mode == CONVT4_S2 || mode == CONV3_S1P || mode == CONV_STEMT || mode == CONVT4_SP ? 4
         : mode == CONVT4_HALF || mode == CONVT4_SPH ? 2 : 1;
}
// minimum shift over a plane's taps, as a*L + b
__host__ __device__ constexpr int plane_lo_a(int mode, int pl) {
  return mode == CONV3_S2 ? (pl >= 2 ? -1 : 0) : mode == CONV3_S1P ? -(pl >> 1) : mode == CONV_STEMT || mode == CONVT4_SP || mode == CONVT4_SPH ? 0 : -1;
}
__host__ __device__ constexpr int plane_lo_b(int mode, int pl) {
  return mode == CONV3_S2 ? ((pl & 1) ? -1 : 0) : mode == CONV3_S1P ? -(pl & 1) : mode == CONV_STEMT || mode == CONVT4_SP || mode == CONVT4_SPH ? 0 : -1;
}
__host__ __device__ constexpr int n_planes_of(int mode) { return mode == CONV3_S2 || mode == CONV3_S1P ? 4 : 1; }

// ---- phase-plane stride-1 conv (CONV3_S1P) ------------------------------------------------
// Input: the 4 phase planes (qy, qx) of a 2Hp x 2Wp tensor (PP, planes.cuh); output: the
// 2x2 pixel block (2y+py, 2x+px) of every half-resolution position q = y*L + x, phase
// p = py*2 + px in accumulator p.  Output phase py reads full-resolution row 2y+py+dy =
// 2(y+sy)+qy, i.e. input plane parity qy = (py+dy)&1 at half-resolution shift
// sy = floor((py+dy)/2).  Per input parity the 3 taps x 2 output parities collapse onto 2
// shifts:  qy = 0: sy = 0 -> py in {0,1}, sy = +1 -> py = 1;
//          qy = 1: sy = -1 -> py = 0,     sy = 0  -> py in {0,1}.
// So one A read per (input plane, shift) — 4 per plane, 16 per K chunk for 4 output pixels —
// feeds the stacked B tiles of every output phase using that shift (9 taps x 4 phases = 36
// products from 16 A reads, against 36 A reads for four stride-1 M-tiles).  The phases of
// a shift group form the accumulator run p0 .. p0+n-1 (zero B tile for a phase in the run
// that does not use the shift: 40 tiles per 36 products).  Group 0 of plane 0 is shift (0,0)
// over all four phases (it initialises the accumulators in chunk 0).
__host__ __device__ constexpr int s1p_shift(int q, int g) { return q == 0 ? (g == 0 ? 0 : 1) : (g == 0 ? -1 : 0); }
__host__ __device__ constexpr int s1p_pmin(int q, int g) { return q == 0 ? (g == 0 ? 0 : 1) : 0; }
__host__ __device__ constexpr int s1p_pmax(int q, int g) { return q == 0 ? 1 : (g == 0 ? 0 : 1); }
__host__ __device__ constexpr int s1p_dy(int pl, int gi) { return s1p_shift(pl >> 1, gi >> 1); }
__host__ __device__ constexpr int s1p_dx(int pl, int gi) { return s1p_shift(pl & 1, gi & 1); }
__host__ __device__ constexpr int s1p_p0(int pl, int gi) {
  return s1p_pmin(pl >> 1, gi >> 1) * 2 + s1p_pmin(pl & 1, gi & 1);
}
__host__ __device__ constexpr int s1p_n(int pl, int gi) {
  return s1p_pmax(pl >> 1, gi >> 1) * 2 + s1p_pmax(pl & 1, gi & 1) - s1p_p0(pl, gi) + 1;
}
// does accumulator (phase) acc of group gi use the group's shift?
__host__ __device__ constexpr bool s1p_uses(int pl, int gi, int acc) {
  return (acc >> 1) >= s1p_pmin(pl >> 1, gi >> 1) && (acc >> 1) <= s1p_pmax(pl >> 1, gi >> 1) &&
         (acc & 1) >= s1p_pmin(pl & 1, gi & 1) && (acc & 1) <= s1p_pmax(pl & 1, gi & 1);
}
__host__ __device__ constexpr int s1p_slot0(int pl, int gi) {
  int s = 0;
  for (int i = 0; i < gi; ++i) s += s1p_n(pl, i);
  return s;
}

// ---- shift groups of the transposed conv (fp32 concat scheme) ------------------------
// The 16 (phase, tap) products of a ConvT item read only 9 distinct A shifts: shift
// (dy, dx) is used by every phase (py, px) with dy - py, dx - px in {-1, 0} (tap
// a = dy - py + 1, b = dx - px + 1).  One MMA per shift covers a contiguous run of
// accumulators [p0, p0 + n) — their TMEM blocks are adjacent — with the B tiles of those
// phases stacked along N (a zero tile for a phase in the run that does not use the shift):
// 9 A reads per source and chunk instead of 16 (HALF: 6 instead of 8).  Group 0 touches
// every accumulator (it initialises them in chunk 0).
//   T    (acc = py*2+px): (0,0)x4 (-1,0)x2@0 (1,0)x2@2 (0,-1)x3@0 (0,1)x3@1 and the 4 corners
//   HALF (acc = px, shifts relative to the item origin): (0,0)x2 (-1,0)x2 (0,-1) (0,1)
//        (-1,-1) (-1,1)
__host__ __device__ constexpr bool grouped_t(int mode, int npm) {
  return (mode == CONVT4_S2 || mode == CONVT4_HALF) && npm == kNpmConcat;
}
__host__ __device__ constexpr int ngroups(int mode) { return mode == CONVT4_S2 ? 9 : 6; }
__host__ __device__ constexpr int grp_dy(int mode, int g) {
  return mode == CONVT4_S2 ? (g == 1 || g == 5 || g == 6 ? -1 : g == 2 || g == 7 || g == 8 ? 1 : 0)
                           : (g == 1 || g == 4 || g == 5 ? -1 : 0);
}
__host__ __device__ constexpr int grp_dx(int mode, int g) {
  return mode == CONVT4_S2 ? (g == 3 || g == 5 || g == 7 ? -1 : g == 4 || g == 6 || g == 8 ? 1 : 0)
                           : (g == 2 || g == 4 ? -1 : g == 3 || g == 5 ? 1 : 0);
}
__host__ __device__ constexpr int grp_p0(int mode, int g) {
  return mode == CONVT4_S2 ? (g == 2 ? 2 : g == 4 ? 1 : g >= 5 ? g - 5 : 0) : (g == 3 || g == 5 ? 1 : 0);
}
__host__ __device__ constexpr int grp_n(int mode, int g) {
  return mode == CONVT4_S2 ? (g == 0 ? 4 : g <= 2 ? 2 : g <= 4 ? 3 : 1) : (g <= 1 ? 2 : 1);
}
__host__ __device__ constexpr int grp_slot0(int mode, int g) {  // first B tile of group g
  int s = 0;
  for (int i = 0; i < g; ++i) s += grp_n(mode, i);
  return s;
}
// B tiles per source and chunk: T 18 (16 + 2 zero tiles), HALF 8
__host__ __device__ constexpr int grp_slots(int mode) { return grp_slot0(mode, ngroups(mode)); }

// ---- row-band 3x3 conv (CONV3_ROWS: stride 1, plane width a multiple of 128) -----------
// An item is T = G output rows x 128 columns; M-tile = one row segment.  The item's input
// rows y0-1 .. y0+T are staged one per kRowsSL positions (columns x0-1 .. x0+128, the
// plane's pad column / margins supplying the zero borders), so the A tile of input row i
// and column shift dx is the staged range starting at i*kRowsSL + dx + 1.  One A read
// serves the three dy taps of the output rows i+1, i, i-1: B = the dx group's three tap
// blocks [W(dy=-1) | W(0) | W(+1)] stacked along N, and the accumulator of output row j
// sits at TMEM column (T-1-j)*AW, so block b of the MMA for input row i (output row
// i-b) lands on its row's accumulator (a window sliding one block per input row).
// 3 A reads per input row and K chunk instead of 9 per output row.
constexpr int kRowsSL = 130;

// ---- PTX helpers -----------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// 256-bit global store (sm_100): 8 floats at a 32-byte aligned address
__device__ __forceinline__ void st_global_v8(float* dst, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Issue from one lane of a converged warp: all lanes run the loop, `leader` issues.
__device__ __forceinline__ void tc_mma(bool leader, uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if (leader)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit(bool leader, uint32_t bar) {
  if (leader)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}"
      : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical ((8,m),(T,2)) layout):
// core matrix = 8 rows x 16 B contiguous; SBO = byte stride between 8-row groups,
// LBO = byte stride between the two 8-element K halves.  version = 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// kind::f16 instruction descriptor: A/B bf16, D f32, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// All MMAs of one staged chunk (plane PL).  Descriptors advance in 16-byte units
// (one position of one 8-channel group = 16 B).
// All MMAs of one staged chunk (plane PL), fully unrolled over sources, taps and the G
// M-tiles of the item (G is a template parameter): ~2-3 uniform ops per tcgen05.mma.
// (A runtime tap/tile loop spent ~55 uniform instructions per tap, ~110 cycles per MMA;
// the unrolled stream is a few hundred instructions per chunk and stays in the I-cache.)
template <int N, int MODE, int PL, bool DUAL, int NPM, int G>
__device__ __forceinline__ void issue_chunk(bool leader, uint64_t a0, uint64_t b0, uint32_t dslot,
                                            int L, bool first_chunk, uint32_t src_units,
                                            uint32_t lo_units) {
  constexpr int NT = ntaps(MODE, PL);
  constexpr int NACC_SRC = nacc_src(MODE);
  constexpr int NACC = (DUAL ? 2 : 1) * NACC_SRC;
  constexpr int AW = NPM == kNpmConcat ? 2 * N : N;
  constexpr uint32_t TAP_UNITS = (NPM == kNpmBf16 ? 32u * N : 64u * N) / 16u;
  constexpr uint32_t BLO_UNITS = 32u * N / 16u;
  constexpr uint32_t IDESC_N = idesc_bf16(N);
  constexpr uint32_t IDESC_W = idesc_bf16(AW);
  if constexpr (MODE == CONV3_ROWS) {
    // b0 carries LBO = 3 blocks of AW rows (one dx group = [kgrp 2][block 3][AW rows][16 B])
    constexpr int T = G;
    constexpr uint32_t GRP_UNITS = 6u * AW;
#pragma unroll
    for (int i = 0; i < T + 2; ++i) {
      const int b_lo = i - T + 1 > 0 ? i - T + 1 : 0, b_hi = i < 2 ? i : 2;
      const int nb = b_hi - b_lo + 1;
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const uint64_t ad = a0 + (uint32_t)(i * L + dx);
        const uint64_t bd = b0 + (uint32_t)dx * GRP_UNITS + (uint32_t)(b_lo * AW);
        const uint32_t dcol = dslot + (uint32_t)((T - 1 - i + b_lo) * AW);
        if (first_chunk && dx == 0 && b_lo == 0) {
          // block 0 starts output row i's accumulator; the others continue theirs
          tc_mma(leader, dcol, ad, bd, idesc_bf16(AW), 0u);
          if (nb > 1) tc_mma(leader, dcol + AW, ad, bd + AW, idesc_bf16((nb - 1) * AW), 1u);
        } else {
          tc_mma(leader, dcol, ad, bd, idesc_bf16(nb * AW), 1u);
        }
        if (NPM == kNpmConcat) tc_mma(leader, dcol, ad + lo_units, bd, idesc_bf16(nb * AW), 1u);  // A_lo
      }
    }
  } else {
  const int lo = plane_lo_a(MODE, PL) * L + plane_lo_b(MODE, PL);
  if constexpr (MODE == CONVT4_SP || MODE == CONVT4_SPH) {
    // shifted-phase ConvT: output phase (py, px) of accumulator row m is the half-resolution
    // position q0 + m + (1-py)*L + (1-px), so its 2x2 sub-kernel tap (a, b) reads input
    // position q0 + m + a*L + b for every phase: four A windows per source, each one MMA
    // pair over the four stacked phase tiles [B_hi | B_lo] (N = 4 * AW)
    // (SPH: the item's two px phases of one output-row parity, the same four windows)
    constexpr int NPH = NACC_SRC;
    constexpr uint32_t idesc = idesc_bf16(NPH * AW);
#pragma unroll
    for (int s = 0; s < (DUAL ? 2 : 1); ++s) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint64_t ad0 = a0 + (uint32_t)s * src_units + (uint32_t)((w >> 1) * L + (w & 1));
        const uint64_t bd = b0 + (uint32_t)((s * 4 + w) * NPH) * TAP_UNITS + ((uint64_t)((NPH - 1) * AW) << 16);
        const uint32_t accum0 = (first_chunk && w == 0) ? 0u : 1u;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint64_t ad = ad0 + (uint32_t)(g * 128);
          const uint32_t dcol = dslot + (uint32_t)((g * NACC + s * NACC_SRC) * AW);
          tc_mma(leader, dcol, ad, bd, idesc, accum0);
          if (NPM != kNpmBf16) tc_mma(leader, dcol, ad + lo_units, bd, idesc, 1u);
          // 3-MMA scheme (no concat): [pass][kgrp][phase][N] blocks, + A_hi x B_lo
          if (NPM == kNpm3) tc_mma(leader, dcol, ad, bd + (uint32_t)(2 * NPH * N), idesc, 1u);
        }
      }
    }
    (void)lo;
    return;
  }
  if constexpr (MODE == CONV_STEMT) {
    // one chunk = one frame's 4x4 window per position: A_hi (and A_lo) x the 4 stacked
    // phase tiles [B_hi | B_lo] (K-half stride = 4 tiles of AW rows)
    constexpr uint32_t idesc = idesc_bf16(4 * AW);
    const uint64_t bd = b0 + ((uint64_t)(3 * AW) << 16);
    const uint32_t accum0 = first_chunk ? 0u : 1u;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint64_t ad = a0 + (uint32_t)(g * 128);
      const uint32_t dcol = dslot + (uint32_t)(g * NACC * AW);
      tc_mma(leader, dcol, ad, bd, idesc, accum0);
      if (NPM != kNpmBf16) tc_mma(leader, dcol, ad + lo_units, bd, idesc, 1u);
    }
    (void)lo;
    return;
  }
  if constexpr (MODE == CONV3_S1P) {
    // one MMA (pair) per shift group over the stacked phase tiles of input plane PL
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const int n = s1p_n(PL, gi);
      const uint32_t idesc = idesc_bf16(n * AW);
      const uint64_t ad0 = a0 + (uint32_t)(s1p_dy(PL, gi) * L + s1p_dx(PL, gi) - lo);
      const uint64_t bd = b0 + (uint32_t)s1p_slot0(PL, gi) * TAP_UNITS + ((uint64_t)((n - 1) * AW) << 16);
      const uint32_t accum0 = (first_chunk && gi == 0) ? 0u : 1u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint64_t ad = ad0 + (uint32_t)(g * 128);
        const uint32_t dcol = dslot + (uint32_t)((g * NACC + s1p_p0(PL, gi)) * AW);
        tc_mma(leader, dcol, ad, bd, idesc, accum0);                                // A_hi x tiles
        if (NPM != kNpmBf16) tc_mma(leader, dcol, ad + lo_units, bd, idesc, 1u);  // A_lo x tiles
        if (NPM == kNpm3) tc_mma(leader, dcol, ad, bd + (uint32_t)(2 * n * N), idesc, 1u);  // A_hi x B_lo
      }
    }
    return;
  }
  if constexpr (grouped_t(MODE, NPM)) {
    // one MMA pair per shift group: A_hi x [tiles] + A_lo x [tiles], each tile [B_hi | B_lo]
    // (the A_lo x B_lo product is kept: it costs nothing extra at this width)
    constexpr int NG = ngroups(MODE), NS = grp_slots(MODE);
#pragma unroll
    for (int s = 0; s < (DUAL ? 2 : 1); ++s) {
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        const int n = grp_n(MODE, gi);
        const uint32_t idesc = idesc_bf16(n * AW);
        const uint64_t ad0 = a0 + (uint32_t)s * src_units + (uint32_t)(grp_dy(MODE, gi) * L + grp_dx(MODE, gi) - lo);
        // B descriptor of the stacked tiles: K-half stride (LBO) = n * AW rows of 16 B
        const uint64_t bd = b0 + (uint32_t)(s * NS + grp_slot0(MODE, gi)) * TAP_UNITS +
                            ((uint64_t)((n - 1) * AW) << 16);
        const uint32_t accum0 = (first_chunk && gi == 0) ? 0u : 1u;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint64_t ad = ad0 + (uint32_t)(g * 128);
          const uint32_t dcol = dslot + (uint32_t)((g * NACC + s * NACC_SRC + grp_p0(MODE, gi)) * AW);
          tc_mma(leader, dcol, ad, bd, idesc, accum0);      // A_hi x [B_hi | B_lo] (n tiles)
          tc_mma(leader, dcol, ad + lo_units, bd, idesc, 1u);  // A_lo x [B_hi | B_lo]
        }
      }
    }
    return;
  }
#pragma unroll
  for (int s = 0; s < (DUAL ? 2 : 1); ++s) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int acc = s * NACC_SRC + tap_acc(MODE, t);
      const uint64_t ad0 =
          a0 + (uint32_t)s * src_units + (uint32_t)(tap_dy(MODE, PL, t) * L + tap_dx(MODE, PL, t) - lo);
      const uint64_t bd = b0 + (uint32_t)(s * NT + t) * TAP_UNITS;
      const uint32_t accum0 = (first_chunk && tap_first(MODE, t)) ? 0u : 1u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint64_t ad = ad0 + (uint32_t)(g * 128);
        const uint32_t dcol = dslot + (uint32_t)((g * NACC + acc) * AW);
        if (NPM == kNpmBf16) {
          tc_mma(leader, dcol, ad, bd, IDESC_N, accum0);
        } else if (NPM == kNpmConcat) {
          tc_mma(leader, dcol, ad, bd, IDESC_W, accum0);          // A_hi x [B_hi | B_lo]
          tc_mma(leader, dcol, ad + lo_units, bd, IDESC_N, 1u);   // A_lo x B_hi
        } else {
          tc_mma(leader, dcol, ad, bd, IDESC_N, accum0);          // hi*hi
          tc_mma(leader, dcol, ad + lo_units, bd, IDESC_N, 1u);   // lo*hi
          tc_mma(leader, dcol, ad, bd + BLO_UNITS, IDESC_N, 1u);  // hi*lo
        }
      }
    }
  }
  }
}

// ---- the kernel ----------------------------------------------------------------------
// Channel sums of one warp: v[c] of the 32 lanes summed per channel, written to out[c].
// Reduce-scatter butterfly: at offset o = 16, 8, ... each lane sends the half of its values
// it does not keep and adds the partner's half of the kept ones (N/2 + N/4 + ... shuffles
// instead of 5 per channel); after the halving levels lane l holds channel(s)
//   N = 64: 2l, 2l+1;  N = 32: l;  N = 16: l/2 (the last offset 1 is a plain add, a + b ==
// b + a in IEEE arithmetic, so both lanes of a pair hold identical bits).  The addition
// order per channel is fixed by the lane numbering: deterministic and batch-invariant.
template <int N>
__device__ __forceinline__ void gap_lane_reduce(float (&v)[N], int lane, float* out) {
  constexpr int LV = N >= 32 ? 5 : (N == 16 ? 4 : (N == 8 ? 3 : 0));
  static_assert(LV > 0, "gap_lane_reduce: N in {8, 16, 32, 64}");
#pragma unroll
  for (int lv = 0; lv < LV; ++lv) {
    const int o = 16 >> lv;
    const int n = N >> (lv + 1);  // values kept after this level
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float send = up ? v[i] : v[i + n];
      const float keep = up ? v[i + n] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  if constexpr (N >= 32) {
    constexpr int K = N / 32;  // values per lane
#pragma unroll
    for (int i = 0; i < K; ++i) out[lane * K + i] = v[i];
  } else {
    // remaining offsets: plain pairwise adds (all lanes of a group end with identical bits)
#pragma unroll
    for (int o = 16 >> LV; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    if ((lane & ((32 / N) - 1)) == 0) out[lane / (32 / N)] = v[0];
  }
}

// floor division for possibly negative positions
__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

template <int N, int MODE, bool DUAL, int NPM, int G, int CPS, int STEM = 0>
__global__ void __launch_bounds__(threads_of(MODE, STEM), 1) tc_conv_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NSRC = DUAL ? 2 : 1;
  constexpr int NACC_SRC = nacc_src(MODE);
  constexpr int NACC = NSRC * NACC_SRC;
  constexpr int NPLANES = n_planes_of(MODE);
  constexpr int NPASS_A = NPM == kNpmBf16 ? 1 : 2;
  constexpr int AW = NPM == kNpmConcat ? 2 * N : N;  // TMEM columns per accumulator
  constexpr int EPW = STEM ? kEpiWarps : epi_warps(MODE);  // epilogue warps
  const TcLayerDesc& d = p.d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cgroups = d.cin / 16;
  const int n_chunks = NPLANES * cgroups;

  uint8_t* a_base = smem;
  uint8_t* b_base = smem + (size_t)p.stages * p.a_stage_bytes;
  const size_t b_region = p.resident ? (size_t)(p.w_total + 127) / 128 * 128
                                     : (size_t)p.stages * p.b_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + b_region);
  uint64_t* full = bars;
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint64_t* tempty = tfull + p.slots;
  uint64_t* wbar = tempty + p.slots;  // resident weights landed
  uint64_t* xfull = wbar + 1;         // STEM: frame rows of x ring stage landed
  uint64_t* xempty = xfull + 4;       // STEM: stem warps done with x ring stage (<= 4 stages)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(xempty + 2);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [EPW][N]
  // STEM: x ring [2][F][rows][W] (offset from the dynamic smem base: the compiler keeps
  // the shared address space, i.e. LDS rather than generic loads)
  float* xring = reinterpret_cast<float*>(
      smem + ((size_t)(reinterpret_cast<uint8_t*>(red + kEpiWarpsMax * 64) - smem) + 127) / 128 * 128);

  if (threadIdx.x == 0) {
    trace_at(p.trace, 4, 0);
    trace_cta(p.trace, 0);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full[s]), STEM ? stem_threads(MODE, STEM) : 1);  // STEM: every stem thread arrives
      mbar_init(smem_u32(&empty[s]), 1);
    }
    if (STEM > 0) {
      for (int s = 0; s < 4; ++s) {
        mbar_init(smem_u32(&xfull[s]), 1);
        mbar_init(smem_u32(&xempty[s]), stem_threads(MODE, STEM));
      }
    }
    for (int s = 0; s < p.slots; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), EPW * 32);
    }
    mbar_init(smem_u32(wbar), 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t src_bytes = (uint32_t)NPASS_A * 2 * p.P_max * 16;
  // single-wave persistent grid: let the next kernel's CTAs take SMs as ours retire
  if (p.early_trigger) grid_dep_launch();

  constexpr int NPW = STEM == 0 ? 1 + kProd2 : 1;  // producer warps
  const bool two_prod = NPW == 2 && p.prod2 != 0;
  if (warp == kProdWarp || (two_prod && warp == kEpiWarp0 + EPW)) {
    const uint32_t pw = warp == kProdWarp ? 0u : 1u;  // takes ring-stage steps k with k % NPW == pw
    // ===================== producer: cp.async.bulk of A ranges + packed weights =========
    // The whole warp runs the loop; lane 0 posts the stage's byte count, then lane l
    // issues copy l (source, pass, 8-channel group) — the per-copy address arithmetic runs
    // in parallel instead of ~130 serial cycles per copy on one thread.
    constexpr int NCOPY = NSRC * NPASS_A * 2;
    const int cs = lane / (NPASS_A * 2), cpass = (lane >> 1) % NPASS_A, ccg8 = lane & 1;
    if (lane == 0 && p.resident && pw == 0) {
      mbar_arrive_expect_tx(smem_u32(wbar), p.w_total);
      // HALF: this CTA's py block only (even grid: item parity == blockIdx.x parity)
      bulk_g2s(smem_u32(b_base),
               reinterpret_cast<const uint8_t*>(d.w) +
                   (MODE == CONVT4_HALF || MODE == CONVT4_SPH ? (blockIdx.x & 1) * d.half_bytes : 0),
               p.w_total, smem_u32(wbar));
    }
    grid_dep_wait();  // weights are static; activations come from the previous kernel
    if constexpr (STEM == kGateIn) {
      // gate-in: per item and 16-channel chunk, the staged rows of the input's chunk plane
      // (chunk-planar fp32, one contiguous range) and the skip's staged positions (one range
      // per (pass, cg8) block) into the 2-stage x ring
      constexpr int NP = NPASS_A;
      const bool has_skip = p.gskip.base != nullptr;
      const int L = p.L, W = p.W, H = p.H, C = p.C;
      const int P = G * 128 + 2 * L + 2;
      int xs = 0;
      uint32_t xph = 0;
      for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        int b, it;
        item_coords(item, p, b, it);
        const int qa = it * G * 128 - L - 1;
        const int y_lo = max(floordiv(qa, L), 0);
        const int y_hi = min(floordiv(qa + P - 1, L), H - 1);
        for (int c = 0; c < C / 16; ++c) {
          mbar_wait(smem_u32(&xempty[xs]), xph ^ 1);
          if (lane == 0) {
            const uint32_t xb = (uint32_t)max(y_hi - y_lo + 1, 0) * W * 64;
            const uint32_t sb = has_skip ? (uint32_t)NP * 2 * P * 16 : 0u;
            const uint32_t bar = smem_u32(&xfull[xs]);
            mbar_arrive_expect_tx(bar, xb + sb);
            uint8_t* dst = reinterpret_cast<uint8_t*>(xring) + (size_t)xs * p.stem_xstage;
            if (xb)
              bulk_g2s(smem_u32(dst), p.gx + (((size_t)b * (C / 16) + c) * H * W + (size_t)y_lo * W) * 16, xb, bar);
            if (has_skip) {
              const uint16_t* skb = p.gskip.base + (int64_t)b * p.gskip.img_stride;
              for (int blk = 0; blk < NP * 2; ++blk)
                bulk_g2s(smem_u32(dst + p.gx_skip_off + (size_t)blk * P * 16),
                         skb + (p.gskip.block_index(c, blk >> 1, blk & 1) + qa + p.gskip.off) * 8, (uint32_t)P * 16,
                         bar);
            }
          }
          __syncwarp();
          if (++xs == p.gx_nst) {
            xs = 0;
            xph ^= 1u;
          }
        }
      }
    } else if constexpr (STEM > 0) {
      // frame rows of each item's staged positions (+1 row each side), one copy per frame
      // into the 2-stage x ring; rows outside the image are never read (the stem masks them)
      int xs = 0;
      uint32_t xph = 0;
      for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        int b, it;
        item_coords(item, p, b, it);
        // (STEMT: the item's half-resolution rows y.. -> frame rows 2y-1 ..)
        const int xr0 = MODE == CONV_STEMT ? 2 * (int)__umulhi((uint32_t)(it * G * 128), p.L_mul) - 1
                                           : floordiv(it * G * 128 - p.L - 1, p.L) - 1;
        const int r_lo = max(xr0, 0), r_hi = min(xr0 + p.stem_xrows - 1, p.H - 1);
        mbar_wait(smem_u32(&xempty[xs]), xph ^ 1);
        if (lane == 0) {
          const uint32_t rb = (uint32_t)(r_hi - r_lo + 1) * p.W * 4;
          mbar_arrive_expect_tx(smem_u32(&xfull[xs]), rb * p.sF);
          for (int ci = 0; ci < p.sF; ++ci)
            bulk_g2s(smem_u32(xring + ((size_t)(xs * p.sF + ci) * p.stem_xrows + (r_lo - xr0)) * p.W),
                     p.sx + (int64_t)b * p.sxb + (int64_t)ci * p.sxc + (int64_t)r_lo * p.W, rb,
                     smem_u32(&xfull[xs]));
        }
        __syncwarp();
        if (++xs == 2) {
          xs = 0;
          xph ^= 1u;
        }
      }
    } else {
    const PlBuf& S = p.src[lane < NCOPY ? cs : 0];
    uint32_t k = 0;
    int pstage = 0;
    uint32_t pphase = 0;
    for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
      int b, it;
      item_coords(item, p, b, it);
      // HALF: items (tile, py) interleaved; the tile origin moves down py rows
      // (SP: tile origins start one row and column above the image: phase (0,0) at q0 + L + 1)
      const int q0 = MODE == CONVT4_HALF ? (it >> 1) * p.G * 128 + (it & 1) * p.L
                     : MODE == CONVT4_SP ? it * p.G * 128 - p.L - 1
                     : MODE == CONVT4_SPH ? (it >> 1) * p.G * 128 - p.L - 1
                                          : it * p.G * 128;
      const uint16_t* img = S.base + (int64_t)b * S.img_stride;
      if constexpr (MODE == CONV3_ROWS) {
        // per staged row and (pass, cg8) block one copy of kRowsSL positions (weights resident)
        const int tpr = p.Wp / 128, band = it / tpr;
        const int y0 = band * p.G, x0 = (it - band * tpr) * 128;
        constexpr int NCP = NPASS_A * 2;
        for (int c0 = 0; c0 < n_chunks; c0 += CPS, ++k) {
          const int stage = pstage;
          const uint32_t phase = pphase;
          if (++pstage == p.stages) {
            pstage = 0;
            pphase ^= 1u;
          }
          if (two_prod && (k & 1u) != pw) continue;  // the other producer warp's stage
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          if (lane == 0) mbar_arrive_expect_tx(fb, (uint32_t)(CPS * (p.G + 2) * NCP * kRowsSL * 16));
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < CPS; ++cc) {
            const int cgi = c0 + cc;
            for (int u = lane; u < (p.G + 2) * NCP; u += 32) {
              const int i = u / NCP, blk = u - i * NCP;
              const uint16_t* src =
                  img + (S.block_index(cgi, blk >> 1, blk & 1) + (int64_t)(y0 - 1 + i) * p.L + x0 - 1 + S.off) * 8;
              bulk_g2s(smem_u32(a_base + (size_t)stage * p.a_stage_bytes + (size_t)cc * p.chunk_a_bytes +
                                (size_t)blk * p.P_max * 16 + (size_t)i * kRowsSL * 16),
                       src, (uint32_t)(kRowsSL * 16), fb);
            }
          }
        }
      } else {
      for (int c0 = 0; c0 < n_chunks; c0 += CPS, ++k) {  // one ring stage = cps chunks
        const int stage = pstage;
        const uint32_t phase = pphase;
        if (++pstage == p.stages) {
          pstage = 0;
          pphase ^= 1u;
        }
        if (two_prod && (k & 1u) != pw) continue;  // the other producer warp's stage
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        if (lane == 0) trace_at(p.trace, 0, 2 * k);
        const uint32_t fb = smem_u32(&full[stage]);
        if ((p.dbg & 4) && k >= (uint32_t)p.stages) {
          if (lane == 0) mbar_arrive(fb);
          continue;
        }
        uint32_t tx = 0;
#pragma unroll
        for (int cc = 0; cc < CPS; ++cc) {
          const int c = c0 + cc;
          const PlaneTaps& pt = d.planes[c / cgroups];
          tx += (uint32_t)NCOPY * (uint32_t)(p.G * 128 + pt.hi - pt.lo) * 16 +
                (p.resident ? 0u : (uint32_t)(d.chunk_off[c + 1] - d.chunk_off[c]));
        }
        if (lane == 0) mbar_arrive_expect_tx(fb, tx);
        __syncwarp();  // byte count posted before any copy can complete
#pragma unroll
        for (int cc = 0; cc < CPS; ++cc) {
          const int c = c0 + cc;
          const int pl = c / cgroups, cgi = c - pl * cgroups;
          const PlaneTaps& pt = d.planes[pl];
          const uint32_t a_bytes = (uint32_t)(p.G * 128 + pt.hi - pt.lo) * 16;
          if (lane == NCOPY && !p.resident)
            bulk_g2s(smem_u32(b_base + (size_t)stage * p.b_stage_bytes + (size_t)cc * p.chunk_b_bytes),
                     reinterpret_cast<const uint8_t*>(d.w) +
                         (MODE == CONVT4_HALF || MODE == CONVT4_SPH ? (it & 1) * d.half_bytes : 0) +
                         d.chunk_off[c],
                     (uint32_t)(d.chunk_off[c + 1] - d.chunk_off[c]), fb);
          if (lane < NCOPY) {
            const uint16_t* src = img + (int64_t)(NPLANES == 4 ? pl : 0) * S.plane_stride +
                                  (S.block_index(cgi, cpass, ccg8) + q0 + pt.lo + S.off) * 8;
            bulk_g2s(smem_u32(a_base + (size_t)stage * p.a_stage_bytes + (size_t)cc * p.chunk_a_bytes +
                              (size_t)cs * src_bytes + (size_t)(cpass * 2 + ccg8) * p.P_max * 16),
                     src, a_bytes, fb);
          }
        }
        if (lane == 0) trace_at(p.trace, 0, 2 * k + 1);
      }
      }
    }
    }  // !STEM
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer: whole warp runs the loop, one lane issues ========
    const bool leader = elect_one();
    const uint32_t lboA = (uint32_t)p.P_max * 16;
    const uint32_t lboB = (uint32_t)AW * 16 * (MODE == CONV3_ROWS ? 3 : 1);
    const int a_rs = MODE == CONV3_ROWS ? kRowsSL : p.L;  // ROWS: staged row stride
    const uint32_t src_units = src_bytes >> 4;
    const uint32_t lo_units = (2 * lboA) >> 4;  // A_lo planes follow the A_hi planes
    uint32_t k = 0, ic = 0;
    if (p.resident) {
      mbar_wait(smem_u32(wbar), 0);
      __syncwarp();
    }
    int mstage = 0, slot = 0;
    uint32_t mphase = 0, sphase = 0;
    for (int item = blockIdx.x; item < p.total_items; item += gridDim.x, ++ic) {
      if (ic > 0 && ++slot == p.slots) {
        slot = 0;
        sphase ^= 1u;
      }
      mbar_wait(smem_u32(&tempty[slot]), sphase ^ 1);
      __syncwarp();
      tc_fence_after();
      if (leader) trace_at(p.trace, 2, ic);
      const uint32_t dslot = tmem_base + (uint32_t)slot * p.slot_cols;
      for (int c0 = 0; c0 < n_chunks; c0 += CPS, ++k) {
        // ring position by counters (no integer division between the MMA bursts: the
        // issue runs in lockstep with the tensor pipe, so this code is pipe idle time)
        const int stage = mstage;
        const uint32_t phase = mphase;
        if (++mstage == p.stages) {
          mstage = 0;
          mphase ^= 1u;
        }
        mbar_wait(smem_u32(&full[stage]), phase);  // TMA -> MMA: both async proxy, no fence
        __syncwarp();
        if (leader) trace_at(p.trace, 1, 2 * k);
        if (leader && k == 0) trace_cta_item(p.trace, 31);
#pragma unroll
        for (int cc = 0; cc < CPS; ++cc) {  // CPS chunks per barrier round trip
          const int c = c0 + cc;
          const uint64_t a0 = smem_desc(
              smem_u32(a_base + (size_t)stage * p.a_stage_bytes + (size_t)cc * p.chunk_a_bytes), lboA, 128);
          // (HALF: the resident block / the staged chunk is already the item's py block)
          const uint64_t b0 = smem_desc(
              smem_u32(b_base + (p.resident ? (size_t)d.chunk_off[c]
                                            : (size_t)stage * p.b_stage_bytes + (size_t)cc * p.chunk_b_bytes)),
              lboB, 128);
          if constexpr (MODE == CONV3_S2 || MODE == CONV3_S1P) {
            switch (c / cgroups) {
              case 0: issue_chunk<N, MODE, 0, DUAL, NPM, G>(leader, a0, b0, dslot, p.L, c == 0, src_units, lo_units); break;
              case 1: issue_chunk<N, MODE, 1, DUAL, NPM, G>(leader, a0, b0, dslot, p.L, c == 0, src_units, lo_units); break;
              case 2: issue_chunk<N, MODE, 2, DUAL, NPM, G>(leader, a0, b0, dslot, p.L, c == 0, src_units, lo_units); break;
              default: issue_chunk<N, MODE, 3, DUAL, NPM, G>(leader, a0, b0, dslot, p.L, c == 0, src_units, lo_units); break;
            }
          } else {
            issue_chunk<N, MODE, 0, DUAL, NPM, G>(leader, a0, b0, dslot, a_rs, c == 0, src_units, lo_units);
          }
        }
        __syncwarp();
        tc_commit(leader, smem_u32(&empty[stage]));
        if (leader) trace_at(p.trace, 1, 2 * k + 1);
      }
      tc_commit(leader, smem_u32(&tfull[slot]));
    }
    __syncwarp();
  } else if (warp < kEpiWarp0 + EPW) {
    // ===================== epilogue warps 2..9 ==========================================
    // Two warps per TMEM lane quarter; the (tile, phase, 16-channel) units of an item
    // alternate between them so each SM sub-partition has two independent epilogue
    // streams to interleave (one warp alone is latency-bound on the LDTM -> convert ->
    // store chain).
    constexpr int NJ = N / 16;
    const int ew = warp & 3;                               // TMEM lane quarter of this warp
    constexpr int NH = EPW / 4;                            // warps per TMEM lane quarter
    const int half = (warp - kEpiWarp0) / 4;               // which units of the item (u % NH)
    const int et = threadIdx.x - kEpiWarp0 * 32;
    grid_dep_wait();  // outputs may still be read by the previous kernel
    uint32_t ic = 0;
    for (int item = blockIdx.x; item < p.total_items; item += gridDim.x, ++ic) {
      const int slot = ic % p.slots;
      const uint32_t sphase = (ic / p.slots) & 1;
      int b, it;
      item_coords(item, p, b, it);
      const int q0 = (MODE == CONVT4_HALF || MODE == CONVT4_SPH ? it >> 1 : it) * p.G * 128 -
                     (MODE == CONVT4_SP || MODE == CONVT4_SPH ? p.L + 1 : 0);
      const int py = MODE == CONVT4_HALF || MODE == CONVT4_SPH ? (it & 1) : 0;  // output row parity
      int ry0 = 0, rx0 = 0;  // ROWS: the item's first output row / column
      if (MODE == CONV3_ROWS) {
        const int tpr = p.Wp / 128, band = it / tpr;
        ry0 = band * G;
        rx0 = (it - band * tpr) * 128;
      }
      mbar_wait(smem_u32(&tfull[slot]), sphase);
      __syncwarp();
      tc_fence_after();
      if (et == 0) trace_at(p.trace, 3, 2 * ic);
      if (p.dbg & 8) {
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty[slot]));
        continue;
      }
      float gsum[N];
#pragma unroll
      for (int c = 0; c < N; ++c) gsum[c] = 0.f;
      const uint32_t trow = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)slot * p.slot_cols;
      for (int g = 0; g < G; ++g) {
        int y, x;
        if (MODE == CONV3_ROWS) {
          y = ry0 + g;
          x = rx0 + ew * 32 + lane;
        } else {
          const int q = q0 + g * 128 + ew * 32 + lane;
          y = (int)__umulhi((uint32_t)q, p.L_mul);  // q / L (host-checked exact)
          x = q - y * p.L;
        }
        const bool valid = y < p.Hp && x < p.Wp;
        // the output row's pad position: ROWS tiles never cover it, the last lane of the
        // row's last tile clears it
        const bool padpos = MODE == CONV3_ROWS ? (rx0 + 128 == p.Wp && ew == 3 && lane == 31)
                                               : (y < p.Hp && x == p.Wp);
        if (p.out.mode != 0 && ((g * NACC_SRC * NJ) % NH) == half && padpos) {
          // this position is a pad of the output grid: keep the operand plane's pad
          // column zero (planes.cuh border contract)
          if (p.out.mode == 1) {
            pl_zero_pos(p.out.pl, b, 0, y * p.out.pl.L + p.Wp);
          } else if (MODE == CONV3_S1P || MODE == CONV_STEMT) {  // the half-res pad column of all 4 planes
#pragma unroll
            for (int pz = 0; pz < 4; ++pz) pl_zero_pos(p.out.pl, b, pz, y * p.out.pl.L + p.Wp);
          } else {
            pl_zero_pos(p.out.pl, b, (y & 1) * 2, (y >> 1) * p.out.pl.L + p.Wp / 2);
            pl_zero_pos(p.out.pl, b, (y & 1) * 2 + 1, (y >> 1) * p.out.pl.L + p.Wp / 2);
          }
        }
#pragma unroll
        for (int ph = 0; ph < NACC_SRC; ++ph) {
          int oy = y, ox = x;
          bool pvalid = true;  // SP: this phase's row of the tile is an output position
          if constexpr (MODE == CONVT4_SP || MODE == CONVT4_SPH) {
            const int ppy = MODE == CONVT4_SP ? ph >> 1 : py, ppx = MODE == CONVT4_SP ? ph & 1 : ph;
            const int qp = q0 + g * 128 + ew * 32 + lane + (1 - ppy) * p.L + (1 - ppx);
            const int yy = (int)__umulhi((uint32_t)(qp + 2 * p.L), p.L_mul) - 2;  // floor(qp / L)
            const int xx = qp - yy * p.L;
            pvalid = yy >= 0 && yy < p.Hp && xx < p.Wp;
            oy = 2 * yy + ppy;
            ox = 2 * xx + ppx;
          } else if (MODE == CONVT4_S2 || MODE == CONV3_S1P || MODE == CONV_STEMT) {
            oy = 2 * y + (ph >> 1);
            ox = 2 * x + (ph & 1);
          } else if (MODE == CONVT4_HALF) {
            oy = 2 * y + py;
            ox = 2 * x + ph;
          }
#pragma unroll
          for (int j = 0; j < N; j += 16) {
            if ((((g * NACC_SRC + ph) * NJ + j / 16) % NH) != half) continue;  // warp-uniform
            float a0[16], a1[16];
            const int gt = MODE == CONV3_ROWS ? G - 1 - g : g;  // ROWS: row j at column (T-1-j)*AW
            const uint32_t c0 = (uint32_t)((gt * NACC + ph) * AW + j);
            const uint32_t c1 = (uint32_t)((gt * NACC + NACC_SRC + ph) * AW + j);
            auto ld = [&](uint32_t a, float(&v)[16]) {
              if (p.dbg & 2) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
              } else {
                tmem_ld16(a, v);
              }
            };
            ld(trow + c0, a0);
            if (DUAL) ld(trow + c1, a1);
            if (NPM == kNpmConcat) {  // + the hi*lo half of the concatenated accumulator
              float h0[16], h1[16];
              ld(trow + c0 + N, h0);
              if (DUAL) ld(trow + c1 + N, h1);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                a0[i] += h0[i];
                if (DUAL) a1[i] += h1[i];
              }
            } else {
              tmem_wait_ld();
            }
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float t = a0[i] + d.bias0_c[j + i];
              if (p.relu0) t = fmaxf(t, 0.f);
              if (DUAL) t = t + (a1[i] + d.bias1_c[j + i]);
              v[i] = t;
            }
            if (p.out.mode == 0 && MODE == CONV3_S2) {  // measured: slower for the ConvT phases
              // NHWC fp32: the 64-byte pixel rows of a lane quad are transposed in registers
              // (4x4 exchange of 16-byte chunks by shfl_xor 2, then 1), so each store
              // instruction writes 8 whole 64-byte pixel segments instead of 32 scattered
              // 16-byte pieces (half the L2 sector writes, a third of the L1 wavefronts)
              if (valid) {
#pragma unroll
                for (int i = 0; i < 16; ++i) gsum[j + i] += v[i];
              }
              float4 c4[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) c4[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
              const int r = lane & 3;
              auto xchg = [&](float4& keep_or_recv_a, float4& keep_or_recv_b, bool hi, int m) {
                // hi lanes send a and receive into a; lo lanes send b and receive into b
                const float4 x = hi ? keep_or_recv_a : keep_or_recv_b;
                float4 y;
                y.x = __shfl_xor_sync(0xffffffffu, x.x, m);
                y.y = __shfl_xor_sync(0xffffffffu, x.y, m);
                y.z = __shfl_xor_sync(0xffffffffu, x.z, m);
                y.w = __shfl_xor_sync(0xffffffffu, x.w, m);
                if (hi) keep_or_recv_a = y;
                else keep_or_recv_b = y;
              };
              xchg(c4[0], c4[2], (r & 2) != 0, 2);
              xchg(c4[1], c4[3], (r & 2) != 0, 2);
              xchg(c4[0], c4[1], (r & 1) != 0, 1);
              xchg(c4[2], c4[3], (r & 1) != 0, 1);
              // c4[c] = channels j + 4r .. j + 4r + 3 of the pixel of lane (lane & ~3) + c
              if (!(p.dbg & 1)) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const int qc = q0 + g * 128 + ew * 32 + (lane & ~3) + c;
                  const int yc = (int)__umulhi((uint32_t)qc, p.L_mul);
                  const int xc = qc - yc * p.L;
                  if (yc >= p.Hp || xc >= p.Wp) continue;
                  const size_t e = p.out.cp ? (((size_t)b * (N / 16) + j / 16) * p.Ho * p.Wo +
                                               (size_t)yc * p.Wo + xc) * 16 + 4 * r
                                            : (((size_t)b * p.Ho + yc) * p.Wo + xc) * N + j + 4 * r;
                  if (p.out.bf)  // bf16 variant: 4 values as 8 bytes
                    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.out.f32) + e) =
                        make_uint2(pack_bf16x2(c4[c].x, c4[c].y), pack_bf16x2(c4[c].z, c4[c].w));
                  else
                    *reinterpret_cast<float4*>(p.out.f32 + e) = c4[c];
                }
              }
              continue;
            }
            if (!(MODE == CONVT4_SP || MODE == CONVT4_SPH ? pvalid : valid) || (p.dbg & 1)) continue;
            if (p.out.mode == 0) {
              const size_t e = p.out.cp ? (((size_t)b * (N / 16) + j / 16) * p.Ho * p.Wo + (size_t)oy * p.Wo + ox) * 16
                                        : (((size_t)b * p.Ho + oy) * p.Wo + ox) * N + j;
              if (p.out.bf) {  // bf16 variant: 16 values as one 32-byte store
                uint32_t w8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w8[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
                st_global_v8(reinterpret_cast<float*>(reinterpret_cast<uint16_t*>(p.out.f32) + e),
                             reinterpret_cast<const float*>(w8));
              } else {
                // 32-byte stores: each lane writes whole L2 sectors (the lanes' pixels are
                // 2 apart in the ConvT phases, so a warp's stores cannot coalesce further)
#pragma unroll
                for (int i = 0; i < 16; i += 8) st_global_v8(p.out.f32 + e + i, v + i);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) gsum[j + i] += v[i];
            } else {
              int plane = 0, qo;
              if (p.out.mode == 1) {
                qo = oy * p.out.pl.L + ox;
              } else {
                plane = (oy & 1) * 2 + (ox & 1);
                qo = (oy >> 1) * p.out.pl.L + (ox >> 1);
              }
              float v0[8], v1[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                v0[i] = v[i];
                v1[i] = v[8 + i];
              }
              pl_store8(p.out.pl, b, plane, j / 8, qo, v0);
              pl_store8(p.out.pl, b, plane, j / 8 + 1, qo, v1);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty[slot]));
      if (et == 0) trace_at(p.trace, 3, 2 * ic + 1);
      if (et == 0) trace_cta_item(p.trace, (int)ic);
      if (p.out.mode != 0 && it == 0) pl_zero_margins(p.out.pl, b, et, EPW * 32);
      if (p.out.mode == 0 && p.out.gap) {
        // deterministic: a fixed butterfly over the lanes, then a fixed-order sum of the
        // 8 warp partials
        gap_lane_reduce<N>(gsum, lane, red + (warp - kEpiWarp0) * N);
        asm volatile("bar.sync 1, %0;" ::"n"(EPW * 32) : "memory");
        if (et < N) {
          float s = red[et];
#pragma unroll
          for (int w = 1; w < EPW; ++w) s += red[w * N + et];
          p.out.gap[((size_t)b * p.items_per_image + it) * N + et] = s;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(EPW * 32) : "memory");
      }
    }
  } else {
    if constexpr (MODE == CONV_STEMT) {
      // ===================== im2col warps of the tensor-core stem ==========================
      // A stage of chunk f (frame f) = the 4x4 frame window of every half-resolution
      // position's 2x2 pixel block: K index e of 8-channel group kg is window pixel
      // (wy, wx) = (2kg + e/4, e%4), i.e. frame pixel (2y - 1 + wy, 2x - 1 + wx), zero
      // outside the frame, split into bf16 hi (+ lo).  Unit = (kg, position): consecutive
      // threads write consecutive 16-byte core-matrix rows.
      constexpr int F = STEM;
      constexpr int NP = NPASS_A;
      grid_dep_wait();
      const int st = threadIdx.x - kStemWarp0 * 32;
      const int L = p.L, W = p.W, H = p.H;
      const int PG = G * 128;
      int stage = 0, xs = 0;
      uint32_t phase = 0, xph = 0;
      for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        int b, it;
        item_coords(item, p, b, it);
        const int q0 = it * PG;
        const int xr0 = 2 * (int)__umulhi((uint32_t)q0, p.L_mul) - 1;
        mbar_wait(smem_u32(&xfull[xs]), xph);
#pragma unroll 1
        for (int f = 0; f < F; ++f) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const float* xr = xring + ((size_t)xs * F + f) * p.stem_xrows * W;
          uint8_t* a = a_base + (size_t)stage * p.a_stage_bytes;
          // UB units per thread and pass: all frame loads first, then the conversions and
          // stores (one builder warp per SM sub-partition: the LDS latency must overlap)
          constexpr int UB = 4;
          for (int u0 = st; u0 < 2 * PG; u0 += UB * kStemtThreads) {
            float v[UB][8];
#pragma unroll
            for (int k = 0; k < UB; ++k) {
              const int u = u0 + k * kStemtThreads;
              const int kg = u >= PG ? 1 : 0, i = u - kg * PG;
              const int q = q0 + i;
              const int y = (int)__umulhi((uint32_t)q, p.L_mul), x = q - y * L;
              const bool pos_ok = u < 2 * PG && y < p.Hp && x < p.Wp;
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                const int iy = 2 * y - 1 + 2 * kg + r;
                const bool row_ok = pos_ok && iy >= 0 && iy < H;
                const float* row = xr + (size_t)(iy - xr0) * W;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const int ix = 2 * x - 1 + c;
                  v[k][r * 4 + c] = (row_ok && ix >= 0 && ix < W) ? row[ix] : 0.f;
                }
              }
            }
#pragma unroll
            for (int k = 0; k < UB; ++k) {
              const int u = u0 + k * kStemtThreads;
              if (u >= 2 * PG) break;
              const int kg = u >= PG ? 1 : 0, i = u - kg * PG;
              uint32_t hw[4], lw[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[k][2 * e], v[k][2 * e + 1]);
                hw[e] = *reinterpret_cast<const uint32_t*>(&h2);
                if (NP == 2) {
                  const float2 hf = __bfloat1622float2(h2);
                  const __nv_bfloat162 l2 = __floats2bfloat162_rn(v[k][2 * e] - hf.x, v[k][2 * e + 1] - hf.y);
                  lw[e] = *reinterpret_cast<const uint32_t*>(&l2);
                }
              }
              *reinterpret_cast<uint4*>(a + ((size_t)kg * p.P_max + i) * 16) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
              if (NP == 2)
                *reinterpret_cast<uint4*>(a + ((size_t)(2 + kg) * p.P_max + i) * 16) =
                    make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> UMMA
          mbar_arrive(smem_u32(&full[stage]));
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mbar_arrive(smem_u32(&xempty[xs]));
        if (++xs == 2) {
          xs = 0;
          xph ^= 1u;
        }
      }
    } else if constexpr (STEM == kGateIn) {
      // ===================== gate-in builder warps ======================================
      // A stage of K chunk c (16 channels): staged positions i = 0..P-1 at q = q0 - L - 1 + i
      // (P = 128G + 2L + 2, the S1 taps' span); unit (i, quad j) = channels c*16 + 4j..+3 of
      // that pixel of the previous block's NHWC fp32 output: v = x * gate (+ skip hi + lo),
      // the gate kernels' arithmetic (planes.cuh gate_mul / gate_fma) so every plane value is
      // bitwise the one gate_apply writes, split into bf16 hi (+ lo): 8 bytes per pass at
      // core-matrix row i, byte (j & 1) * 8 of cg8 block j >> 1.  Zero outside the image and
      // at the pad column.  The item's own positions [q0, q0 + 128G) leave as the gated
      // tensor's operand planes (planes.cuh border contract kept): PL by one bulk copy per
      // (pass, cg8) block range of the stage, PP by 8-byte stores.
      constexpr int NP = NPASS_A;
      constexpr int NT = kGateInThreads;
      constexpr int UB = 4;  // units per thread in flight
      grid_dep_wait();       // x, the gates and the skip come from the previous kernels
      const int st = threadIdx.x - kStemWarp0 * 32;
      const int L = p.L, W = p.W, H = p.H, C = p.C;
      const int P = G * 128 + 2 * L + 2;
      const int Lp = W / 2 + 1;
      const bool has_skip = p.gskip.base != nullptr, has_pp = p.gpp.base != nullptr;
      int stage = 0, xs = 0;
      uint32_t phase = 0, xph = 0;
      for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        int b, it;
        item_coords(item, p, b, it);
        const int q0 = it * G * 128, qa = q0 - L - 1;
        const int y_lo = max(floordiv(qa, L), 0);  // first staged row (as the producer)
        if (it == 0) {  // top / bottom margins of the side-output planes, once per image
          pl_zero_margins(p.gpl, b, st, NT);
          if (has_pp) pl_zero_margins(p.gpp, b, st, NT);
        }
        for (int c = 0; c < C / 16; ++c) {
          // the PL bulk stores that last read this stage (>= 2 chunks ago) are done
          if (st == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory");
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          uint8_t* a = a_base + (size_t)stage * p.a_stage_bytes;
          const int j = st & 3;  // NT % 4 == 0: a thread keeps its channel quad
          const float4 g4 = *reinterpret_cast<const float4*>(p.gates + (size_t)b * C + c * 16 + 4 * j);
          mbar_wait(smem_u32(&xfull[xs]), xph);
          const uint8_t* xr = reinterpret_cast<const uint8_t*>(xring) + (size_t)xs * p.stem_xstage;
          const uint8_t* skr = xr + p.gx_skip_off + (size_t)(j >> 1) * P * 16 + (j & 1) * 8;  // pass 0 block
          for (int u0 = st; u0 < 4 * P; u0 += UB * NT) {
            float4 xv[UB];
            uint2 sh[UB], sl[UB];
            bool ok[UB];
#pragma unroll
            for (int k = 0; k < UB; ++k) {
              const int u = u0 + k * NT, i = u >> 2;
              const int q = qa + i;
              const int y = (int)__umulhi((uint32_t)(q + 2 * L), p.L_mul) - 2;  // floor(q / L), q >= -2L
              const int x = q - y * L;
              ok[k] = u < 4 * P && y >= 0 && y < H && x < W;
              xv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
              sh[k] = sl[k] = make_uint2(0u, 0u);
              if (ok[k]) {
                xv[k] = *reinterpret_cast<const float4*>(xr + ((size_t)(y - y_lo) * W + x) * 64 + j * 16);
                if (has_skip) {
                  sh[k] = *reinterpret_cast<const uint2*>(skr + (size_t)i * 16);
                  if (NP == 2) sl[k] = *reinterpret_cast<const uint2*>(skr + (size_t)(2 * P + i) * 16);
                }
              }
            }
#pragma unroll
            for (int k = 0; k < UB; ++k) {
              const int u = u0 + k * NT, i = u >> 2;
              if (u >= 4 * P) break;
              float v[4] = {0.f, 0.f, 0.f, 0.f};
              if (ok[k]) {
                const float xs4[4] = {xv[k].x, xv[k].y, xv[k].z, xv[k].w};
                const float gs4[4] = {g4.x, g4.y, g4.z, g4.w};
                if (has_skip) {
                  float s4[4];
                  s4[0] = __uint_as_float(sh[k].x << 16);
                  s4[1] = __uint_as_float(sh[k].x & 0xFFFF0000u);
                  s4[2] = __uint_as_float(sh[k].y << 16);
                  s4[3] = __uint_as_float(sh[k].y & 0xFFFF0000u);
                  if (NP == 2) {
                    s4[0] += __uint_as_float(sl[k].x << 16);
                    s4[1] += __uint_as_float(sl[k].x & 0xFFFF0000u);
                    s4[2] += __uint_as_float(sl[k].y << 16);
                    s4[3] += __uint_as_float(sl[k].y & 0xFFFF0000u);
                  }
#pragma unroll
                  for (int e = 0; e < 4; ++e) v[e] = gate_fma(xs4[e], gs4[e], s4[e]);
                } else {
#pragma unroll
                  for (int e = 0; e < 4; ++e) v[e] = gate_mul(xs4[e], gs4[e]);
                }
              }
              float hi[4], lo[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                hi[e] = bf16_round(v[e]);
                lo[e] = v[e] - hi[e];
              }
              const uint2 hw = make_uint2(pack_bf16x2(hi[0], hi[1]), pack_bf16x2(hi[2], hi[3]));
              const uint32_t off = ((uint32_t)(j >> 1) * p.P_max + i) * 16 + (j & 1) * 8;
              *reinterpret_cast<uint2*>(a + off) = hw;
              uint2 lw = make_uint2(0u, 0u);
              if (NP == 2) {
                lw = make_uint2(pack_bf16x2(lo[0], lo[1]), pack_bf16x2(lo[2], lo[3]));
                *reinterpret_cast<uint2*>(a + off + 2u * p.P_max * 16) = lw;
              }
              // phase-plane side output of own positions (pad column: both px planes' pad)
              if (has_pp && i >= L + 1 && i < L + 1 + G * 128) {
                const int q = qa + i;
                const int y = (int)__umulhi((uint32_t)q, p.L_mul), x = q - y * L;
                if (y < H) {
                  uint16_t* ppb = p.gpp.base + (int64_t)b * p.gpp.img_stride +
                                  (p.gpp.block_index(c, 0, j >> 1) + p.gpp.off) * 8 + (j & 1) * 4;
                  const size_t lod = (size_t)(NP == 2 ? 2 : 0) * p.gpp.Q * 8;
                  if (x < W) {
                    uint16_t* d = ppb + (int64_t)((y & 1) * 2 + (x & 1)) * p.gpp.plane_stride +
                                  (size_t)((y >> 1) * Lp + (x >> 1)) * 8;
                    *reinterpret_cast<uint2*>(d) = hw;
                    if (NP == 2) *reinterpret_cast<uint2*>(d + lod) = lw;
                  } else {
#pragma unroll
                    for (int px = 0; px < 2; ++px) {
                      uint16_t* d = ppb + (int64_t)((y & 1) * 2 + px) * p.gpp.plane_stride +
                                    (size_t)((y >> 1) * Lp + W / 2) * 8;
                      *reinterpret_cast<uint2*>(d) = make_uint2(0u, 0u);
                      if (NP == 2) *reinterpret_cast<uint2*>(d + lod) = make_uint2(0u, 0u);
                    }
                  }
                }
              }
            }
          }
          mbar_arrive(smem_u32(&xempty[xs]));  // this thread is done reading the x stage
          if (++xs == p.gx_nst) {
            xs = 0;
            xph ^= 1u;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> UMMA / bulk copies
          asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory");
          if (st == 0) {
            // PL side output: the own positions of each (pass, cg8) block, one range each
            // (zeros at pad columns and past the last row: the border contract)
            const int own = min(G * 128, p.Hp * L + L + 8 - q0);  // stay inside the bottom margin
            uint16_t* img = p.gpl.base + (int64_t)b * p.gpl.img_stride;
#pragma unroll
            for (int pass = 0; pass < NP; ++pass)
#pragma unroll
              for (int cg8 = 0; cg8 < 2; ++cg8)
                bulk_s2g(img + (p.gpl.block_index(c, pass, cg8) + q0 + p.gpl.off) * 8,
                         smem_u32(a + ((size_t)(pass * 2 + cg8) * p.P_max + L + 1) * 16), (uint32_t)own * 16);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          mbar_arrive(smem_u32(&full[stage]));
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      if (st == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // PL stores complete
    } else if constexpr (STEM > 0) {
      // ===================== stem warps: relu(conv3x3(frames)) into the A stages ==========
      // Every staged position of the item (its 128G positions and the 2L+2 halo) is
      // computed from the frame rows in the x ring — the stem never makes an HBM round trip
      // for this conv — and written as bf16 hi (+ lo) core-matrix rows of the A stage.
      // Thread = (position slot, channel pair j): the pair's F*9 weight pairs live in
      // registers, a warp covers 4 positions x 8 pairs, so each frame value is one
      // broadcast shared-memory load for 8 lanes.  Arithmetic is stem_const_kernel's
      // (edge_conv.cu): FFMA2 per channel pair in the order (frame, kx, ky) from the bias,
      // then ReLU — bitwise the unfused stem.  The item's own positions then leave as the
      // stem's operand planes: PL rows by bulk copies of the staged block ranges, PP by
      // 16-byte copies (enc0.s2's residual source and the head's skip).
      constexpr int F = STEM;
      constexpr int NP = NPASS_A;  // 2: hi + lo (fp32 contract), 1: bf16
      grid_dep_wait();             // the stem planes may still be read by the previous kernel
      const int st = threadIdx.x - kStemWarp0 * 32;
      const int j = st & 7;                      // channel pair
      const int slot = st >> 3;                  // position slot 0..31
      const int L = p.L, W = p.W, H = p.H, Lp = W / 2 + 1;
      const int P = G * 128 + 2 * L + 2;
      unsigned long long w2[F * 9];
#pragma unroll
      for (int t = 0; t < F * 9; ++t) {
        // through an opaque move: the pair stays in a register for the whole kernel instead
        // of an indexed constant-bank reload per use
        const unsigned long long wc = *reinterpret_cast<const unsigned long long*>(&p.stem_w[t * kStemC + 2 * j]);
        asm volatile("mov.b64 %0, %1;" : "=l"(w2[t]) : "l"(wc));
      }
      unsigned long long b2;
      asm volatile("mov.b64 %0, %1;" : "=l"(b2) : "l"(*reinterpret_cast<const unsigned long long*>(&p.stem_b[2 * j])));
      const uint32_t row_hi = (uint32_t)((j >> 2) * p.P_max) * 16 + (uint32_t)(j & 3) * 4;  // pass 0, cg8
      const uint32_t row_lo = row_hi + 2u * p.P_max * 16;                                   // pass 1
      const size_t QB = (size_t)p.s_pl.Q * 8, QBp = (size_t)p.s_pp.Q * 8;
      int stage = 0, xs = 0;
      uint32_t phase = 0, xph = 0;
      for (int item = blockIdx.x; item < p.total_items; item += gridDim.x) {
        int b, it;
        item_coords(item, p, b, it);
        const int q0 = it * G * 128, qa = q0 - L - 1;
        const int xr0 = floordiv(qa, L) - 1;
        if (it == 0) {  // top / bottom margins of the stem planes, once per image
          if (p.s_has_pl) pl_zero_margins(p.s_pl, b, st, kStemThreads);
          pl_zero_margins(p.s_pp, b, st, kStemThreads);
        }
        // the PL bulk store that last read this stage (stages >= 2 items ago) is done
        if (st == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"n"(kStemThreads) : "memory");
        mbar_wait(smem_u32(&xfull[xs]), xph);
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        const float* xr = xring + (size_t)xs * F * p.stem_xrows * W;
        uint8_t* a = a_base + (size_t)stage * p.a_stage_bytes;
        for (int i = slot; i < P; i += kStemThreads / 8) {
          const int q = qa + i;
          const int y = (int)__umulhi((uint32_t)(q + 2 * L), p.L_mul) - 2;  // floor(q / L), q >= -2L
          const int x = q - y * L;
          float v0 = 0.f, v1 = 0.f;
          if (y >= 0 && y < H && x < W) {
            unsigned long long acc = b2;
#pragma unroll
            for (int ci = 0; ci < F; ++ci) {
              const float* xc = xr + (size_t)ci * p.stem_xrows * W;
#pragma unroll
              for (int kx = 0; kx < 3; ++kx) {
                const int ix = x + kx - 1;
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) {
                  const int iy = y - 1 + ky;
                  float t = (ix >= 0 && ix < W && iy >= 0 && iy < H) ? xc[(iy - xr0) * W + ix] : 0.f;
                  if (NP == 1) t = bf16_round(t);
                  f2_fma(acc, f2_pack(t, t), w2[(ci * 3 + ky) * 3 + kx]);
                }
              }
            }
            f2_unpack(acc, v0, v1);
            v0 = fmaxf(v0, 0.f);
            v1 = fmaxf(v1, 0.f);
          }
          const __nv_bfloat162 hb = __floats2bfloat162_rn(v0, v1);
          *reinterpret_cast<__nv_bfloat162*>(a + row_hi + (uint32_t)i * 16) = hb;
          if (NP == 2) {
            const float2 hf = __bfloat1622float2(hb);
            *reinterpret_cast<__nv_bfloat162*>(a + row_lo + (uint32_t)i * 16) = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> UMMA / bulk copies
        asm volatile("bar.sync 2, %0;" ::"n"(kStemThreads) : "memory");
        // the item's own positions [q0, q0 + 128G) sit at stage rows L+1 .. : PL = the staged
        // block ranges (zeros at pad columns and past the last row, i.e. the border contract)
        const int own = min(G * 128, p.Hp * L + L + 8 - q0);  // stay inside the bottom margin
        if (p.s_has_pl && st == 0) {
          uint16_t* img = p.s_pl.base + (int64_t)b * p.s_pl.img_stride;
#pragma unroll
          for (int blk = 0; blk < 2 * NP; ++blk)
            bulk_s2g(img + ((size_t)blk * p.s_pl.Q + q0 + p.s_pl.off) * 8,
                     smem_u32(a + ((size_t)blk * p.P_max + L + 1) * 16), (uint32_t)own * 16);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // PP: 16-byte copies of the owned valid positions, pad columns zeroed
        uint16_t* ppb = p.s_pp.base + (int64_t)b * p.s_pp.img_stride + (size_t)p.s_pp.off * 8;
        for (int u = st; u < G * 128 * 2 * NP; u += kStemThreads) {
          const int k = u % (G * 128), blk = u / (G * 128);  // blk = pass * 2 + cg8
          const int q = q0 + k;
          const int y = (int)__umulhi((uint32_t)q, p.L_mul), x = q - y * L;
          if (y >= H) continue;
          if (x < W) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + ((size_t)blk * p.P_max + L + 1 + k) * 16);
            *reinterpret_cast<uint4*>(ppb + (int64_t)((y & 1) * 2 + (x & 1)) * p.s_pp.plane_stride +
                                      (size_t)blk * QBp + (size_t)((y >> 1) * Lp + (x >> 1)) * 8) = v;
          } else {  // x == W: the pad columns of both px planes of this plane row
#pragma unroll
            for (int px = 0; px < 2; ++px)
              *reinterpret_cast<uint4*>(ppb + (int64_t)((y & 1) * 2 + px) * p.s_pp.plane_stride +
                                        (size_t)blk * QBp + (size_t)((y >> 1) * Lp + W / 2) * 8) =
                  make_uint4(0, 0, 0, 0);
          }
        }
        (void)QB;
        mbar_arrive(smem_u32(&full[stage]));
        mbar_arrive(smem_u32(&xempty[xs]));
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1u;
        }
        if (++xs == 2) {
          xs = 0;
          xph ^= 1u;
        }
      }
      if (st == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // PL stores complete
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_at(p.trace, 4, 1);
    trace_cta(p.trace, 1);
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols)
                 : "memory");
  }
}

template <int N, int NPM, int G, int F>
void launch_stem_k(const Params& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = tc_conv_kernel<N, CONV3_S1, false, NPM, G, 1, F>;
  ensure_dyn_smem(kern, kMaxSmem);
  launch_pdl(kern, dim3(grid), dim3(kThreadsStem), smem, st, "tc_conv_kernel<stem>", p);
}

template <int NPM, int G, int F>
void launch_stemt_k(const Params& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = tc_conv_kernel<16, CONV_STEMT, false, NPM, G, 1, F>;
  ensure_dyn_smem(kern, kMaxSmem);
  launch_pdl(kern, dim3(grid), dim3(threads_of(CONV_STEMT, F)), smem, st, "tc_conv_kernel<stemt>", p);
}

template <int N, int MODE, bool DUAL, int NPM, int G>
void launch_k(const Params& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = p.cps == 2 ? tc_conv_kernel<N, MODE, DUAL, NPM, G, 2> : tc_conv_kernel<N, MODE, DUAL, NPM, G, 1>;
  ensure_dyn_smem(kern, kMaxSmem);
  launch_pdl(kern, dim3(grid), dim3(threads_of(MODE, 0)), smem, st, "tc_conv_kernel", p);
}

template <int MODE, bool DUAL>
void dispatch_mode(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st) {
  auto by_g = [&](auto n_c, auto npm_c) {
    constexpr int NN = decltype(n_c)::value, PM = decltype(npm_c)::value;
    switch (G) {
      case 1: return launch_k<NN, MODE, DUAL, PM, 1>(p, grid, smem, st);
      case 2: return launch_k<NN, MODE, DUAL, PM, 2>(p, grid, smem, st);
      default: return launch_k<NN, MODE, DUAL, PM, 4>(p, grid, smem, st);
    }
  };
  auto by_npm = [&](auto n_c) {
    switch (npm) {
      case kNpmBf16: return by_g(n_c, std::integral_constant<int, kNpmBf16>{});
      case kNpm3: return by_g(n_c, std::integral_constant<int, kNpm3>{});
      default: return by_g(n_c, std::integral_constant<int, kNpmConcat>{});
    }
  };
  switch (n) {
    case 16: return by_npm(std::integral_constant<int, 16>{});
    case 32: return by_npm(std::integral_constant<int, 32>{});
    default: return by_npm(std::integral_constant<int, 64>{});
  }
}

void dispatch_s1(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_s2(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_t(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_th(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_rows(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_s1p(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_stem(int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_stemt(int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_sp(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_sph(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);
void dispatch_gatein(int n, int npm, int G, const Params& p, int grid, size_t smem, cudaStream_t st);

}  // namespace detail
}  // namespace tc
}  // namespace stda
