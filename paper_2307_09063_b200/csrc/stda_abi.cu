// C ABI of the engine (include/stda_b200.h): plans, workspace planning, the forward
// sequencer, the pipelined host-buffer path, block-level entries and the synthesiser.
//
// Forward dataflow (reference model.py:185-199), one launch per row:
//   stem          conv3x3 s1 + relu                          x        -> s
//   enc i  s1     reparameterised conv3x3 s1 + relu          cur      -> m
//          s2     relu(conv3x3s2(m)+b) + conv3x3s2(cur)+b    m, cur   -> e_i, GAP tiles
//          gate   sigmoid(conv1d(mean))                      GAP      -> g_i      cur = e_i*g_i
//   dec j  s1     reparameterised conv3x3 s1 + relu          cur      -> m
//          s2     relu(convT(m)+b) + convT(cur)+b (4 phases) m, cur   -> d_j, GAP tiles
//          gate                                              GAP      -> g'_j     cur = d_j*g'_j + skip
//   head   conv3x3 s1                                        cur      -> y
// Gates and skip adds are applied while the NEXT kernel stages its input tile.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/stda_b200.h"
#include "common.cuh"
#include "simt_conv.cuh"
#include "tc_conv.cuh"
#include "edge_conv.cuh"

namespace stda {

void launch_synth(uint64_t seed, int scene, int64_t seq0, int64_t seq_step, int64_t frame0,
                  int frames_per_seq, int frame_order, int64_t n_out, int H, int W, float* out,
                  cudaStream_t st);
void launch_denoise_epilogue(const float* y, float* out, int64_t B, int H, int W, float scale, float z_min,
                             float stdv, float mean, cudaStream_t st);
void launch_rd_frontend(const float2* beat, int64_t n, int N, int M, int P, int Q, const double* stats,
                        bool clutter, int layout, float* out, cudaStream_t st);
void launch_linear(const float* X, int64_t xs, const float* Wt, const float* b, float* Y, int M, int N, int K,
                   bool relu, float* partial, cudaStream_t st);
int linear_splits(int K);
void launch_maxpool2(const float* x, float* y, int64_t planes, int H, int W, cudaStream_t st);
void launch_score(const void* clean, int clean_kind, const float* test_db, int64_t n, int P, int Q, int guard0,
                  int guard1, int train0, int train1, double alpha_obj, double alpha_det, int margin, double* out,
                  unsigned char* det_hits, cudaStream_t st);

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// Programmatic dependent launch edges between the forward's kernels.  Measured at the end
// of round 1: inside a CUDA graph plain stream order is 0.3 % faster (165.95K vs 165.45K
// triplets/s at C2: no CTA of the next kernel fits beside a running one, so the early
// launch buys nothing), while eager launches (the host-buffer path) are 7 % faster with
// the edges (they hide the kernel-to-kernel launch gap).  So: on unless the stream is
// being captured.  env STDA_PDL=1 / 0 forces them on / off.
// bf16 variant: stage-2 outputs (ECA inputs) stored as bf16 NHWC — the variant rounds the
// gated values to bf16 anyway; halves their HBM round trip.  env STDA_BF_NHWC=0 keeps fp32.
bool bf_nhwc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_BF_NHWC");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ... except the head's input: the strip head rewrites d in place as u, and bf16 u costs the
// conv an unpack per value (measured +3 us head vs -3 us dec1.s2: a wash).  env STDA_HEAD_BF=1.
bool head_bf_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_HEAD_BF");
    return e && e[0] == '1';
  }();
  return on;
}

bool pdl_enabled(cudaStream_t st) {
  static const int mode = [] {
    const char* e = std::getenv("STDA_PDL");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  if (mode >= 0) return mode == 1;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return true;
  return cs == cudaStreamCaptureStatusNone;
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    STDA_CUDA(cudaGetDevice(&prev));
    if (prev != dev) STDA_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

}  // namespace
}  // namespace stda

using namespace stda;

struct EncLayers {
  ConvLayer s1, dn, rs;
  tc::TcLayerDesc s1_tc{}, s2_tc{};  // tensor-core versions (dn+rs dual in s2_tc)
  float* eca = nullptr;
};
struct DecLayers {
  ConvLayer s1, up, rs;
  tc::TcLayerDesc s1_tc{}, s2_tc{};
  float* eca = nullptr;
};

struct stda_plan {
  int kind = 0;  // 0 = network, 1 = encoder block, 2 = decoder block
  stda_config cfg{};
  int device = 0;
  bool bf16 = false;
  int block_channels = 0;
  ConvLayer stem, head;
  std::vector<EncLayers> enc;
  std::vector<DecLayers> dec;
  std::vector<void*> allocations;

  ~stda_plan() {
    for (void* p : allocations) cudaFree(p);
  }

  float* upload(const std::vector<float>& v) {
    void* p = nullptr;
    STDA_CUDA(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(float)));
    allocations.push_back(p);
    STDA_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
    return static_cast<float*>(p);
  }

  // canonical weights at `src` -> SIMT layout on device; advances src
  ConvLayer make_layer(int mode, int cin, int cout, const float*& src) {
    ConvLayer L;
    L.mode = mode;
    L.cin = cin;
    L.cout = cout;
    L.cob = simt_cob_for(cout);
    L.tapsz = simt_tapsz(mode, L.cob);
    const int nblk = cdiv(cout, L.cob);
    const size_t wn = (size_t)cout * cin * (mode == CONVT4_S2 ? 16 : 9);
    std::vector<float> w((size_t)nblk * cin * L.tapsz), b((size_t)nblk * L.cob);
    simt_pack(mode, cin, cout, src, src + wn, bf16, w.data(), b.data());
    src += wn + cout;
    L.w = upload(w);
    L.b = upload(b);
    return L;
  }

  float* make_vec(int n, const float*& src) {
    std::vector<float> v(src, src + n);
    src += n;
    return upload(v);
  }

  void* upload_bytes(const void* data, size_t bytes) {
    void* p = nullptr;
    STDA_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    allocations.push_back(p);
    STDA_CUDA(cudaMemcpy(p, data, bytes, cudaMemcpyHostToDevice));
    return p;
  }

  // tensor-core layer from canonical weights w0/b0 (+ w1/b1 for a dual stage)
  tc::TcLayerDesc make_tc(int mode, int cin, int cout, const float* w0, const float* b0,
                          const float* w1, const float* b1, int plane_w) {
    tc::TcLayerDesc d;
    std::vector<uint16_t> packed;
    tc::tc_pack_layer(d, mode, cin, cout, w0, w1, bf16, packed, plane_w);
    d.w = static_cast<const uint16_t*>(upload_bytes(packed.data(), packed.size() * 2));
    d.bias0 = upload(std::vector<float>(b0, b0 + cout));
    d.bias1 = w1 ? upload(std::vector<float>(b1, b1 + cout)) : nullptr;
    for (int c = 0; c < cout && c < 64; ++c) {
      d.bias0_c[c] = b0[c];
      d.bias1_c[c] = w1 ? b1[c] : 0.f;
    }
    return d;
  }

  bool use_tc = false;  // every encoder/decoder conv runs on the tcgen05 kernel
  bool stem_fused = false;  // the stem runs inside the enc0.s1 tcgen05 kernel (tc_launch_stem)
  bool stem_pp = false;     // the stem writes phase planes only; enc0.s1 = CONV3_S1P, head skip from PP
  bool stem_tc_on = false;  // ... computed on the tensor cores (CONV_STEMT, tc_launch_stemt)
  tc::TcLayerDesc stem_tc;
  float* head_wt = nullptr;  // head weights [9][c0] for the NHWC head kernel
  std::vector<float> stem_canon;  // host copy of the stem's canonical weights + bias (constant-bank stem)
  std::vector<float> head_host;   // host copy of head_wt (constant-bank strip head)
  // baselines (kind 3 = MLP, kind 4 = CAE; stda_baseline_plan_create)
  int bh = 0, bw = 0, hidden = 0;
  float* lin_w[3] = {};
  float* lin_b[3] = {};
  ConvLayer cae[6];  // conv1, conv2, convT1, its all-zero twin, convT2, its all-zero twin
};

namespace {

size_t canonical_floats(const stda_config& c) {
  const size_t c0 = c.stem_channels, f = c.input_frames, k = c.eca_kernel;
  size_t n = c0 * f * 9 + c0;
  for (int i = 0; i < c.stages; ++i) {
    const size_t ch = c0 << i;
    n += ch * ch * 9 + ch + 2 * (2 * ch * ch * 9 + 2 * ch) + k;
  }
  for (int j = 0; j < c.stages; ++j) {
    const size_t c2 = c0 << (c.stages - j), ch = c2 / 2;
    n += c2 * c2 * 9 + c2 + 2 * (ch * c2 * 16 + ch) + k;
  }
  return n + c0 * 9 + 1;
}

void validate(const stda_config& c) {
  STDA_CHECK(c.input_frames >= 1 && c.stem_channels >= 1 && c.stages >= 1,
             "config values must be positive");
  STDA_CHECK(c.eca_kernel >= 1 && c.eca_kernel % 2 == 1, "ECA kernel size must be odd");
  const int d = 1 << c.stages;
  STDA_CHECK(c.map_height > 0 && c.map_width > 0 && c.map_height % d == 0 && c.map_width % d == 0,
             "map size must be divisible by 2^stages");
  STDA_CHECK(c.precision == STDA_PRECISION_FP32 || c.precision == STDA_PRECISION_BF16,
             "unknown precision");
  STDA_CHECK(((int64_t)c.stem_channels << c.stages) <= 4096, "channel count too large");
}

// Workspace for a batch of B triplets; base == nullptr only sizes it.
struct NetWs {
  float* s = nullptr;
  float* m = nullptr;
  std::vector<float*> e, ge, pe, d, gd, pd;
  // tensor-core path: operand planes
  PlBuf pl_s, pp_s;
  std::vector<PlBuf> pl_a, pp_a, pl_b, pl_m;
  size_t bytes = 0;
};

NetWs plan_ws(const stda_plan& p, int64_t B, char* base) {
  const stda_config& c = p.cfg;
  const int S = c.stages;
  NetWs w;
  size_t off = 0;
  auto take = [&](size_t nfloat) -> float* {
    float* r = base ? reinterpret_cast<float*>(base + off) : nullptr;
    off += align_up(nfloat * sizeof(float));
    return r;
  };
  const size_t HW = (size_t)c.map_height * c.map_width;
  w.s = take(B * c.stem_channels * HW);
  // the "mixed" stage-1 buffer is reused by every block: size of the largest
  size_t mmax = 0;
  for (int i = 0; i < S; ++i) mmax = std::max(mmax, (size_t)(c.stem_channels << i) * (HW >> (2 * i)));
  for (int j = 0; j < S; ++j) {
    const int lvl = S - j;  // decoder input level
    mmax = std::max(mmax, (size_t)(c.stem_channels << lvl) * (HW >> (2 * lvl)));
  }
  w.m = take(B * mmax);
  for (int i = 0; i < S; ++i) {
    const int ch = c.stem_channels << (i + 1);
    const int h = c.map_height >> (i + 1), wd = c.map_width >> (i + 1);
    w.e.push_back(take(B * ch * (size_t)h * wd));
    // GAP partials: SIMT tiles or tensor-core items (<= one per 128 linear positions)
    const size_t tiles = std::max<size_t>(conv_tiles(CONV3_S2, h, wd), cdiv(h * (wd + 1), 128));
    w.pe.push_back(take(B * ch * tiles));
    w.ge.push_back(take(B * ch));
  }
  for (int j = 0; j < S; ++j) {
    const int lvl = S - j - 1;  // output level
    const int ch = c.stem_channels << lvl;
    const int h = c.map_height >> lvl, wd = c.map_width >> lvl;
    w.d.push_back(take(B * ch * (size_t)h * wd));
    const size_t tiles =
        std::max<size_t>(conv_tiles(CONVT4_S2, h, wd),
                         2 * cdiv((h / 2) * (wd / 2 + 1) + wd / 2 + 2, 128));  // x2: half-phase items; +1 row: SP
    w.pd.push_back(take(B * ch * tiles));
    w.gd.push_back(take(B * ch));
  }
  if (p.use_tc) {
    // operand planes (planes.cuh) of every tensor a tcgen05 conv reads
    const int np = p.bf16 ? 1 : 2;
    const int H = c.map_height, W = c.map_width, c0 = c.stem_channels;
    auto take_pl = [&](PlBuf b) -> PlBuf {
      const size_t bytes = plbuf_bytes(b, B);
      b.base = base ? reinterpret_cast<uint16_t*>(base + off) : nullptr;
      off += align_up(bytes);
      return b;
    };
    w.pl_s = take_pl(make_plbuf(1, H, W, c0, np));
    w.pp_s = take_pl(make_plbuf(4, H / 2, W / 2, c0, np));
    // stage-1 outputs: PP for encoder stride-2 consumers, PL for decoder ConvT consumers
    // (separate regions, so every border stays zero after the single zeroing pass)
    for (int i = 0; i < S; ++i)
      w.pl_m.push_back(take_pl(make_plbuf(4, (H >> i) / 2, (W >> i) / 2, c0 << i, np)));
    for (int j = 0; j < S; ++j) {
      const int lvl = S - j;
      w.pl_m.push_back(take_pl(make_plbuf(1, H >> lvl, W >> lvl, c0 << lvl, np)));
    }
    for (int i = 0; i < S; ++i) {
      const int ch = c0 << (i + 1), h = H >> (i + 1), wd = W >> (i + 1);
      w.pl_a.push_back(take_pl(make_plbuf(1, h, wd, ch, np)));
      w.pp_a.push_back(i + 1 < S ? take_pl(make_plbuf(4, h / 2, wd / 2, ch, np)) : PlBuf{});
    }
    for (int j = 0; j + 1 < S; ++j) {
      const int lvl = S - j - 1, ch = c0 << lvl;
      w.pl_b.push_back(take_pl(make_plbuf(1, H >> lvl, W >> lvl, ch, np)));
    }
  }
  w.bytes = off;
  return w;
}

// Optional per-launch event marks (stda_forward_profiled): ev[0] before the first
// launch, ev[i+1] after launch i.
// `only` >= 0 launches that slot alone (stda_forward_launch_repeat; tensor-core path).
struct Marks {
  std::vector<cudaEvent_t>* ev = nullptr;
  int i = 0;
  int n = 0;      // marks so far: the next launch is slot n - 1
  int only = -1;
  bool go() const { return only < 0 || n - 1 == only; }
  void mark(cudaStream_t st) {
    ++n;
    if (ev) STDA_CUDA(cudaEventRecord((*ev)[i++], st));
  }
};

// Tensor-core forward: stem and head on the SIMT kernel (Cin = 3 / Cout = 1), every
// encoder/decoder conv on the tcgen05 kernel; intermediates NHWC fp32.
void run_net_tc(const stda_plan& p, const Src& x, float* y, int64_t B, const NetWs& w,
                cudaStream_t st, Marks mk) {
  const stda_config& c = p.cfg;
  const int S = c.stages, k = c.eca_kernel, c0 = c.stem_channels;
  const bool bf = p.bf16;
  int h = c.map_height, wd = c.map_width;
  const int np = bf ? 1 : 2;
  mk.mark(st);
  // Every operand plane is fully rewritten each forward by its writer, including the
  // tap-reachable borders (pad column, top/bottom margins): no zeroing pass is needed.
  // stage-1 outputs: PP for encoder stride-2 consumers, PL for decoder ConvT consumers
  const std::vector<PlBuf>& mviews = w.pl_m;
  (void)np;
  // stem: fused into the enc0.s1 kernel when the plan and this input allow it
  tc::TcStem stem;
  stem.x = x;
  stem.F = c.input_frames;
  stem.s_pl = w.pl_s;
  stem.s_pp = w.pp_s;
  stem.has_pl = true;
  stem.canon = p.stem_canon.empty() ? nullptr : p.stem_canon.data();
  const bool fuse_stem = p.stem_fused && tc::tc_stem_fusable(p.enc[0].s1_tc, stem, h, wd);
  if (!fuse_stem && p.stem_pp && p.stem_tc_on && tc::tc_stemt_ok(stem, h, wd)) {
    // the stem as a tcgen05 GEMM per half-resolution position, writing the phase planes
    tc::TcLayerDesc ds = p.stem_tc;
    const tc::TcGeometry gs = tc::tc_plan_stemt(ds, (int)B, h, wd, c.input_frames);
    tc::TcOut os;
    os.mode = 2;
    os.pl = w.pp_s;
    if (mk.go()) tc::tc_launch_stemt(ds, gs, stem, os, st);
    mk.mark(st);
  } else if (!fuse_stem) {
    PlBuf no_pl = w.pl_s;
    no_pl.base = nullptr;  // stem_pp: phase planes only
    if (mk.go())
      launch_stem_planes(p.stem.w, p.stem.b, x, c.input_frames, c0, p.stem_pp ? no_pl : w.pl_s, w.pp_s, B, h, wd,
                       bf, st, p.stem_canon.empty() ? nullptr : p.stem_canon.data());
    if (!p.stem_fused) mk.mark(st);  // (fused plans profile stem + enc0.s1 as one launch)
  }
  PlBuf cur_pl = w.pl_s, cur_pp = w.pp_s;
  std::vector<PlBuf> skips{p.stem_pp ? w.pp_s : w.pl_s};
  // gate-on-load: an ECA gate (+ skip) whose consumer is a plain stride-1 conv is applied
  // inside that conv (tc_launch_gatein), which also writes the gated planes; the gate slot
  // then only forms the gates (eca_gates_kernel)
  bool pend = false;
  tc::TcGateIn gin;
  auto s1_launch = [&](tc::TcLayerDesc& d1, const PlBuf& src, const tc::TcOut& o1, int hh, int ww) {
    if (pend) {
      const tc::TcGeometry g1 = tc::tc_plan_gatein(d1, (int)B, hh, ww, gin);
      if (mk.go()) tc::tc_launch_gatein(d1, g1, gin, o1, st, /*rev=*/true);
      pend = false;
    } else {
      const tc::TcGeometry g1 = tc::tc_plan(d1, (int)B, hh, ww);
      if (mk.go()) tc::tc_launch(d1, g1, src, nullptr, o1, true, st, /*rev=*/true);
    }
  };
  // can the next stride-1 conv take this gate on load?
  auto gatein_next = [&](const tc::TcLayerDesc& nxt, const float* x, const float* gates, const PlBuf* skip,
                         const PlBuf& out_pl, const PlBuf* out_pp, int hh, int ww) {
    tc::TcGateIn g;
    g.x = x;
    g.gates = gates;
    if (skip) g.skip = *skip;
    g.out_pl = out_pl;
    if (out_pp) g.out_pp = *out_pp;
    if (!tc::tc_gatein_ok(nxt, g, hh, ww) || !tc::tc_gatein_fits(nxt, (int)B, hh, ww, g)) return false;
    gin = g;
    pend = true;
    return true;
  };
  for (int i = 0; i < S; ++i) {
    const EncLayers& E = p.enc[i];
    tc::TcLayerDesc d1 = E.s1_tc, d2 = E.s2_tc;
    tc::TcOut o1;
    o1.mode = 2;  // phase planes for the stride-2 consumer
    o1.pl = mviews[i];
    if (i == 0 && fuse_stem) {
      const tc::TcGeometry g1 = tc::tc_plan_stem(d1, (int)B, h, wd, c.input_frames);
      if (mk.go()) tc::tc_launch_stem(d1, g1, stem, o1, st, /*rev=*/true);
    } else {
      s1_launch(d1, d1.mode == CONV3_S1P ? cur_pp : cur_pl, o1, h, wd);
    }
    mk.mark(st);
    const tc::TcGeometry g2 = tc::tc_plan(d2, (int)B, h, wd);
    // gate-on-load by the next stride-1 conv: e_i goes out chunk-planar for its builder
    const tc::TcLayerDesc& nxt = i + 1 < S ? p.enc[i + 1].s1_tc : p.dec[0].s1_tc;
    const bool gi_on =
        gatein_next(nxt, w.e[i], w.ge[i], nullptr, w.pl_a[i], i + 1 < S ? &w.pp_a[i] : nullptr, h / 2, wd / 2);
    tc::TcOut o2;
    o2.f32 = w.e[i];
    o2.gap = w.pe[i];
    o2.cp = gi_on ? 1 : 0;
    // bf16 variant: e_i stored as bf16 for the strip gate kernel
    o2.bf = bf && !gi_on && bf_nhwc_enabled() && gate_apply_bf16_ok(false, &w.pl_a[i], B, d2.cout, h / 2, wd / 2);
    if (mk.go()) tc::tc_launch(d2, g2, mviews[i], &cur_pp, o2, true, st);
    mk.mark(st);
    h /= 2;
    wd /= 2;
    // a_i = e_i * gate_i -> PL (next stage-1 / decoder input / skip) and PP (next stride-2)
    // large maps: the gate once per image (planes.cuh kGatesReady), not once per CTA
    const float* gsrc = w.pe[i];
    int gitems = g2.items_per_image;
    if (gi_on) {
      if (mk.go()) launch_eca_gates(gsrc, gitems, E.eca, k, w.ge[i], B, d2.cout, (int64_t)h * wd, st);
    } else {
      if (precompute_gates(gitems, d2.cout)) {
        if (mk.go()) launch_eca_gates(gsrc, gitems, E.eca, k, w.ge[i], B, d2.cout, (int64_t)h * wd, st);
        gsrc = w.ge[i];
        gitems = kGatesReady;
      }
      if (mk.go())
        launch_gate_apply(gsrc, gitems, E.eca, k, w.e[i], nullptr, &w.pl_a[i],
                          i + 1 < S ? &w.pp_a[i] : nullptr, nullptr, B, d2.cout, h, wd, st, o2.bf != 0);
    }
    mk.mark(st);
    cur_pl = w.pl_a[i];
    cur_pp = w.pp_a[i];
    skips.push_back(cur_pl);
  }
  for (int j = 0; j < S; ++j) {
    const DecLayers& D = p.dec[j];
    tc::TcLayerDesc d1 = D.s1_tc, d2 = D.s2_tc;
    const tc::TcGeometry g1 = tc::tc_plan(d1, (int)B, h, wd);
    tc::TcOut o1;
    o1.mode = 1;  // plane for the ConvT consumer
    o1.pl = mviews[S + j];
    (void)g1;
    s1_launch(d1, cur_pl, o1, h, wd);
    mk.mark(st);
    const tc::TcGeometry g2 = tc::tc_plan(d2, (int)B, h, wd);
    const PlBuf& sk = skips[S - 1 - j];
    const bool gi_on = j + 1 < S && sk.planes == 1 &&
                       gatein_next(p.dec[j + 1].s1_tc, w.d[j], w.gd[j], &sk, w.pl_b[j], nullptr, 2 * h, 2 * wd);
    tc::TcOut o2;
    o2.f32 = w.d[j];
    o2.gap = w.pd[j];
    o2.cp = gi_on ? 1 : 0;
    // bf16 variant: d_j stored as bf16 for the strip gate kernel / the strip or tile head
    o2.bf = bf && !gi_on && bf_nhwc_enabled() &&
            (j + 1 < S ? gate_apply_bf16_ok(true, &w.pl_b[j], B, d2.cout, 2 * h, 2 * wd)
                       : head_bf_enabled() && !p.head_host.empty() && head_bf16_ok(c0, B, 2 * h, 2 * wd, sk));
    if (mk.go()) tc::tc_launch(d2, g2, mviews[S + j], &cur_pl, o2, true, st);
    mk.mark(st);
    h *= 2;
    wd *= 2;
    // b_j = d_j * gate + skip  (model.py:197-198); the last one is fused into the head
    const float* gsrc = w.pd[j];
    int gitems = g2.items_per_image;
    if (gi_on) {
      // b_j formed inside dec_{j+1}.s1 (gate-on-load with the skip)
      if (mk.go()) launch_eca_gates(gsrc, gitems, D.eca, k, w.gd[j], B, d2.cout, (int64_t)h * wd, st);
      mk.mark(st);
      cur_pl = w.pl_b[j];
      continue;
    }
    if (precompute_gates(gitems, d2.cout)) {
      if (mk.go()) launch_eca_gates(gsrc, gitems, D.eca, k, w.gd[j], B, d2.cout, (int64_t)h * wd, st);
      gsrc = w.gd[j];
      gitems = kGatesReady;
    }
    if (j + 1 < S) {
      if (mk.go())
        launch_gate_apply(gsrc, gitems, D.eca, k, w.d[j], &sk, &w.pl_b[j], nullptr, nullptr, B, d2.cout, h, wd,
                          st, o2.bf != 0);
      mk.mark(st);
      cur_pl = w.pl_b[j];
    } else {
      if (mk.go())
        launch_head_fused(p.head_wt, p.head.b, gsrc, gitems, D.eca, k, w.d[j], sk, c0, y, B, h,
                        wd, bf, st, p.head_host.empty() ? nullptr : p.head_host.data(), o2.bf != 0);
      mk.mark(st);
    }
  }
}

void run_net(const stda_plan& p, const Src& x, float* y, int64_t B, const NetWs& w, cudaStream_t st,
             Marks mk = Marks{}) {
  if (p.use_tc) return run_net_tc(p, x, y, B, w, st, mk);
  const stda_config& c = p.cfg;
  const int S = c.stages, k = c.eca_kernel;
  const bool bf = p.bf16;
  int h = c.map_height, wd = c.map_width;
  mk.mark(st);
  launch_conv(p.stem, nullptr, x, nullptr, w.s, nullptr, B, h, wd, true, bf, st);
  mk.mark(st);
  Src cur = plain_src(w.s, c.stem_channels, h, wd);
  std::vector<Src> skips{cur};
  for (int i = 0; i < S; ++i) {
    const int ch = c.stem_channels << i;
    const EncLayers& E = p.enc[i];
    launch_conv(E.s1, nullptr, cur, nullptr, w.m, nullptr, B, h, wd, true, bf, st);
    mk.mark(st);
    const Src mixed = plain_src(w.m, ch, h, wd);
    launch_conv(E.dn, &E.rs, mixed, &cur, w.e[i], w.pe[i], B, h, wd, true, bf, st);
    mk.mark(st);
    h /= 2;
    wd /= 2;
    launch_gate(w.pe[i], conv_tiles(CONV3_S2, h, wd), E.eca, k, w.ge[i], B, 2 * ch, h * wd, st);
    mk.mark(st);
    cur = plain_src(w.e[i], 2 * ch, h, wd);
    cur.gx = w.ge[i];
    skips.push_back(cur);
  }
  for (int j = 0; j < S; ++j) {
    const int c2 = c.stem_channels << (S - j), ch = c2 / 2;
    const DecLayers& D = p.dec[j];
    launch_conv(D.s1, nullptr, cur, nullptr, w.m, nullptr, B, h, wd, true, bf, st);
    mk.mark(st);
    const Src mixed = plain_src(w.m, c2, h, wd);
    launch_conv(D.up, &D.rs, mixed, &cur, w.d[j], w.pd[j], B, h, wd, true, bf, st);
    mk.mark(st);
    h *= 2;
    wd *= 2;
    launch_gate(w.pd[j], conv_tiles(CONVT4_S2, h, wd), D.eca, k, w.gd[j], B, ch, h * wd, st);
    mk.mark(st);
    Src nxt = plain_src(w.d[j], ch, h, wd);
    nxt.gx = w.gd[j];
    const Src& sk = skips[S - 1 - j];
    nxt.s = sk.x;
    nxt.sb = sk.xb;
    nxt.sc = sk.xc;
    nxt.gs = sk.gx;
    cur = nxt;
  }
  launch_conv(p.head, nullptr, cur, nullptr, y, nullptr, B, h, wd, false, bf, st);
  mk.mark(st);
}

std::string launch_names(const stda_config& c, bool tc, bool stem_fused = false) {
  std::string s = stem_fused ? "" : "stem;";
  for (int i = 0; i < c.stages; ++i)
    s += std::string(i ? ";" : "") + (i == 0 && stem_fused ? "stem+" : "") + "enc" + std::to_string(i) +
         ".s1;enc" + std::to_string(i) + ".s2;enc" + std::to_string(i) + ".gate";
  for (int j = 0; j < c.stages; ++j) {
    s += ";dec" + std::to_string(j) + ".s1;dec" + std::to_string(j) + ".s2";
    if (!tc || j + 1 < c.stages) s += ";dec" + std::to_string(j) + ".gate";  // tc: last gate fused into head
  }
  return s + ";head";
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    set_error(e.msg);
  } catch (const std::exception& e) {
    set_error(e.what());
  } catch (...) {
    set_error("unknown error");
  }
  return 1;
}

void check_ws(const stda_plan* p, const void* ws, size_t have, size_t need) {
  STDA_CHECK(p != nullptr, "null plan");
  STDA_CHECK(have >= need, "workspace too small: need " + std::to_string(need) + " bytes, got " +
                               std::to_string(have));
  STDA_CHECK(need == 0 || ws != nullptr, "null workspace");
}

}  // namespace

extern "C" {

int stda_abi_version(void) { return STDA_ABI_VERSION; }

const char* stda_last_error(void) { return g_last_error.c_str(); }

size_t stda_blob_floats(const stda_config* cfg) { return cfg ? canonical_floats(*cfg) : 0; }

int stda_plan_create(const stda_config* cfg, const float* blob, size_t n_floats, int device,
                     stda_plan** out) {
  return guarded([&] {
    STDA_CHECK(cfg && blob && out, "null argument");
    validate(*cfg);
    STDA_CHECK(n_floats == canonical_floats(*cfg),
               "blob has " + std::to_string(n_floats) + " floats, config needs " +
                   std::to_string(canonical_floats(*cfg)));
    DeviceGuard g(device);
    auto p = std::make_unique<stda_plan>();
    p->kind = 0;
    p->cfg = *cfg;
    p->device = device;
    p->bf16 = cfg->precision == STDA_PRECISION_BF16;
    const float* src = blob;
    const int c0 = cfg->stem_channels, S = cfg->stages, k = cfg->eca_kernel;
    // the tensor-core path needs every encoder/decoder conv in its supported shape set
    bool tc_ok = true;
    for (int i = 0; i < S; ++i) {
      const int ch = c0 << i;
      tc_ok = tc_ok && tc::tc_supported(CONV3_S1, ch, ch) && tc::tc_supported(CONV3_S2, ch, 2 * ch);
    }
    for (int j = 0; j < S; ++j) {
      const int c2 = c0 << (S - j);
      tc_ok = tc_ok && tc::tc_supported(CONV3_S1, c2, c2) && tc::tc_supported(CONVT4_S2, c2, c2 / 2);
    }
    const char* force = std::getenv("STDA_ENGINE_PATH");  // "simt" forces the generic path
    p->use_tc = tc_ok && !(force && std::strcmp(force, "simt") == 0);
    {
      const size_t n_stem = (size_t)c0 * cfg->input_frames * 9 + c0;
      p->stem_canon.assign(src, src + n_stem);
      if (p->bf16)
        for (float& v : p->stem_canon) v = __bfloat162float(__float2bfloat16_rn(v));
    }
    const float* stem_src = src;  // canonical stem weights [c0][F][3][3] + bias [c0]
    p->stem = p->make_layer(CONV3_S1, cfg->input_frames, c0, src);
    for (int i = 0; i < S; ++i) {
      const int ch = c0 << i;
      EncLayers E;
      const float* w_s1 = src;
      E.s1 = p->make_layer(CONV3_S1, ch, ch, src);
      const float* w_dn = src;
      E.dn = p->make_layer(CONV3_S2, ch, 2 * ch, src);
      const float* w_rs = src;
      E.rs = p->make_layer(CONV3_S2, ch, 2 * ch, src);
      if (p->use_tc) {
        const size_t n1 = (size_t)ch * ch * 9, n2 = (size_t)2 * ch * ch * 9;
        // encoder stage 1 reads the phase planes its stride-2 partner reads anyway (stem /
        // encoder gate PP) and writes the 2x2 output phases of one A read per shift
        // (enc0: also when the stem writes phase planes only, stem_pp)
        static const bool stem_pp_on = [] {
          const char* e = std::getenv("STDA_STEM_PP");
          return !(e && e[0] == '0');
        }();
        if (i == 0)
          p->stem_pp = stem_pp_on && tc::tc_supported(CONV3_S1P, ch, ch) &&
                       stem_pp_only_ok(c0, cfg->input_frames, cfg->map_height, cfg->map_width);
        const int m1 = (tc::s1p_enabled() || (i == 0 && p->stem_pp)) && tc::tc_supported(CONV3_S1P, ch, ch)
                           ? CONV3_S1P
                           : CONV3_S1;
        E.s1_tc = p->make_tc(m1, ch, ch, w_s1, w_s1 + n1, nullptr, nullptr, cfg->map_width >> i);
        E.s2_tc = p->make_tc(CONV3_S2, ch, 2 * ch, w_dn, w_dn + n2, w_rs, w_rs + n2, 0);
      }
      E.eca = p->make_vec(k, src);
      p->enc.push_back(E);
      if (i == 0 && p->use_tc) {
        // static part of tc_stem_fusable (the input's alignment / strides are checked per call)
        static const bool fused_on = [] {
          const char* e = std::getenv("STDA_STEM_FUSED");
          return e && e[0] == '1';
        }();
        p->stem_fused = fused_on && !p->stem_pp && E.s1_tc.mode == CONV3_S1 && c0 == 16 && cfg->input_frames <= 4 &&
                        cfg->map_width % 4 == 0 && cfg->map_width <= 128;
        // the phase-plane stem on the tensor cores (CONV_STEMT)
        const int F = cfg->input_frames;
        if (p->stem_pp && !p->stem_fused && F <= 4 && tc::tc_supported(CONV_STEMT, 16 * F, c0)) {
          const float* sw = stem_src;
          p->stem_tc = p->make_tc(CONV_STEMT, 16 * F, c0, sw, sw + (size_t)c0 * F * 9, nullptr, nullptr,
                                  cfg->map_width);
          p->stem_tc_on = true;
        }
      }
    }
    for (int j = 0; j < S; ++j) {
      const int c2 = c0 << (S - j), ch = c2 / 2;
      DecLayers D;
      const float* w_s1 = src;
      D.s1 = p->make_layer(CONV3_S1, c2, c2, src);
      const float* w_up = src;
      D.up = p->make_layer(CONVT4_S2, c2, ch, src);
      const float* w_rs = src;
      D.rs = p->make_layer(CONVT4_S2, c2, ch, src);
      if (p->use_tc) {
        const size_t n1 = (size_t)c2 * c2 * 9, n2 = (size_t)ch * c2 * 16;
        D.s1_tc = p->make_tc(CONV3_S1, c2, c2, w_s1, w_s1 + n1, nullptr, nullptr, cfg->map_width >> (S - j));
        D.s2_tc = p->make_tc(CONVT4_S2, c2, ch, w_up, w_up + n2, w_rs, w_rs + n2, cfg->map_width >> (S - j));
      }
      D.eca = p->make_vec(k, src);
      p->dec.push_back(D);
    }
    if (p->use_tc) {
      std::vector<float> wt(9 * (size_t)c0);
      for (int ci = 0; ci < c0; ++ci)
        for (int t = 0; t < 9; ++t) {
          const float v = src[(size_t)ci * 9 + t];
          wt[(size_t)t * c0 + ci] = p->bf16 ? __bfloat162float(__float2bfloat16_rn(v)) : v;
        }
      p->head_wt = p->upload(wt);
      p->head_host = wt;  // [9][c0] for the constant-bank strip head
    }
    p->head = p->make_layer(CONV3_S1, c0, 1, src);
    STDA_CHECK((size_t)(src - blob) == n_floats, "internal: blob parse mismatch");
    *out = p.release();
  });
}

void stda_plan_destroy(stda_plan* plan) {
  if (!plan) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  delete plan;
  if (prev >= 0) cudaSetDevice(prev);
}

int stda_launches_per_forward(const stda_plan* plan) {
  if (!plan) return -1;
  if (plan->kind != 0) return 2;
  // tensor-core path: last gate fused in head; the stem fused into enc0.s1 when possible
  return (plan->use_tc ? 1 : 2) + 6 * plan->cfg.stages - (plan->stem_fused ? 1 : 0);
}

int stda_kernels_per_forward(const stda_plan* plan) {
  if (!plan) return -1;
  int n = stda_launches_per_forward(plan);
  if (plan->kind != 0 || !plan->use_tc) return n;
  // + the separate gate kernels of large maps (run_net_tc: precompute_gates)
  const stda_config& c = plan->cfg;
  int h = c.map_height, wd = c.map_width;
  for (int i = 0; i < c.stages; ++i) {
    tc::TcLayerDesc d2 = plan->enc[i].s2_tc;
    n += precompute_gates(tc::tc_plan(d2, 1, h, wd).items_per_image, d2.cout);
    h /= 2;
    wd /= 2;
  }
  for (int j = 0; j < c.stages; ++j) {
    tc::TcLayerDesc d2 = plan->dec[j].s2_tc;
    n += precompute_gates(tc::tc_plan(d2, 1, h, wd).items_per_image, d2.cout);
    h *= 2;
    wd *= 2;
  }
  return n;
}

size_t stda_workspace_bytes(const stda_plan* plan, int64_t batch) {
  if (!plan || plan->kind != 0 || batch < 0) return 0;
  return plan_ws(*plan, batch, nullptr).bytes;
}

int stda_forward(const stda_plan* plan, const float* x, float* y, int64_t batch, void* ws,
                 size_t ws_bytes, void* stream) {
  return guarded([&] {
    STDA_CHECK(plan && plan->kind == 0, "not a network plan");
    STDA_CHECK(batch >= 0, "negative batch");
    if (batch == 0) return;
    STDA_CHECK(x && y, "null tensor");
    const NetWs need = plan_ws(*plan, batch, nullptr);
    check_ws(plan, ws, ws_bytes, need.bytes);
    DeviceGuard g(plan->device);
    const stda_config& c = plan->cfg;
    const Src xs = plain_src(x, c.input_frames, c.map_height, c.map_width);
    run_net(*plan, xs, y, batch, plan_ws(*plan, batch, static_cast<char*>(ws)),
            static_cast<cudaStream_t>(stream));
  });
}

int stda_forward_profiled(const stda_plan* plan, const float* x, float* y, int64_t batch, void* ws,
                          size_t ws_bytes, void* stream, float* ms_per_launch, int32_t n) {
  return guarded([&] {
    STDA_CHECK(plan && plan->kind == 0, "not a network plan");
    STDA_CHECK(batch > 0 && x && y, "bad arguments");
    const int L = stda_launches_per_forward(plan);
    STDA_CHECK(ms_per_launch && n >= L, "ms_per_launch must hold launches_per_forward floats");
    const NetWs need = plan_ws(*plan, batch, nullptr);
    check_ws(plan, ws, ws_bytes, need.bytes);
    DeviceGuard g(plan->device);
    const stda_config& c = plan->cfg;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<cudaEvent_t> ev(L + 1);
    for (auto& e : ev) STDA_CUDA(cudaEventCreate(&e));
    Marks mk;
    mk.ev = &ev;
    run_net(*plan, plain_src(x, c.input_frames, c.map_height, c.map_width), y, batch,
            plan_ws(*plan, batch, static_cast<char*>(ws)), st, mk);
    STDA_CUDA(cudaEventSynchronize(ev[L]));
    for (int i = 0; i < L; ++i) STDA_CUDA(cudaEventElapsedTime(&ms_per_launch[i], ev[i], ev[i + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int stda_forward_launch_repeat(const stda_plan* plan, const float* x, float* y, int64_t batch, void* ws,
                               size_t ws_bytes, void* stream, int32_t slot, int32_t reps, float* ms_per_launch) {
  return guarded([&] {
    STDA_CHECK(plan && plan->kind == 0 && plan->use_tc, "not a tensor-core network plan");
    STDA_CHECK(batch > 0 && x && y && ms_per_launch && reps > 0, "bad arguments");
    STDA_CHECK(slot >= 0 && slot < stda_launches_per_forward(plan), "launch slot out of range");
    const NetWs need = plan_ws(*plan, batch, nullptr);
    check_ws(plan, ws, ws_bytes, need.bytes);
    DeviceGuard g(plan->device);
    const stda_config& c = plan->cfg;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Src xs = plain_src(x, c.input_frames, c.map_height, c.map_width);
    const NetWs w = plan_ws(*plan, batch, static_cast<char*>(ws));
    run_net(*plan, xs, y, batch, w, st);  // every intermediate of this input in place
    cudaEvent_t e0, e1;
    STDA_CUDA(cudaEventCreate(&e0));
    STDA_CUDA(cudaEventCreate(&e1));
    STDA_CUDA(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) {
      Marks mk;
      mk.only = slot;
      run_net(*plan, xs, y, batch, w, st, mk);
    }
    STDA_CUDA(cudaEventRecord(e1, st));
    STDA_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    STDA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_launch = ms / (float)reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

const char* stda_launch_names(const stda_plan* plan) {
  static thread_local std::string names;
  names = (plan && plan->kind == 0) ? launch_names(plan->cfg, plan->use_tc, plan->stem_fused) : std::string();
  return names.c_str();
}

int stda_forward_window(const stda_plan* plan, const float* frames, int64_t n_frames, float* y,
                        void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    STDA_CHECK(plan && plan->kind == 0, "not a network plan");
    const stda_config& c = plan->cfg;
    const int64_t B = n_frames - (c.input_frames - 1);
    if (B <= 0) return;
    STDA_CHECK(frames && y, "null tensor");
    const NetWs need = plan_ws(*plan, B, nullptr);
    check_ws(plan, ws, ws_bytes, need.bytes);
    DeviceGuard g(plan->device);
    const int64_t HW = (int64_t)c.map_height * c.map_width;
    // output b <-> t = b + F-1; channel ch reads frame t - ch
    Src xs;
    xs.x = frames + (int64_t)(c.input_frames - 1) * HW;
    xs.xb = HW;
    xs.xc = -HW;
    xs.C = c.input_frames;
    run_net(*plan, xs, y, B, plan_ws(*plan, B, static_cast<char*>(ws)),
            static_cast<cudaStream_t>(stream));
  });
}

int64_t stda_host_chunk(const stda_plan* plan, int64_t batch) {
  if (!plan || plan->kind != 0 || batch <= 0) return 0;
  const stda_config& c = plan->cfg;
  const int64_t per = (int64_t)c.input_frames * c.map_height * c.map_width * 4;
  // input bytes per pipelined chunk: 1/16 of the call's input, clamped to [16, 128] MB —
  // large chunks keep the per-forward efficiency of big batches (256^2 / 512^2 maps: 21 / 5
  // triplets per 16 MB chunk cost 10-15 % of e2e throughput), and 16 chunks keep the
  // exposed first copy-in / last copy-out small.  env STDA_HOST_CHUNK_MB fixes it (A/B).
  static const int64_t mb_env = [] {
    const char* e = std::getenv("STDA_HOST_CHUNK_MB");
    return e ? std::max<int64_t>(1, std::atoll(e)) : 0;
  }();
  const int64_t bytes = mb_env ? (mb_env << 20)
                               : std::min<int64_t>(128ll << 20, std::max<int64_t>(16ll << 20, batch * per / 16));
  const int64_t chunk = std::max<int64_t>(1, bytes / per);
  return std::min(batch, chunk);
}

size_t stda_host_workspace_bytes(const stda_plan* plan, int64_t chunk) {
  if (!plan || plan->kind != 0 || chunk <= 0) return 0;
  const stda_config& c = plan->cfg;
  const size_t HW = (size_t)c.map_height * c.map_width;
  return 2 * align_up(chunk * c.input_frames * HW * 4) + 2 * align_up(chunk * HW * 4) +
         plan_ws(*plan, chunk, nullptr).bytes;
}

namespace {
struct HostPipe {
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  HostPipe() {
    STDA_CUDA(cudaStreamCreateWithFlags(&copy_in, cudaStreamNonBlocking));
    STDA_CUDA(cudaStreamCreateWithFlags(&copy_out, cudaStreamNonBlocking));
    STDA_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    for (int s = 0; s < 2; ++s) {
      STDA_CUDA(cudaEventCreateWithFlags(&ev_in[s], cudaEventDisableTiming));
      STDA_CUDA(cudaEventCreateWithFlags(&ev_comp[s], cudaEventDisableTiming));
      STDA_CUDA(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
    }
  }
  ~HostPipe() {  // work already enqueued completes; handles are released afterwards
    if (copy_in) cudaStreamDestroy(copy_in);
    if (copy_out) cudaStreamDestroy(copy_out);
    for (cudaEvent_t e : {ev_start, ev_in[0], ev_in[1], ev_comp[0], ev_comp[1], ev_out[0], ev_out[1]})
      if (e) cudaEventDestroy(e);
  }
  HostPipe(const HostPipe&) = delete;
  HostPipe& operator=(const HostPipe&) = delete;
};

// One pipe per (host thread, device), created on the thread's first host-buffer call and
// reused by its later ones: creating and destroying two streams and seven events costs
// ~150-200 us per call, more than a batch-1 forward.  Calls of one thread are sequential and
// each ends with the copy-out stream drained, so a pipe is idle whenever its thread starts a
// new call; threads never share one (the plan stays immutable, concurrent calls on one plan
// with distinct workspaces never share a stream or an event).
HostPipe& thread_pipe(int device) {
  thread_local std::vector<std::pair<int, std::unique_ptr<HostPipe>>> pipes;
  for (auto& e : pipes)
    if (e.first == device) return *e.second;
  pipes.emplace_back(device, std::make_unique<HostPipe>());
  return *pipes.back().second;
}
}  // namespace

int stda_forward_host(const stda_plan* plan, const float* x_host, float* y_host, int64_t batch,
                      int64_t chunk, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    STDA_CHECK(plan && plan->kind == 0, "not a network plan");
    if (batch <= 0) return;
    STDA_CHECK(x_host && y_host, "null host buffer");
    STDA_CHECK(chunk >= 1, "chunk must be >= 1");
    chunk = std::min(chunk, batch);
    check_ws(plan, ws, ws_bytes, stda_host_workspace_bytes(plan, chunk));
    DeviceGuard g(plan->device);
    // copy streams and events belong to the calling thread (thread_pipe)
    HostPipe* p = &thread_pipe(plan->device);
    const stda_config& c = plan->cfg;
    const size_t HW = (size_t)c.map_height * c.map_width;
    const size_t in_tri = c.input_frames * HW, in_bytes = align_up(chunk * in_tri * 4),
                 out_bytes = align_up(chunk * HW * 4);
    char* base = static_cast<char*>(ws);
    float* d_in[2] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + in_bytes)};
    float* d_out[2] = {reinterpret_cast<float*>(base + 2 * in_bytes),
                       reinterpret_cast<float*>(base + 2 * in_bytes + out_bytes)};
    const NetWs nw = plan_ws(*plan, chunk, base + 2 * in_bytes + 2 * out_bytes);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    STDA_CUDA(cudaEventRecord(p->ev_start, st));
    STDA_CUDA(cudaStreamWaitEvent(p->copy_in, p->ev_start, 0));
    STDA_CUDA(cudaStreamWaitEvent(p->copy_out, p->ev_start, 0));
    // chunk sequence: a short first chunk (a quarter) when the call spans several, so the
    // first copy-in the forwards cannot overlap is short; then full chunks (env
    // STDA_HOST_RAMP=0: equal chunks, A/B timing)
    static const bool ramp_on = [] {
      const char* e = std::getenv("STDA_HOST_RAMP");
      return !(e && e[0] == '0');
    }();
    const int64_t first = ramp_on && batch > 2 * chunk ? std::max<int64_t>(1, chunk / 4) : chunk;
    const int64_t n_chunks = 1 + (batch - std::min(first, batch) + chunk - 1) / chunk;
    int64_t b0 = 0;
    for (int64_t k = 0; k < n_chunks; ++k) {
      const int s = (int)(k & 1);
      const int64_t nb = std::min(k == 0 ? first : chunk, batch - b0);
      if (k >= 2) STDA_CUDA(cudaStreamWaitEvent(p->copy_in, p->ev_comp[s], 0));
      STDA_CUDA(cudaMemcpyAsync(d_in[s], x_host + b0 * in_tri, nb * in_tri * 4,
                                cudaMemcpyHostToDevice, p->copy_in));
      STDA_CUDA(cudaEventRecord(p->ev_in[s], p->copy_in));
      STDA_CUDA(cudaStreamWaitEvent(st, p->ev_in[s], 0));
      if (k >= 2) STDA_CUDA(cudaStreamWaitEvent(st, p->ev_out[s], 0));
      run_net(*plan, plain_src(d_in[s], c.input_frames, c.map_height, c.map_width), d_out[s], nb, nw,
              st);
      STDA_CUDA(cudaEventRecord(p->ev_comp[s], st));
      STDA_CUDA(cudaStreamWaitEvent(p->copy_out, p->ev_comp[s], 0));
      STDA_CUDA(cudaMemcpyAsync(y_host + b0 * HW, d_out[s], nb * HW * 4, cudaMemcpyDeviceToHost,
                                p->copy_out));
      STDA_CUDA(cudaEventRecord(p->ev_out[s], p->copy_out));
      b0 += nb;
    }
    for (int s = 0; s < 2 && s < n_chunks; ++s) STDA_CUDA(cudaStreamWaitEvent(st, p->ev_out[s], 0));
    STDA_CUDA(cudaStreamSynchronize(p->copy_out));
  });
}

// ---- block level ------------------------------------------------------------------
int stda_block_plan_create(int32_t kind, int32_t channels, const float* blob, size_t n_floats,
                           int device, stda_plan** out) {
  return guarded([&] {
    STDA_CHECK(blob && out, "null argument");
    STDA_CHECK(kind == 0 || kind == 1, "kind must be 0 (encoder) or 1 (decoder)");
    STDA_CHECK(channels >= 1 && (kind == 0 || channels % 2 == 0), "bad channel count");
    const size_t c = channels;
    const size_t need = kind == 0 ? c * c * 9 + c + 2 * (2 * c * c * 9 + 2 * c)
                                  : c * c * 9 + c + 2 * ((c / 2) * c * 16 + c / 2);
    STDA_CHECK(n_floats == need, "block blob size mismatch");
    DeviceGuard g(device);
    auto p = std::make_unique<stda_plan>();
    p->kind = kind + 1;
    p->device = device;
    p->block_channels = channels;
    const float* src = blob;
    if (kind == 0) {
      EncLayers E;
      E.s1 = p->make_layer(CONV3_S1, channels, channels, src);
      E.dn = p->make_layer(CONV3_S2, channels, 2 * channels, src);
      E.rs = p->make_layer(CONV3_S2, channels, 2 * channels, src);
      p->enc.push_back(E);
    } else {
      DecLayers D;
      D.s1 = p->make_layer(CONV3_S1, channels, channels, src);
      D.up = p->make_layer(CONVT4_S2, channels, channels / 2, src);
      D.rs = p->make_layer(CONVT4_S2, channels, channels / 2, src);
      p->dec.push_back(D);
    }
    *out = p.release();
  });
}

size_t stda_block_workspace_bytes(const stda_plan* b, int64_t batch, int32_t h, int32_t w) {
  if (!b || b->kind == 0 || batch < 0) return 0;
  return align_up((size_t)batch * b->block_channels * h * w * sizeof(float));
}

int stda_block_forward(const stda_plan* b, const float* x, float* y, int64_t batch, int32_t h,
                       int32_t w, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    STDA_CHECK(b && b->kind != 0, "not a block plan");
    if (batch == 0) return;
    STDA_CHECK(x && y, "null tensor");
    STDA_CHECK(h > 0 && w > 0, "bad spatial size");
    if (b->kind == 1) STDA_CHECK(h % 2 == 0 && w % 2 == 0, "spatial dims must be even");
    check_ws(b, ws, ws_bytes, stda_block_workspace_bytes(b, batch, h, w));
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int C = b->block_channels;
    float* m = static_cast<float*>(ws);
    const Src xin = plain_src(x, C, h, w);
    const Src mixed = plain_src(m, C, h, w);
    if (b->kind == 1) {
      const EncLayers& E = b->enc[0];
      launch_conv(E.s1, nullptr, xin, nullptr, m, nullptr, batch, h, w, true, false, st);
      launch_conv(E.dn, &E.rs, mixed, &xin, y, nullptr, batch, h, w, true, false, st);
    } else {
      const DecLayers& D = b->dec[0];
      launch_conv(D.s1, nullptr, xin, nullptr, m, nullptr, batch, h, w, true, false, st);
      launch_conv(D.up, &D.rs, mixed, &xin, y, nullptr, batch, h, w, true, false, st);
    }
  });
}

int stda_debug_trace(void* dev_buf, int32_t launch_index) {
  return guarded([&] { tc::tc_debug_trace(dev_buf, launch_index); });
}

int stda_eca(const float* w_dev, int32_t k, const float* x, float* gates, float* y, int64_t batch,
             int32_t channels, int32_t h, int32_t w, void* stream) {
  return guarded([&] {
    STDA_CHECK(k >= 1 && k % 2 == 1, "ECA kernel size must be odd");
    if (batch == 0) return;
    STDA_CHECK(w_dev && x && gates, "null tensor");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int hw = h * w;
    launch_channel_sum(x, gates, batch, channels, hw, st);                  // gates <- sums
    launch_gate(gates, 1, w_dev, k, gates, batch, channels, hw, st);        // in place
    if (y) launch_scale(x, gates, y, batch, channels, hw, st);
  });
}

// ---- synthesiser --------------------------------------------------------------------
int stda_synth_frames(uint64_t seed, int32_t scene, int64_t seq, int64_t first_frame,
                      int64_t n_frames, int32_t h, int32_t w, float* out, void* stream) {
  return guarded([&] {
    STDA_CHECK(n_frames >= 0 && first_frame >= 0, "bad frame range");
    if (n_frames == 0) return;
    STDA_CHECK(out, "null output");
    STDA_CHECK(n_frames < (1ll << 31), "too many frames");
    launch_synth(seed, scene, seq, 0, first_frame, (int)n_frames, 0, n_frames, h, w, out,
                 static_cast<cudaStream_t>(stream));
  });
}

namespace {
size_t baseline_blob_floats(int kind, int h, int w, int hidden) {
  const size_t hw = (size_t)h * w, hd = hidden;
  if (kind == 0) return hd * hw + hd + hd * hd + hd + hw * hd + hw;
  return 32 * 9 + 32 + 64 * 32 * 9 + 64 + 32 * 64 * 16 + 32 + 1 * 32 * 16 + 1;
}
}  // namespace

int stda_baseline_plan_create(int32_t kind, int32_t h, int32_t w, int32_t hidden, const float* blob,
                              size_t n_floats, int device, stda_plan** out) {
  return guarded([&] {
    STDA_CHECK(blob && out, "null argument");
    STDA_CHECK(kind == 0 || kind == 1, "kind must be 0 (MLP) or 1 (CAE)");
    STDA_CHECK(h > 0 && w > 0 && (kind == 1 || hidden > 0), "bad baseline shape");
    STDA_CHECK(kind == 0 || (h % 4 == 0 && w % 4 == 0), "CAE needs h, w divisible by 4");
    STDA_CHECK(n_floats == baseline_blob_floats(kind, h, w, hidden), "baseline blob size mismatch");
    DeviceGuard g(device);
    auto p = std::make_unique<stda_plan>();
    p->kind = 3 + kind;
    p->device = device;
    p->bh = h;
    p->bw = w;
    p->hidden = hidden;
    const float* src = blob;
    if (kind == 0) {
      const size_t hw = (size_t)h * w;
      const size_t dims[3][2] = {{(size_t)hidden, hw}, {(size_t)hidden, (size_t)hidden}, {hw, (size_t)hidden}};
      for (int l = 0; l < 3; ++l) {
        const size_t nw = dims[l][0] * dims[l][1];
        p->lin_w[l] = p->upload(std::vector<float>(src, src + nw));
        src += nw;
        p->lin_b[l] = p->upload(std::vector<float>(src, src + dims[l][0]));
        src += dims[l][0];
      }
    } else {
      p->cae[0] = p->make_layer(CONV3_S1, 1, 32, src);
      p->cae[1] = p->make_layer(CONV3_S1, 32, 64, src);
      const std::vector<float> z1(32 * 64 * 16 + 32, 0.f), z2(32 * 16 + 1, 0.f);
      p->cae[2] = p->make_layer(CONVT4_S2, 64, 32, src);
      const float* zs = z1.data();
      p->cae[3] = p->make_layer(CONVT4_S2, 64, 32, zs);
      p->cae[4] = p->make_layer(CONVT4_S2, 32, 1, src);
      zs = z2.data();
      p->cae[5] = p->make_layer(CONVT4_S2, 32, 1, zs);
    }
    *out = p.release();
  });
}

size_t stda_baseline_workspace_bytes(const stda_plan* p, int64_t batch) {
  if (!p || batch < 0 || p->kind < 3) return 0;
  const size_t B = batch, hw = (size_t)p->bh * p->bw;
  if (p->kind == 3) {
    const int S = linear_splits((int)hw);
    return 2 * align_up(B * p->hidden * sizeof(float)) +
           (S > 1 ? align_up((size_t)S * B * p->hidden * sizeof(float)) : 0);
  }
  return align_up(B * 32 * hw * 4) + align_up(B * 32 * hw) + align_up(B * 64 * hw) + align_up(B * 64 * hw / 4) +
         align_up(B * 32 * hw);
}

int stda_baseline_forward(const stda_plan* p, const float* x, int32_t x_channels, float* y, int64_t batch,
                          void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    STDA_CHECK(p && p->kind >= 3, "not a baseline plan");
    STDA_CHECK(batch >= 0 && x_channels >= 1, "bad batch/channels");
    if (batch == 0) return;
    STDA_CHECK(x && y && ws, "null buffer");
    STDA_CHECK(ws_bytes >= stda_baseline_workspace_bytes(p, batch), "workspace too small");
    DeviceGuard g(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int H = p->bh, W = p->bw;
    const int64_t hw = (int64_t)H * W;
    char* base = static_cast<char*>(ws);
    size_t off = 0;
    auto take = [&](size_t nf) {
      float* r = reinterpret_cast<float*>(base + off);
      off += align_up(nf * sizeof(float));
      return r;
    };
    if (p->kind == 3) {  // frame t (channel 0) of each triplet, flattened
      float* h1 = take((size_t)batch * p->hidden);
      float* h2 = take((size_t)batch * p->hidden);
      const int S = linear_splits((int)hw);
      float* part = S > 1 ? take((size_t)S * batch * p->hidden) : nullptr;
      launch_linear(x, (int64_t)x_channels * hw, p->lin_w[0], p->lin_b[0], h1, (int)batch, p->hidden, (int)hw, true,
                    part, st);
      launch_linear(h1, p->hidden, p->lin_w[1], p->lin_b[1], h2, (int)batch, p->hidden, p->hidden, true, nullptr,
                    st);
      launch_linear(h2, p->hidden, p->lin_w[2], p->lin_b[2], y, (int)batch, (int)hw, p->hidden, false, nullptr, st);
      return;
    }
    float* a1 = take((size_t)batch * 32 * hw);
    float* p1 = take((size_t)batch * 32 * hw / 4);
    float* a2 = take((size_t)batch * 64 * hw / 4);
    float* p2 = take((size_t)batch * 64 * hw / 16);
    float* t1 = take((size_t)batch * 32 * hw / 4);
    Src in = plain_src(x, 1, H, W);
    in.xb = (int64_t)x_channels * hw;  // channel 0 of each triplet
    launch_conv(p->cae[0], nullptr, in, nullptr, a1, nullptr, batch, H, W, true, false, st);
    launch_maxpool2(a1, p1, batch * 32, H, W, st);
    const Src s1 = plain_src(p1, 32, H / 2, W / 2);
    launch_conv(p->cae[1], nullptr, s1, nullptr, a2, nullptr, batch, H / 2, W / 2, true, false, st);
    launch_maxpool2(a2, p2, batch * 64, H / 2, W / 2, st);
    const Src s2 = plain_src(p2, 64, H / 4, W / 4);
    launch_conv(p->cae[2], &p->cae[3], s2, &s2, t1, nullptr, batch, H / 4, W / 4, true, false, st);
    const Src s3 = plain_src(t1, 32, H / 2, W / 2);
    launch_conv(p->cae[4], &p->cae[5], s3, &s3, y, nullptr, batch, H / 2, W / 2, false, false, st);
  });
}

int stda_score(const void* clean, int32_t clean_kind, const float* test_db, int64_t n, int32_t P, int32_t Q,
               int32_t guard0, int32_t guard1, int32_t train0, int32_t train1, double alpha_obj, double alpha_det,
               int32_t margin, double* out, unsigned char* det_hits, void* stream) {
  return guarded([&] {
    STDA_CHECK(n >= 0 && P > 0 && Q > 0, "bad map count/shape");
    if (n == 0) return;
    STDA_CHECK(clean && test_db && out && det_hits, "null buffer");
    launch_score(clean, clean_kind, test_db, n, P, Q, guard0, guard1, train0, train1, alpha_obj, alpha_det, margin,
                 out, det_hits, static_cast<cudaStream_t>(stream));
  });
}

int stda_rd_frontend(const void* beat, int64_t n, int32_t N, int32_t M, int32_t P, int32_t Q,
                     const double* stats, int32_t clutter, int32_t layout, float* out, void* stream) {
  return guarded([&] {
    STDA_CHECK(n >= 0, "bad frame count");
    if (n == 0) return;
    STDA_CHECK(beat && out, "null buffer");
    launch_rd_frontend(static_cast<const float2*>(beat), n, N, M, P, Q, stats, clutter != 0, layout, out,
                       static_cast<cudaStream_t>(stream));
  });
}

int stda_denoise_epilogue(const float* y, float* out, int64_t batch, int32_t h, int32_t w, float scale,
                          float z_min, float std_, float mean, void* stream) {
  return guarded([&] {
    STDA_CHECK(batch >= 0 && h > 0 && w > 0, "bad epilogue shape");
    if (batch == 0) return;
    STDA_CHECK(y && out, "null buffer");
    launch_denoise_epilogue(y, out, batch, h, w, scale, z_min, std_, mean, static_cast<cudaStream_t>(stream));
  });
}

int stda_synth_triplets(uint64_t seed, int32_t scene, int64_t first_seq, int64_t batch,
                        int32_t frames, int32_t h, int32_t w, float* x, void* stream) {
  return guarded([&] {
    STDA_CHECK(batch >= 0 && frames >= 1, "bad batch/frames");
    if (batch == 0) return;
    STDA_CHECK(x, "null output");
    launch_synth(seed, scene, first_seq, 1, 0, frames, 1, batch * frames, h, w, x,
                 static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
