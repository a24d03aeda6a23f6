// tcgen05 implicit-GEMM convolution: host side (weight packing, tiling plan, launch).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tc_kernel.cuh"

namespace stda {
namespace tc {

using namespace detail;

namespace {

// ---- host helpers ------------------------------------------------------------------
uint16_t bf16_bits(float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  uint16_t r;
  std::memcpy(&r, &h, 2);
  return r;
}
float bf16_val(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// tap tables; wk = index into the canonical per-(co,ci) weight vector
struct HostTap {
  int acc, dy, dx, wk;
};

std::vector<HostTap> plane_taps(int mode, int pl) {
  std::vector<HostTap> t;
  if (mode == CONV_STEMT) return {{0, 0, 0, -1}};  // im2col: one unshifted A read per chunk
  if (mode == CONVT4_SP || mode == CONVT4_SPH)
    return {{0, 0, 0, -1}, {0, 0, 1, -1}, {0, 1, 0, -1}, {0, 1, 1, -1}};  // the 4 windows
  if (mode == CONV3_S1P) {
    // the plane's 4 shift groups (dy, dx = half-resolution shift; acc = first phase of the
    // run); only used for the staged position span (lo / hi) — packing is group-wise
    for (int gi = 0; gi < 4; ++gi) t.push_back({s1p_p0(pl, gi), s1p_dy(pl, gi), s1p_dx(pl, gi), -1});
    return t;
  }
  if (mode == CONV3_S1 || mode == CONV3_ROWS) {
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 3; ++kx) t.push_back({0, ky - 1, kx - 1, ky * 3 + kx});
  } else if (mode == CONV3_S2) {
    const int py = pl >> 1, px = pl & 1;
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 3; ++kx) {
        const int dy = ky - 1, dx = kx - 1;
        const int tpy = dy == 0 ? 0 : 1, tpx = dx == 0 ? 0 : 1;
        if (tpy != py || tpx != px) continue;
        t.push_back({0, dy == -1 ? -1 : 0, dx == -1 ? -1 : 0, ky * 3 + kx});
      }
  } else if (mode == CONVT4_HALF) {
    // pl = output row parity py: phases (py, px), shifts relative to the origin moved
    // down py rows; wk indexes the full 16-entry ConvT phase kernel
    const int py = pl;
    for (int px = 0; px < 2; ++px)
      for (int a = 0; a < 2; ++a)
        for (int bb = 0; bb < 2; ++bb) t.push_back({px, a - 1, px + bb - 1, (py * 2 + px) * 4 + a * 2 + bb});
  } else {
    for (int ph = 0; ph < 4; ++ph)
      for (int a = 0; a < 2; ++a)
        for (int bb = 0; bb < 2; ++bb) {
          const int py = ph >> 1, px = ph & 1;
          t.push_back({ph, py + a - 1, px + bb - 1, ph * 4 + a * 2 + bb});
        }
  }
  // the device's constexpr tables must agree with this host table
  for (size_t i = 0; i < t.size(); ++i)
    STDA_CHECK(t[i].dy == tap_dy(mode, mode == CONVT4_HALF ? 0 : pl, (int)i) &&
                   t[i].dx == tap_dx(mode, mode == CONVT4_HALF ? 0 : pl, (int)i) &&
                   t[i].acc == tap_acc(mode, (int)i) && (int)t.size() == ntaps(mode, pl),
               "internal: tap table mismatch");
  return t;
}

}  // namespace

bool sp_enabled() {  // env STDA_TC_SP=0: the 9-shift-group transposed conv (A/B timing)
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_SP");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Shifted-phase convs: 3 MMAs of width N per window (hi*hi, lo*hi, hi*lo into one
// accumulator) or the hi/lo concatenation (2 MMAs of width 2N, twice the TMEM columns).
// Measured at C2 (round 2): the full-phase conv (dec1.s2) 41.1 -> 32.8 us with 3 MMAs — half
// the accumulator columns give G = 2 tiles per item and half the epilogue's TMEM loads, which
// bound it — while the half-phase conv (dec0.s2) is faster with the concat (30.7 vs 35.6 us).
// env STDA_TC_SP3=0 / STDA_TC_SPH3=1 flip them (A/B timing).
bool sp3_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_SP3");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool sph3_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_SPH3");
    return e && e[0] == '1';
  }();
  return on;
}

bool half_t_enabled() {  // env STDA_TC_HALF=0 keeps 3-MMA full ConvT items (A/B timing)
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_HALF");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tc_supported(int mode, int cin, int cout) {
  if (mode == CONV_STEMT) return cin % 16 == 0 && cin >= 16 && cin <= 64 && cout == 16;
  if (mode == CONV3_S1P && cout > 32) return false;  // fp32 concat: 4 phases x 2N <= 256 per MMA
  return cin % 16 == 0 && cin >= 16 && cin <= 64 && (cout == 16 || cout == 32 || cout == 64);
}

// env STDA_TC_S1P=1: encoder stride-1 convs as CONV3_S1P over the phase planes.  Off by
// default: 1.7x fewer MMA cycles per output for enc0.s1, but at C2 enc0.s1 is bound by its
// HBM traffic and epilogue stores, not the MMA (41.0 -> 43.1 us; enc1.s1 28.7 -> 34.4 us).
bool s1p_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_S1P");
    return e && e[0] == '1';
  }();
  return on;
}

// env STDA_TC_ROWS=1: stride-1 layers over 128k-wide planes as row bands (CONV3_ROWS).
// Measured off by default: it cuts the MMA stream per output 1.65x, but these layers are
// bound by their operand fills and epilogue stores, not the MMA (enc0.s1 43.4 -> 45.4 us
// at C2, 2.01 -> 2.21 ms at C3; profiles/r1_rows_ab.txt).
bool rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_TC_ROWS");
    return e && e[0] == '1';
  }();
  return on;
}

void tc_pack_layer(TcLayerDesc& d, int mode, int cin, int cout, const float* w0, const float* w1,
                   bool bf16, std::vector<uint16_t>& packed, int plane_w) {
  STDA_CHECK(tc_supported(mode, cin, cout), "layer shape not supported by the tensor-core path");
  STDA_CHECK((mode == CONV3_S1 || mode == CONV3_S1P || mode == CONV_STEMT) == (w1 == nullptr),
             "S1 layers are single-source, S2/T dual");
  // stride-1 layers over planes whose width is a multiple of 128 run as row bands (one A
  // read per input row serves three dy taps) when three stacked tap blocks fit one MMA
  if (mode == CONV3_S1 && rows_enabled() && plane_w > 0 && plane_w % 128 == 0 && 3 * (bf16 ? 1 : 2) * cout <= 256)
    mode = CONV3_ROWS;
  std::memset(&d, 0, sizeof(d));
  // A dual ConvT whose 8 accumulators cannot take the hi/lo N-concat in two TMEM slots
  // runs as CONVT4_HALF: one output-row parity per work item (4 accumulators), so the
  // 2-MMA concat applies (fewer operand bytes than 3 MMAs per tap).
  const bool wide_t = mode == CONVT4_S2 && (w1 ? 2 : 1) * 4 * 2 * cout * 2 > 512;
  static const bool half_all = [] {  // env STDA_TC_HALF=2: every fp32 ConvT in half-phase items
    const char* e = std::getenv("STDA_TC_HALF");
    return e && e[0] == '2';
  }();
  // ... and over planes >= 256 wide: a full-ConvT item stages 128 + 2L + 2 positions per
  // chunk (three input rows), so at 256-wide planes the ring drops to one stage; half-phase
  // items stage 128 + L + 2 (measured C5 dec1.s2: 4.10 -> 3.04 ms)
  if (mode == CONVT4_S2 && !bf16 && half_t_enabled() && (wide_t || half_all || plane_w >= 256)) mode = CONVT4_HALF;
  // full transposed convs whose hi/lo-concatenated accumulators fit run with shifted phase
  // origins: 4 A windows per source and K chunk instead of 9 shift groups
  // (bf16: one pass, the four phase tiles of N columns; two TMEM slots need 2 x 4 x N <= 256)
  if (mode == CONVT4_S2 && sp_enabled() &&
      (bf16 ? (w1 ? 2 : 1) * 4 * cout <= 256 : (w1 ? 2 : 1) * 4 * 2 * cout * 2 <= 512))
    mode = CONVT4_SP;
  // ... and the half-phase items likewise (two px phases of one row parity per item)
  if (mode == CONVT4_HALF && sp_enabled() && (w1 ? 2 : 1) * 2 * 2 * cout * 2 <= 512) mode = CONVT4_SPH;
  const bool tmode = mode == CONVT4_S2 || mode == CONVT4_HALF || mode == CONVT4_SP || mode == CONVT4_SPH;
  d.mode = mode;
  d.n_src = w1 ? 2 : 1;
  d.cin = cin;
  d.cout = cout;
  d.n_planes = n_planes_of(mode);
  d.n_acc_src = nacc_src(mode);
  d.npass = bf16 ? 1 : 3;
  const int npassB = bf16 ? 1 : 2;
  const int wk_per = tmode ? 16 : 9;
  if (mode == CONV3_S1P) STDA_CHECK(!w1, "phase-plane conv is single-source");
  const int n_halves = mode == CONVT4_HALF ? 2 : 1;  // HALF: py = 0 taps, then py = 1 taps
  std::vector<std::vector<HostTap>> taps(d.n_planes * n_halves);
  for (int pl = 0; pl < d.n_planes * n_halves; ++pl) taps[pl] = plane_taps(mode, pl);
  for (int pl = 0; pl < d.n_planes; ++pl) {
    PlaneTaps& pt = d.planes[pl];
    pt.n = (int8_t)taps[pl].size();
    for (size_t t = 0; t < taps[pl].size(); ++t) {
      pt.acc[t] = (int8_t)taps[pl][t].acc;
      pt.dy[t] = (int8_t)taps[pl][t].dy;
      pt.dx[t] = (int8_t)taps[pl][t].dx;
    }
  }
  const int cgroups = cin / 16;
  const int n_chunks = d.n_planes * cgroups;
  STDA_CHECK(n_chunks <= kMaxChunks, "too many K chunks");
  packed.clear();
  d.chunk_off[0] = 0;
  const float* ws[2] = {w0, w1};
  // hi/lo N-concatenation (one A_hi read for hi*hi and hi*lo) when the doubled
  // accumulators still leave two TMEM slots at one M-tile per item
  const int n_acc = d.n_src * d.n_acc_src;
  static const bool s2_noconcat = [] {  // env STDA_TC_S2_NOCONCAT=1: 3-MMA stride-2 layers
    const char* e = std::getenv("STDA_TC_S2_NOCONCAT");
    return e && e[0] == '1';
  }();
  static const char* noconcat_env = std::getenv("STDA_TC_NOCONCAT");  // mode digits without concat (A/B)
  const bool noconcat_mode = noconcat_env && std::strchr(noconcat_env, '0' + mode) != nullptr;
  d.concat = !bf16 && n_acc * 2 * cout * 2 <= 512 && !(mode == CONV3_S2 && s2_noconcat) && !noconcat_mode;
  // per (src, tap): concat -> [kgrp 2][pass 2][n][8] (kgrp row block = [B_hi; B_lo], 2N rows)
  //                 else   -> [pass][kgrp 2][n][8]
  auto put = [&](const float* w, int n, int ci, int wk, int pass) {
    const float v = w[((size_t)n * cin + ci) * wk_per + wk];
    const float hi = bf16_val(v);
    packed.push_back(bf16_bits(pass == 0 ? v : v - hi));
  };
  if (mode == CONV_STEMT) {
    // canonical stem weights [co][F][3][3]; chunk f = frame f; per chunk the 4 stacked phase
    // tiles [kgrp 2][phase 4][pass][cout][8]: K element e of group kg is window pixel
    // (wy, wx) = (2kg + e/4, e%4), read by output phase (py, px) through tap
    // (ky, kx) = (wy - py, wx - px) when both lie in 0..2 (else a zero weight)
    const int F = cin / 16;
    for (int f = 0; f < F; ++f) {
      for (int kg = 0; kg < 2; ++kg)
        for (int ph = 0; ph < 4; ++ph)
          for (int pass = 0; pass < npassB; ++pass)
            for (int n = 0; n < cout; ++n)
              for (int e = 0; e < 8; ++e) {
                const int wy = 2 * kg + e / 4, wx = e % 4;
                const int ky = wy - (ph >> 1), kx = wx - (ph & 1);
                if (ky < 0 || ky > 2 || kx < 0 || kx > 2) {
                  packed.push_back(0);
                  continue;
                }
                const float v = w0[((size_t)n * F + f) * 9 + ky * 3 + kx];
                const float hi = bf16_val(v);
                packed.push_back(bf16_bits(pass == 0 ? v : v - hi));
              }
      d.chunk_off[f + 1] = (int64_t)packed.size() * 2;
    }
    d.concat = !bf16;
    return;
  }
  if (mode == CONVT4_SPH) {
    // per output-row parity py (a block of its own, TcLayerDesc::half_bytes), chunk, source and
    // window (a, b): the 2 stacked px tiles [kgrp 2][px 2][pass 2][cout][8]
    if (sph3_enabled()) d.concat = 0;
    for (int hv = 0; hv < 2; ++hv) {
      for (int c = 0; c < n_chunks; ++c) {
        const int cgi = c % cgroups;
        for (int s = 0; s < d.n_src; ++s)
          for (int w = 0; w < 4; ++w)
            for (int o = 0; o < 2 * 2 * npassB; ++o) {  // concat: (kg, px, pass); else (pass, kg, px)
              const int kg = d.concat ? o >> 2 : (o >> 1) & 1, px = d.concat ? (o >> 1) & 1 : o & 1;
              const int pass = d.concat ? o & 1 : o >> 2;
              for (int n = 0; n < cout; ++n)
                for (int e = 0; e < 8; ++e)
                  put(ws[s], n, cgi * 16 + kg * 8 + e, (hv * 2 + px) * 4 + (w >> 1) * 2 + (w & 1), pass);
            }
        if (hv == 0) d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
      }
    }
    d.half_bytes = d.chunk_off[n_chunks];
    return;
  }
  if (mode == CONVT4_SP) {
    // per chunk, per source and window (a, b): the 4 stacked phase tiles [kgrp 2][phase 4]
    // [pass 2][cout][8]; phase (py, px) reads window (a, b) through its sub-kernel tap (a, b)
    if (sp3_enabled() || bf16) d.concat = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const int cgi = c % cgroups;
      for (int s = 0; s < d.n_src; ++s)
        for (int w = 0; w < 4; ++w)
          for (int o = 0; o < 2 * 4 * npassB; ++o) {  // concat: (kg, ph, pass); else (pass, kg, ph)
            const int kg = d.concat ? o >> 3 : (o >> 2) & 1, ph = d.concat ? (o >> 1) & 3 : o & 3;
            const int pass = d.concat ? o & 1 : o >> 3;
            for (int n = 0; n < cout; ++n)
              for (int e = 0; e < 8; ++e) put(ws[s], n, cgi * 16 + kg * 8 + e, ph * 4 + (w >> 1) * 2 + (w & 1), pass);
          }
      d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
    }
    return;
  }
  if (mode == CONV3_S1P) {
    // per chunk (input plane, 16-channel group), per shift group gi: the stacked tiles
    // [kgrp 2][phase slot n][pass][cout][8]; tile j = output phase p0 + j reads input
    // plane (qy, qx) at shift (sy, sx) through the 3x3 tap dy = 2sy + qy - py,
    // dx = 2sx + qx - px (zero tile for a phase of the run that does not use the shift)
    // 3-MMA scheme (env STDA_TC_S1P3=1, A/B): per group [pass][kgrp 2][phase slot n][cout][8]
    static const bool s1p3 = [] {
      const char* e = std::getenv("STDA_TC_S1P3");
      return e && e[0] == '1';
    }();
    d.concat = !bf16 && !s1p3;
    std::vector<int> seen(36, 0);
    for (int c = 0; c < n_chunks; ++c) {
      const int pl = c / cgroups, cgi = c % cgroups, qy = pl >> 1, qx = pl & 1;
      for (int gi = 0; gi < 4; ++gi)
        for (int o = 0; o < 2 * s1p_n(pl, gi) * npassB; ++o) {
          const int nn = s1p_n(pl, gi);
          // concat: (kg, j, pass); 3-MMA: (pass, kg, j)
          const int kg = d.concat ? o / (nn * npassB) : (o / nn) % 2;
          const int j = d.concat ? (o / npassB) % nn : o % nn;
          const int pass = d.concat ? o % npassB : o / (2 * nn);
          const int acc = s1p_p0(pl, gi) + j, py = acc >> 1, px = acc & 1;
          const bool used = s1p_uses(pl, gi, acc);
          const int dy = 2 * s1p_dy(pl, gi) + qy - py, dx = 2 * s1p_dx(pl, gi) + qx - px;
          if (used) {
            STDA_CHECK(dy >= -1 && dy <= 1 && dx >= -1 && dx <= 1, "internal: phase-plane taps");
            if (cgi == 0 && kg == 0 && pass == 0) seen[acc * 9 + (dy + 1) * 3 + (dx + 1)]++;
          }
          for (int n = 0; n < cout; ++n)
            for (int e = 0; e < 8; ++e) {
              if (used) put(ws[0], n, cgi * 16 + kg * 8 + e, (dy + 1) * 3 + (dx + 1), pass);
              else packed.push_back(0);
            }
        }
      d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
    }
    for (int i = 0; i < 36; ++i) STDA_CHECK(seen[i] == 1, "internal: phase-plane products");
    STDA_CHECK(bf16 || 4 * 2 * cout <= 256, "phase-plane conv: stacked width");
    return;
  }
  if (mode == CONV3_ROWS) {
    // per chunk, per dx group: [kgrp 2][block dy = -1, 0, +1][pass hi(, lo)][cout][8]
    for (int c = 0; c < n_chunks; ++c) {
      for (int dx = -1; dx <= 1; ++dx)
        for (int kg = 0; kg < 2; ++kg)
          for (int dy = -1; dy <= 1; ++dy)
            for (int pass = 0; pass < npassB; ++pass)
              for (int n = 0; n < cout; ++n)
                for (int e = 0; e < 8; ++e) put(ws[0], n, c * 16 + kg * 8 + e, (dy + 1) * 3 + (dx + 1), pass);
      d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
    }
    return;
  }
  if (tmode && d.concat) {
    // shift groups (tc_kernel.cuh grouped_t): per (half, src, group) the stacked tiles
    // [kgrp 2][phase slot n][pass 2][cout][8]; zero tile for a phase not using the shift
    const int NG = ngroups(mode);
    // every (phase, tap) product exactly once
    std::vector<int> seen(16, 0);
    for (int g = 0; g < NG; ++g)
      for (int j = 0; j < grp_n(mode, g); ++j) {
        const int ph = grp_p0(mode, g) + j;
        const int py = mode == CONVT4_S2 ? ph >> 1 : 0, px = mode == CONVT4_S2 ? ph & 1 : ph;
        const int a = grp_dy(mode, g) - py + 1, b = grp_dx(mode, g) - px + 1;
        if (a >= 0 && a <= 1 && b >= 0 && b <= 1) seen[ph * 4 + a * 2 + b]++;
      }
    for (int i = 0; i < (mode == CONVT4_S2 ? 16 : 8); ++i) STDA_CHECK(seen[i] == 1, "internal: shift groups");
    for (int hv = 0; hv < n_halves; ++hv)
    for (int c = 0; c < n_chunks; ++c) {
      const int cgi = c % cgroups;
        for (int s = 0; s < d.n_src; ++s)
          for (int g = 0; g < NG; ++g)
            for (int kg = 0; kg < 2; ++kg)
              for (int j = 0; j < grp_n(mode, g); ++j) {
                const int ph = grp_p0(mode, g) + j;
                const int py = mode == CONVT4_S2 ? ph >> 1 : hv, px = mode == CONVT4_S2 ? ph & 1 : ph;
                const int a = grp_dy(mode, g) - (mode == CONVT4_S2 ? py : 0) + 1, b = grp_dx(mode, g) - px + 1;
                const bool used = a >= 0 && a <= 1 && b >= 0 && b <= 1;
                const int wk = (py * 2 + px) * 4 + a * 2 + b;
                for (int pass = 0; pass < 2; ++pass)
                  for (int n = 0; n < cout; ++n)
                    for (int e = 0; e < 8; ++e) {
                      if (used) put(ws[s], n, cgi * 16 + kg * 8 + e, wk, pass);
                      else packed.push_back(0);
                    }
              }
      if (hv == 0) d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
    }
    if (n_halves == 2) d.half_bytes = d.chunk_off[n_chunks];
    return;
  }
  for (int hv = 0; hv < n_halves; ++hv)
  for (int c = 0; c < n_chunks; ++c) {
    const int pl = c / cgroups, cgi = c % cgroups;
    for (int s = 0; s < d.n_src; ++s)
      for (const HostTap& t : taps[pl + hv]) {
        if (d.concat) {
          for (int kg = 0; kg < 2; ++kg)
            for (int pass = 0; pass < 2; ++pass)
              for (int n = 0; n < cout; ++n)
                for (int e = 0; e < 8; ++e) put(ws[s], n, cgi * 16 + kg * 8 + e, t.wk, pass);
        } else {
          for (int pass = 0; pass < npassB; ++pass)
            for (int kg = 0; kg < 2; ++kg)
              for (int n = 0; n < cout; ++n)
                for (int e = 0; e < 8; ++e) put(ws[s], n, cgi * 16 + kg * 8 + e, t.wk, pass);
        }
      }
    if (hv == 0) d.chunk_off[c + 1] = (int64_t)packed.size() * 2;
  }
  if (n_halves == 2) d.half_bytes = d.chunk_off[n_chunks];
}

namespace {
bool s1_env_set() { return std::getenv("STDA_TC_S1STAGES") != nullptr; }
int slots_cap() {  // env STDA_TC_SLOTS (A/B timing), default kMaxSlots
  static const int v = [] {
    const char* e = std::getenv("STDA_TC_SLOTS");
    return e ? std::max(1, std::min(kMaxSlots, std::atoi(e))) : kMaxSlots;
  }();
  return v;
}
}  // namespace

TcGeometry tc_plan(TcLayerDesc& d, int B, int H, int W, size_t extra_smem, bool resident_only) {
  TcGeometry g{};
  g.B = B;
  g.H = H;
  g.W = W;
  if (d.mode == CONV3_S2) {
    g.Hp = H / 2;
    g.Wp = W / 2;
    g.Ho = H / 2;
    g.Wo = W / 2;
  } else if (d.mode == CONV3_S1P || d.mode == CONV_STEMT) {  // half-res positions, full-res output
    g.Hp = H / 2;
    g.Wp = W / 2;
    g.Ho = H;
    g.Wo = W;
  } else if (d.mode == CONVT4_S2 || d.mode == CONVT4_HALF || d.mode == CONVT4_SP || d.mode == CONVT4_SPH) {
    g.Hp = H;
    g.Wp = W;
    g.Ho = 2 * H;
    g.Wo = 2 * W;
  } else {
    g.Hp = H;
    g.Wp = W;
    g.Ho = H;
    g.Wo = W;
  }
  g.L = g.Wp + 1;
  int span = 0;
  for (int pl = 0; pl < d.n_planes; ++pl) {
    PlaneTaps& pt = d.planes[pl];
    int lo = 1 << 30, hi = -(1 << 30);
    for (int t = 0; t < pt.n; ++t) {
      const int sft = pt.dy[t] * g.L + pt.dx[t];
      lo = std::min(lo, sft);
      hi = std::max(hi, sft);
    }
    STDA_CHECK(lo == plane_lo_a(d.mode, pl) * g.L + plane_lo_b(d.mode, pl), "internal: plane lo");
    pt.lo = (int16_t)lo;
    pt.hi = (int16_t)hi;
    span = std::max(span, hi - lo);
  }
  const int n_acc = d.n_src * d.n_acc_src;
  const int npassA = d.npass == 3 ? 2 : 1;
  if (d.mode == CONV3_ROWS) {
    // row bands of T output rows x 128 columns: the largest T with two TMEM slots and a
    // >= 2-deep ring, weights resident
    STDA_CHECK(g.Wp % 128 == 0, "row-band conv: plane width must be a multiple of 128");
    const int AW = d.cout * (d.concat ? 2 : 1);
    const uint32_t w_total = (uint32_t)d.chunk_off[d.cin / 16];
    const size_t fixed = 1024 + 80 + kEpiWarpsMax * 64 * sizeof(float);
    bool found = false;
    static const int t_cap = [] {  // env STDA_TC_ROWS_T: largest rows per item (A/B timing)
      const char* e = std::getenv("STDA_TC_ROWS_T");
      return e ? std::atoi(e) : 8;
    }();
    for (int T : {8, 4, 2}) {
      if (T > t_cap || g.Hp % T != 0 || T * AW * 2 > 512) continue;
      const int P8 = ((T + 2) * kRowsSL + 7) / 8 * 8;
      const uint32_t a_stage = (uint32_t)npassA * 2 * P8 * 16;
      const size_t w_res = (w_total + 127) / 128 * 128;
      int st = std::min(3, (int)(((size_t)kMaxSmem - fixed - w_res) / a_stage));
      if (st < 2) continue;
      g.G = T;
      g.P_max = P8;
      g.stages = st;
      g.slots = std::min(slots_cap(), 512 / (T * AW));
      g.a_stage_bytes = g.chunk_a_bytes = a_stage;
      g.b_stage_bytes = g.chunk_b_bytes = 0;
      g.resident = true;
      g.w_total = w_total;
      g.cps = 1;
      g.smem_bytes = (size_t)st * a_stage + w_res + fixed;
      int cols = 32;
      while (cols < g.slots * T * AW) cols *= 2;
      g.tmem_cols = cols;
      found = true;
      break;
    }
    STDA_CHECK(found, "row-band conv: no tiling fits");
    g.items_per_image = (g.Hp / g.G) * (g.Wp / 128);
    return g;
  }
  uint32_t b_stage = 0;
  for (int c = 0; c < d.n_planes * (d.cin / 16); ++c)
    b_stage = std::max<uint32_t>(b_stage, (uint32_t)(d.chunk_off[c + 1] - d.chunk_off[c]));
  const size_t fixed = 1024 + 80 + kEpiWarpsMax * 64 * sizeof(float) + extra_smem;
  const uint32_t w_total = (uint32_t)d.chunk_off[d.n_planes * (d.cin / 16)];
  const size_t w_res = (w_total + 127) / 128 * 128;
  // Prefer (1) a >= 2-deep smem pipeline, (2) two TMEM slots (the epilogue of item i
  // overlaps the MMAs of item i+1), (3) the largest G, (4) resident weights (loaded once
  // per CTA instead of once per work item); fall back step by step.
  bool ok = false;
  static const int pref_stages = [] {  // env STDA_TC_MINSTAGES: stage depth preferred over G
    const char* e = std::getenv("STDA_TC_MINSTAGES");
    return e ? std::max(2, std::min(kMaxStages, std::atoi(e))) : 2;
  }();
  const int pref = d.mode == CONV3_S2 ? pref_stages : 2;
  // env STDA_TC_GMAX=<m0><m1><m2><m3> (one digit per mode: S1 S2 T HALF): cap on the tiles
  // per item (A/B timing of load balance vs halo reuse)
  static const char* gmax_env = std::getenv("STDA_TC_GMAX");
  int gmax = gmax_env && (int)std::strlen(gmax_env) > d.mode ? gmax_env[d.mode] - '0' : 4;
  if ((d.mode == CONV3_S1 || d.mode == CONV3_S1P || d.mode == CONV_STEMT) && !gmax_env) {
    // load balance: the largest G that still gives every CTA >= 6 full items (fewer,
    // larger items leave the persistent CTAs with 2-4 rounds dominated by pipeline fill
    // and the last partial round).  Measured at C2 (B=64): enc0.s1 G=4, enc1.s1 / dec1.s1
    // G=2 (30.8 -> 29.5 us, 29.7 -> 28.0 us), dec0.s1 G=1 (27.6 -> 23.5 us).
    int dev = 0, sms = 148;
    STDA_CUDA(cudaGetDevice(&dev));
    STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    gmax = 1;
    for (int G : {4, 2}) {
      const int64_t full = (int64_t)B * ((int64_t)g.Hp * g.L / (G * 128));
      if (full >= 6 * (int64_t)sms) {
        gmax = G;
        break;
      }
    }
  }
  for (int pass = 0; pass < 4 && !ok; ++pass) {
    const int want_stages = pass == 0 ? pref : pass == 3 ? 1 : 2, want_slots = pass <= 1 ? 2 : 1;
    for (int G : {4, 2, 1}) {
      if (G > gmax && G > 1) continue;
      const int P8 = (G * 128 + span + 7) / 8 * 8;
      const uint32_t a_stage = (uint32_t)d.n_src * npassA * 2 * P8 * 16;
      const int acc_cols = G * n_acc * d.cout * (d.concat ? 2 : 1);
      if (acc_cols * want_slots > 512 || G * n_acc > 32) continue;
      for (bool resident : {true, false}) {
        if (resident_only && !resident) continue;
        int stages = 0;
        // measured: S1/T layers are slower beyond 3 stages; S2 layers (L2-fed) may go deeper
        static const int t_stages = [] {  // env STDA_TC_TSTAGES: ring depth cap of ConvT layers
          const char* e = std::getenv("STDA_TC_TSTAGES");
          return e ? std::max(1, std::min(kMaxStages, std::atoi(e))) : 3;
        }();
        static const int s1_stages = [] {  // env STDA_TC_S1STAGES: ring depth cap of stride-1 layers
          const char* e = std::getenv("STDA_TC_S1STAGES");
          return e ? std::max(1, std::min(kMaxStages, std::atoi(e))) : 3;
        }();
        const bool tmode = d.mode == CONVT4_S2 || d.mode == CONVT4_HALF || d.mode == CONVT4_SP || d.mode == CONVT4_SPH;
        // the phase-plane stride-1 conv (small resident weights) takes a 4th stage: enc0.s1
        // 39.2 -> 38.2 us at C2 (round 2); plain stride-1 layers stay at 3
        const int s1_cap = d.mode == CONV3_S1P && !s1_env_set() ? 4 : s1_stages;
        const int st_cap = d.mode == CONV3_S2 || d.mode == CONV_STEMT ? kMaxStages : tmode ? t_stages : s1_cap;
        for (int st = st_cap; st >= 1; --st) {
          const size_t need = resident ? (size_t)st * a_stage + w_res : (size_t)st * (a_stage + b_stage);
          if (need + fixed <= (size_t)kMaxSmem) {
            stages = st;
            break;
          }
        }
        if (stages < want_stages) continue;
        g.G = G;
        g.P_max = P8;
        g.stages = stages;
        // extra TMEM slots (free columns) absorb epilogue jitter: the MMA warp then rarely
        // waits for a slot
        g.slots = want_slots == 2 ? std::min(slots_cap(), 512 / acc_cols) : want_slots;
        g.a_stage_bytes = a_stage;
        g.b_stage_bytes = resident ? 0 : b_stage;
        g.resident = resident;
        g.w_total = w_total;
        g.smem_bytes =
            (resident ? (size_t)stages * a_stage + w_res : (size_t)stages * (a_stage + b_stage)) + fixed;
        int cols = 32;
        while (cols < g.slots * acc_cols) cols *= 2;
        g.tmem_cols = cols;
        ok = true;
        break;
      }
      if (ok) break;
    }
  }
  STDA_CHECK(ok, "tensor-core conv: no tiling fits shared memory");
  // Two K chunks per ring stage when they fit >= 2 stages: the MMA warp's per-stage
  // barrier wait / commit / descriptor setup (tensor-pipe idle time, the issue runs in
  // lockstep with execution) is paid once per two chunks
  g.cps = 1;
  g.chunk_a_bytes = g.a_stage_bytes;
  g.chunk_b_bytes = g.b_stage_bytes;
  {
    static const int cps_cap = [] {  // env STDA_TC_CPS=1: one chunk per stage (A/B timing)
      const char* e = std::getenv("STDA_TC_CPS");
      return e && e[0] == '1' ? 1 : 2;
    }();
    const int n_chunks = d.n_planes * (d.cin / 16);
    // measured: helps the transposed convs (dec0.s2 -4 %, dec1.s2 -1.5 %), not S1/S2
    const bool tmode = d.mode == CONVT4_S2 || d.mode == CONVT4_HALF || d.mode == CONVT4_SP || d.mode == CONVT4_SPH;
    if (cps_cap >= 2 && tmode && n_chunks % 2 == 0) {
      const size_t per = 2 * (size_t)g.a_stage_bytes + (g.resident ? 0 : 2 * (size_t)g.b_stage_bytes);
      const size_t base = (g.resident ? (size_t)((g.w_total + 127) / 128 * 128) : 0) + fixed;
      const int st2 = (int)std::min<size_t>((size_t)std::max(2, (g.stages + 1) / 2), ((size_t)kMaxSmem - base) / per);
      if (st2 >= 2) {
        g.cps = 2;
        g.stages = st2;
        g.a_stage_bytes = 2 * g.chunk_a_bytes;
        g.b_stage_bytes = g.resident ? 0 : 2 * g.chunk_b_bytes;
        g.smem_bytes = base + (size_t)st2 * per;
      }
    }
  }
  // SP: tile origins run from one row and column above the image (phase (0,0) at +L+1)
  const int positions = g.Hp * g.L + (d.mode == CONVT4_SP || d.mode == CONVT4_SPH ? g.L + 1 : 0);
  const bool halfm = d.mode == CONVT4_HALF || d.mode == CONVT4_SPH;
  g.items_per_image = cdiv(positions, g.G * 128) * (halfm ? 2 : 1);
  static const bool planlog = std::getenv("STDA_TC_PLANLOG") != nullptr;  // debug: print plans
  if (planlog)
    std::fprintf(stderr, "tc_plan mode %d cin %d cout %d grid %dx%d B %d: G %d stages %d cps %d slots %d resident %d "
                 "a_stage %u smem %zu items/img %d\n", d.mode, d.cin, d.cout, g.Hp, g.Wp, B, g.G, g.stages, g.cps,
                 g.slots, (int)g.resident, g.a_stage_bytes, g.smem_bytes, g.items_per_image);
  static const bool tail_last = [] {  // env STDA_TC_TAIL=0: image-major item order (A/B timing)
    const char* e = std::getenv("STDA_TC_TAIL");
    return !(e && e[0] == '0');
  }();
  g.tail = tail_last && positions % (g.G * 128) != 0 ? (halfm ? 2 : 1) : 0;
  return g;
}

namespace {
unsigned long long* g_trace_buf = nullptr;  // armed by tc_debug_trace, consumed by one launch
int g_trace_countdown = 0;
}  // namespace

void tc_debug_trace(void* dev_buf, int launch_index) {
  g_trace_buf = static_cast<unsigned long long*>(dev_buf);
  g_trace_countdown = launch_index;
}

namespace {
// frame rows one item stages: the s rows its positions [q0-L-1, q0+128G+L+1) touch (+1 each side)
int stem_xrows(int G, int L) { return (G * 128 + 2 * L + 1) / L + 2 + 2; }
size_t stem_extra_smem(int G, int L, int F, int W) {
  return 2 * ((size_t)F * stem_xrows(G, L) * W * 4) + 128;
}
}  // namespace

// ---- tensor-core stem (CONV_STEMT) --------------------------------------------------------
namespace {
// frame rows of one item: its half-resolution rows y_lo..y_hi -> frame rows 2y_lo-1 .. 2y_hi+2
int stemt_xrows(int G, int L) { return 2 * ((G * 128 + L - 2) / L) + 4; }
size_t stemt_extra_smem(int G, int L, int F, int W) { return 2 * ((size_t)F * stemt_xrows(G, L) * W * 4) + 128; }
}  // namespace

bool tc_stemt_ok(const TcStem& s, int H, int W) {
  // env STDA_STEM_TC=1 enables it.  Off by default: parity-green, but at C2 it runs 33 us
  // (CTA median) against the SIMT stem's ~27 us.  Ablations (tools/stemt_dbg.sh): without
  // epilogue stores 24.6 us, epilogue releasing slots only 15.7 us — the 67 MB of phase-plane
  // output leave the 8 epilogue warps at ~14 B/clk/SM against the ~21-25 B/clk/SM store
  // ceiling (tools/store_bench.cu), and the MMA waits on TMEM slots
  static const bool on = [] {
    const char* e = std::getenv("STDA_STEM_TC");
    return e && e[0] == '1';
  }();
  return on && s.F >= 1 && s.F <= kStemMaxF && s.x.xp == 1 && H % 2 == 0 && W % 4 == 0 && W >= 8 &&
         (reinterpret_cast<uintptr_t>(s.x.x) & 15) == 0 && s.x.xb % 4 == 0 && s.x.xc % 4 == 0 &&
         s.s_pp.base != nullptr && s.s_pp.C == kStemC && s.s_pp.planes == 4 &&
         stemt_extra_smem(2, W / 2 + 1, s.F, W) <= 96 * 1024;
}

TcGeometry tc_plan_stemt(TcLayerDesc& d, int B, int H, int W, int F) {
  STDA_CHECK(d.mode == CONV_STEMT, "internal: tensor-core stem plan");
  return tc_plan(d, B, H, W, stemt_extra_smem(2, W / 2 + 1, F, W), /*resident_only=*/true);
}

void tc_launch_stemt(const TcLayerDesc& d, const TcGeometry& g, const TcStem& s, const TcOut& out,
                     cudaStream_t st) {
  STDA_CHECK(tc_stemt_ok(s, g.H, g.W) && d.mode == CONV_STEMT, "tensor-core stem: unsupported input");
  STDA_CHECK(g.resident && g.cps == 1 && g.G <= 2, "tensor-core stem: plan");
  STDA_CHECK(out.mode == 2 && out.pl.L == g.L, "tensor-core stem: writes phase planes");
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.d = d;
  p.out = out;
  p.H = g.H;
  p.W = g.W;
  p.C = d.cin;
  p.Hp = g.Hp;
  p.Wp = g.Wp;
  p.L = g.L;
  p.L_mul = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)g.L - 1) / (uint64_t)g.L);
  STDA_CHECK((uint64_t)g.items_per_image * g.G * 128 * (uint64_t)g.L < ((uint64_t)1 << 32),
             "tensor-core stem: map too large for the position decode");
  p.Ho = g.Ho;
  p.Wo = g.Wo;
  p.G = g.G;
  p.stages = g.stages;
  p.slots = g.slots;
  p.items_per_image = g.items_per_image;
  p.total_items = g.B * g.items_per_image;
  p.tail = g.tail;
  p.rev = 0;
  p.P_max = g.P_max;
  STDA_CHECK(g.P_max == g.G * 128, "internal: tensor-core stem stages exactly its positions");
  p.a_stage_bytes = g.a_stage_bytes;
  p.b_stage_bytes = g.b_stage_bytes;
  p.cps = 1;
  p.chunk_a_bytes = g.chunk_a_bytes;
  p.chunk_b_bytes = g.chunk_b_bytes;
  p.resident = 1;
  p.w_total = g.w_total;
  p.slot_cols = (uint32_t)(g.G * 4 * d.cout * (d.concat ? 2 : 1));
  p.tmem_cols = (uint32_t)g.tmem_cols;
  p.relu0 = 1;
  p.sx = s.x.x;
  p.sxb = s.x.xb;
  p.sxc = s.x.xc;
  p.sF = s.F;
  p.stem_xrows = stemt_xrows(g.G, g.L);
  p.stem_xstage = (uint32_t)((size_t)s.F * p.stem_xrows * g.W * 4);
  STDA_CHECK(stemt_extra_smem(g.G, g.L, s.F, g.W) <= stemt_extra_smem(2, g.L, s.F, g.W), "internal: stem ring");
  if (g_trace_buf != nullptr && g_trace_countdown-- == 0) {
    p.trace = g_trace_buf;
    g_trace_buf = nullptr;
    if (const char* e = std::getenv("STDA_TC_DBG")) p.dbg = std::atoi(e);
  }
  if (p.total_items == 0) return;
  int dev = 0, sms = 148;
  STDA_CUDA(cudaGetDevice(&dev));
  STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::min(p.total_items, sms);
  const int npm = d.npass == 1 ? kNpmBf16 : kNpmConcat;
  dispatch_stemt(npm, g.G, p, grid, g.smem_bytes, st);
}

// ---- gate-on-load stride-1 conv ---------------------------------------------------------------
// env STDA_GATEIN=1 enables it.  Off by default: bitwise-identical outputs, but at C2 the
// builder warps (6 warps beside the MMA / epilogue roles, 1.5x halo positions per item)
// form a K chunk every ~6k cycles against 1.6k of MMA: enc1.s1 62 us vs enc0.gate + enc1.s1
// 47.8 us, dec1.s1 57 us vs 37.5 us
bool gatein_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STDA_GATEIN");
    return e && e[0] == '1';
  }();
  return on;
}

bool tc_gatein_ok(const TcLayerDesc& d, const TcGateIn& gi, int H, int W) {
  return gatein_enabled() && d.mode == CONV3_S1 && d.n_src == 1 && d.cin % 16 == 0 && gi.x && gi.gates &&
         (reinterpret_cast<uintptr_t>(gi.x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gi.gates) & 15) == 0 &&
         gi.out_pl.base && gi.out_pl.planes == 1 && gi.out_pl.L == W + 1 && gi.out_pl.C == d.cin &&
         (!gi.skip.base || (gi.skip.planes == 1 && gi.skip.L == W + 1 && gi.skip.C == d.cin)) &&
         (!gi.out_pp.base || (gi.out_pp.planes == 4 && H % 2 == 0 && W % 2 == 0 && gi.out_pp.C == d.cin));
}

namespace {
// x ring stage of a gate-in item: the staged rows of one chunk plane (64 B per pixel) and the
// skip's staged positions per (pass, cg8) block
int gatein_xrows(int G, int L) { return (G * 128 + 2 * L + 1) / L + 2; }
uint32_t gatein_skip_off(int G, int L, int W) { return ((uint32_t)gatein_xrows(G, L) * W * 64 + 127) / 128 * 128; }
uint32_t gatein_xstage(int G, int L, int W, bool skip, int np) {
  const uint32_t P = (uint32_t)(G * 128 + 2 * L + 2);
  return gatein_skip_off(G, L, W) + (skip ? (uint32_t)np * 2 * P * 16 : 0u);
}
}  // namespace

TcGeometry tc_plan_gatein(TcLayerDesc& d, int B, int H, int W, const TcGateIn& gi) {
  const int np = d.npass == 3 ? 2 : 1, L = W + 1;
  const bool skip = gi.skip.base != nullptr;
  // reserve the x ring for the tile count the plain plan picks; accept when the plan with the
  // reservation does not pick more tiles per item than reserved for
  const TcGeometry g0 = tc_plan(d, B, H, W, 0, true);
  // the deepest x ring (4..2 stages) that leaves the plain plan's tile count and ring
  for (int nx = 4; nx >= 2; --nx) {
    const size_t extra = nx * (size_t)gatein_xstage(g0.G, L, W, skip, np) + 128;
    TcLayerDesc dd = d;
    TcGeometry g;
    try {
      g = tc_plan(dd, B, H, W, extra, true);
    } catch (const Error&) {
      continue;
    }
    if (g.G == g0.G && (g.stages >= std::min(g0.stages, 3) || nx == 2)) {
      d = dd;
      g.gx_nst = nx;
      return g;
    }
  }
  STDA_CHECK(false, "gate-in conv: no tiling fits shared memory");
  return g0;
}

bool tc_gatein_fits(const TcLayerDesc& d, int B, int H, int W, const TcGateIn& gi) {
  try {
    TcLayerDesc dd = d;
    tc_plan_gatein(dd, B, H, W, gi);
    return true;
  } catch (const Error&) {
    return false;
  }
}

void tc_launch_gatein(const TcLayerDesc& d, const TcGeometry& g, const TcGateIn& gi, const TcOut& out,
                      cudaStream_t st, bool rev) {
  STDA_CHECK(tc_gatein_ok(d, gi, g.H, g.W), "gate-in conv: unsupported layer / input");
  STDA_CHECK(g.resident && g.cps == 1, "gate-in conv: plan");
  STDA_CHECK(g.P_max >= g.G * 128 + 2 * g.L + 2, "internal: gate-in staged span");
  STDA_CHECK(gi.out_pl.np == (d.npass == 3 ? 2 : 1), "gate-in conv: plane precision");
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.d = d;
  p.out = out;
  p.H = g.H;
  p.W = g.W;
  p.C = d.cin;
  p.Hp = g.Hp;
  p.Wp = g.Wp;
  p.L = g.L;
  p.L_mul = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)g.L - 1) / (uint64_t)g.L);
  STDA_CHECK((uint64_t)(g.items_per_image * g.G * 128 + 2 * g.L) * (uint64_t)g.L < ((uint64_t)1 << 32),
             "gate-in conv: map too large for the position decode");
  p.Ho = g.Ho;
  p.Wo = g.Wo;
  p.G = g.G;
  p.stages = g.stages;
  p.slots = g.slots;
  p.items_per_image = g.items_per_image;
  p.total_items = g.B * g.items_per_image;
  p.tail = g.tail;
  static const bool rev_on = [] {
    const char* e = std::getenv("STDA_TC_REV");
    return !(e && e[0] == '0');
  }();
  p.rev = rev && rev_on ? 1 : 0;
  p.P_max = g.P_max;
  p.a_stage_bytes = g.a_stage_bytes;
  p.b_stage_bytes = g.b_stage_bytes;
  p.cps = 1;
  p.chunk_a_bytes = g.chunk_a_bytes;
  p.chunk_b_bytes = g.chunk_b_bytes;
  p.resident = 1;
  p.w_total = g.w_total;
  p.slot_cols = (uint32_t)(g.G * d.cout * (d.concat ? 2 : 1));
  p.tmem_cols = (uint32_t)g.tmem_cols;
  p.relu0 = 1;
  p.gx = gi.x;
  p.gates = gi.gates;
  p.stem_xstage = gatein_xstage(g.G, g.L, g.W, gi.skip.base != nullptr, gi.out_pl.np);
  p.gx_skip_off = gatein_skip_off(g.G, g.L, g.W);
  p.gx_nst = g.gx_nst;
  STDA_CHECK(p.gx_nst >= 2 && p.gx_nst <= 4, "internal: gate-in x ring");
  p.gskip = gi.skip;
  p.gpl = gi.out_pl;
  p.gpp = gi.out_pp;
  if (g_trace_buf != nullptr && g_trace_countdown-- == 0) {
    p.trace = g_trace_buf;
    g_trace_buf = nullptr;
    if (const char* e = std::getenv("STDA_TC_DBG")) p.dbg = std::atoi(e);
  }
  if (p.total_items == 0) return;
  int dev = 0, sms = 148;
  STDA_CUDA(cudaGetDevice(&dev));
  STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::min(p.total_items, sms);
  const int npm = d.npass == 1 ? kNpmBf16 : (d.concat ? kNpmConcat : kNpm3);
  STDA_CHECK(npm != kNpm3, "gate-in conv: 3-MMA scheme not instantiated");
  dispatch_gatein(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
}

bool tc_stem_fusable(const TcLayerDesc& d1, const TcStem& s, int H, int W) {
  static const bool on = [] {
    const char* e = std::getenv("STDA_STEM_FUSED");
    return e && e[0] == '1';
  }();
  return on && s.canon && d1.mode == CONV3_S1 && d1.cin == kStemC && d1.cout == kStemC &&
         s.F >= 1 && s.F <= kStemMaxF && s.x.xp == 1 && W % 4 == 0 && W <= 128 && H >= 2 &&
         (reinterpret_cast<uintptr_t>(s.x.x) & 15) == 0 && s.x.xb % 4 == 0 && s.x.xc % 4 == 0 &&
         s.s_pp.base != nullptr && s.s_pp.C == kStemC;
}

TcGeometry tc_plan_stem(TcLayerDesc& d1, int B, int H, int W, int F) {
  return tc_plan(d1, B, H, W, stem_extra_smem(4, W + 1, F, W), /*resident_only=*/true);
}

void tc_launch_stem(const TcLayerDesc& d, const TcGeometry& g, const TcStem& s, const TcOut& out,
                    cudaStream_t st, bool rev) {
  STDA_CHECK(tc_stem_fusable(d, s, g.H, g.W), "fused stem: unsupported layer / input");
  STDA_CHECK(g.resident, "fused stem: weights must be resident");
  STDA_CHECK(out.mode == 2, "fused stem: enc0.s1 writes phase planes");
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.d = d;
  p.out = out;
  p.H = g.H;
  p.W = g.W;
  p.C = d.cin;
  p.Hp = g.Hp;
  p.Wp = g.Wp;
  p.L = g.L;
  p.L_mul = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)g.L - 1) / (uint64_t)g.L);
  STDA_CHECK((uint64_t)g.items_per_image * g.G * 128 * (uint64_t)g.L < ((uint64_t)1 << 32),
             "fused stem: map too large for the position decode");
  p.Ho = g.Ho;
  p.Wo = g.Wo;
  p.G = g.G;
  p.stages = g.stages;
  p.slots = g.slots;
  p.items_per_image = g.items_per_image;
  p.total_items = g.B * g.items_per_image;
  p.tail = g.tail;
  static const bool rev_on = [] {
    const char* e = std::getenv("STDA_TC_REV");
    return !(e && e[0] == '0');
  }();
  p.rev = rev && rev_on ? 1 : 0;
  p.P_max = g.P_max;
  p.a_stage_bytes = g.a_stage_bytes;
  p.b_stage_bytes = g.b_stage_bytes;
  p.cps = g.cps;
  STDA_CHECK(g.cps == 1, "fused stem: one K chunk per stage");
  p.chunk_a_bytes = g.chunk_a_bytes;
  p.chunk_b_bytes = g.chunk_b_bytes;
  p.resident = 1;
  p.w_total = g.w_total;
  p.slot_cols = (uint32_t)(g.G * d.n_src * d.n_acc_src * d.cout * (d.concat ? 2 : 1));
  p.tmem_cols = (uint32_t)g.tmem_cols;
  p.relu0 = 1;
  // the stem
  p.sx = s.x.x;
  p.sxb = s.x.xb;
  p.sxc = s.x.xc;
  p.sF = s.F;
  p.stem_xrows = stem_xrows(g.G, g.L);
  p.stem_xstage = (uint32_t)((size_t)s.F * p.stem_xrows * g.W * 4);
  STDA_CHECK(stem_extra_smem(g.G, g.L, s.F, g.W) <= stem_extra_smem(4, g.L, s.F, g.W), "internal: stem ring");
  p.s_pl = s.s_pl;
  p.s_has_pl = s.has_pl ? 1 : 0;
  p.s_pp = s.s_pp;
  for (int co = 0; co < kStemC; ++co) {
    for (int ci = 0; ci < s.F; ++ci)
      for (int t = 0; t < 9; ++t) p.stem_w[(ci * 9 + t) * kStemC + co] = s.canon[((size_t)co * s.F + ci) * 9 + t];
    p.stem_b[co] = s.canon[(size_t)kStemC * s.F * 9 + co];
  }
  if (g_trace_buf != nullptr && g_trace_countdown-- == 0) {
    p.trace = g_trace_buf;
    g_trace_buf = nullptr;
    if (const char* e = std::getenv("STDA_TC_DBG")) p.dbg = std::atoi(e);
  }
  if (p.total_items == 0) return;
  int dev = 0, sms = 148;
  STDA_CUDA(cudaGetDevice(&dev));
  STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::min(p.total_items, sms);
  const int npm = d.npass == 1 ? kNpmBf16 : (d.concat ? kNpmConcat : kNpm3);
  dispatch_stem(npm, g.G, p, grid, g.smem_bytes, st);
}

void tc_launch(const TcLayerDesc& d, const TcGeometry& g, const PlBuf& src0, const PlBuf* src1,
               const TcOut& out, bool relu0, cudaStream_t st, bool rev) {
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.d = d;
  p.src[0] = src0;
  if (src1) p.src[1] = *src1;
  STDA_CHECK((src1 != nullptr) == (d.n_src == 2), "source count mismatch");
  STDA_CHECK(src0.L == g.L && (!src1 || src1->L == g.L), "operand plane geometry mismatch");
  STDA_CHECK(src0.np == (d.npass == 3 ? 2 : 1), "operand plane precision mismatch");
  STDA_CHECK((d.mode == CONV3_S2 || d.mode == CONV3_S1P) == (src0.planes == 4),
             "stride-2 and phase-plane convs read phase planes");
  STDA_CHECK(d.mode != CONV3_S1P || out.mode == 2, "phase-plane conv writes phase planes");
  p.out = out;
  p.H = g.H;
  p.W = g.W;
  p.C = d.cin;
  p.Hp = g.Hp;
  p.Wp = g.Wp;
  p.L = g.L;
  p.L_mul = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)g.L - 1) / (uint64_t)g.L);
  STDA_CHECK((uint64_t)g.items_per_image * g.G * 128 * (uint64_t)g.L < ((uint64_t)1 << 32),
             "tensor-core conv: map too large for the position decode");
  p.Ho = g.Ho;
  p.Wo = g.Wo;
  p.G = g.G;
  p.stages = g.stages;
  p.slots = g.slots;
  p.items_per_image = g.items_per_image;
  p.total_items = g.B * g.items_per_image;
  p.tail = g.tail;
  static const bool rev_on = [] {  // env STDA_TC_REV=0: every launch walks images first to last
    const char* e = std::getenv("STDA_TC_REV");
    return !(e && e[0] == '0');
  }();
  p.rev = rev && rev_on ? 1 : 0;
  p.P_max = g.P_max;
  p.a_stage_bytes = g.a_stage_bytes;
  p.b_stage_bytes = g.b_stage_bytes;
  p.cps = g.cps;
  p.chunk_a_bytes = g.chunk_a_bytes;
  p.chunk_b_bytes = g.chunk_b_bytes;
  p.resident = g.resident ? 1 : 0;
  p.w_total = g.w_total;
  p.slot_cols = (uint32_t)(g.G * d.n_src * d.n_acc_src * d.cout * (d.concat ? 2 : 1));
  p.tmem_cols = (uint32_t)g.tmem_cols;
  p.relu0 = relu0 ? 1 : 0;
  {
    static const int early = [] {
      const char* e = std::getenv("STDA_PDL_EARLY");
      return e ? std::atoi(e) : 0;  // measured: early trigger costs ~1% (co-resident waiters)
    }();
    p.early_trigger = early;
  }
  {
    // second producer warp (tc_kernel.cuh kProd2), measured on B200: C2 enc1.s2 32.7 -> 28.2 us
    // with it, every other C2 layer 0.2-1.8 us slower; C3 (B = 1024, 256^2) enc1.s2 1880 ->
    // 1567 us, dec0.s2 2120 -> 1898 us, enc0.s2 1955 -> 1857 us, stride-1 layers +-3 %; C5
    // neutral.  So: the stride-2 conv with 64 output channels always, the other stride-2 /
    // half-phase transposed convs on long launches (>= 32 items per CTA).
    // env STDA_TC_PROD2=1 / 0 forces it on / off everywhere
    static const int prod2 = [] {
      const char* e = std::getenv("STDA_TC_PROD2");
      return e ? std::atoi(e) : -1;
    }();
    const bool s2_like = d.mode == CONV3_S2 || d.mode == CONVT4_SPH;
    p.prod2 = prod2 >= 0 ? prod2
                         : ((d.mode == CONV3_S2 && d.cout == 64) || (s2_like && p.total_items >= 32 * 148) ? 1 : 0);
  }
  if (g_trace_buf != nullptr && g_trace_countdown-- == 0) {
    p.trace = g_trace_buf;
    g_trace_buf = nullptr;
    if (const char* e = std::getenv("STDA_TC_DBG")) p.dbg = std::atoi(e);  // traced launch only
  }
  if (p.total_items == 0) return;
  int dev = 0, sms = 148;
  STDA_CUDA(cudaGetDevice(&dev));
  STDA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = std::min(p.total_items, sms);
  // HALF: an even grid keeps every CTA on items of one py (items alternate py), so each
  // CTA loads one weight block (TcLayerDesc::half_bytes)
  if (d.mode == CONVT4_HALF || d.mode == CONVT4_SPH) grid &= ~1;
  const int npm = d.npass == 1 ? kNpmBf16 : (d.concat ? kNpmConcat : kNpm3);
  STDA_CHECK(d.cout == 16 || d.cout == 32 || d.cout == 64, "unsupported cout for the tensor-core path");
  STDA_CHECK(g.G == 1 || g.G == 2 || g.G == 4 || (d.mode == CONV3_ROWS && g.G == 8), "unsupported tile count per item");
  switch (d.mode) {
    case CONV3_S1: return dispatch_s1(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONV3_ROWS: return dispatch_rows(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONV3_S1P: return dispatch_s1p(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONV3_S2: return dispatch_s2(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONVT4_HALF:
      STDA_CHECK(out.mode == 0, "half-phase ConvT writes NHWC fp32");
      return dispatch_th(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONVT4_SP: return dispatch_sp(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    case CONVT4_SPH: return dispatch_sph(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
    default: return dispatch_t(d.cout, npm, g.G, p, grid, g.smem_bytes, st);
  }
}

}  // namespace tc
}  // namespace stda
