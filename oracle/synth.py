"""numpy restatement of the seeded RD-map generator — TEST INFRASTRUCTURE ONLY.

BASELINE.json's generator is not part of the reference (SURVEY §8(d) "Synthetic
inputs"); the product generator is `paper_2307_09063_b200/csrc/synth.cu`.  This file
restates the same specification on the host so that

* `bench.py --impl reference` can build its inputs without touching the product
  package or its shared library, and
* `tests/test_oracle_synth.py` / `tests/test_gpu_synth.py` can check the GPU kernel
  against an independent implementation.

Specification: per frame, complex Gaussian receiver noise (sigma = 1,
rdlab `signal_model.py:263-266` convention) with the noise sigma of 1–3 (dense: 1–5)
random Doppler bands raised by 5–20 dB, plus 1–5 (dense: 10–20) point targets of
10–30 dB drifting by v in {-1,0,1}^2 bins per frame (closed form, like rdlab
`dataset.py:228-241`), then 20*log10(|z| + 1e-12) (`rd_pipeline.py:22-23`) and a
per-frame min-max to [0, 1].  Randomness: Philox4x32-10 keyed by (seed, scene),
counter (purpose | element << 2, seq lo, seq hi, frame) — so a frame depends only on
(seed, scene, seq, frame, H, W).

Arithmetic is float32 in the kernel's operation order; the kernel's fused
multiply-adds are reproduced exactly (float64 product + add, one rounding).  The
transcendental functions (log, sincos, log10, exp10) are libm's, so the result
matches the GPU to a few float32 ulps, not bitwise.
"""

from __future__ import annotations

import numpy as np

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
K_SEQ, K_FRAME, K_NOISE = 1, 2, 3
F32 = np.float32


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10 (Salmon et al., SC'11); arrays of uint32 counters."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint32) for v in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0, k1 = np.uint32(k0), np.uint32(k1)
    for _ in range(10):
        p0 = c0.astype(np.uint64) * _M0
        p1 = c2.astype(np.uint64) * _M1
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _MASK).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _MASK).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        with np.errstate(over="ignore"):
            k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def make_key(seed: int, scene: int):
    k0 = (seed & 0xFFFFFFFF) ^ 0x5354DA00
    k1 = ((seed >> 32) & 0xFFFFFFFF) ^ ((scene * 0x9E3779B9) & 0xFFFFFFFF)
    return k0, k1


def u01(v) -> np.ndarray:
    """(0, 1): ((v >> 8) + 0.5f) * 2^-24 in float32, as the kernel computes it."""
    v = np.asarray(v, dtype=np.uint32)
    return ((v >> np.uint32(8)).astype(F32) + F32(0.5)) * F32(1.0 / 16777216.0)


def _fma(a, b, c) -> np.ndarray:
    """fmaf(a, b, c) for float32 inputs: exact in float64 for these operand widths."""
    return (np.float64(a) * np.asarray(b, np.float64) + np.float64(c)).astype(F32)


def _draw(key, purpose, seq, frame, elem):
    elem = np.asarray(elem, dtype=np.uint64)
    c0 = (np.uint64(purpose) | (elem << np.uint64(2))) & _MASK
    s = int(seq)
    return philox4x32_10(c0.astype(np.uint32), s & 0xFFFFFFFF, (s >> 32) & 0xFFFFFFFF,
                         int(frame) & 0xFFFFFFFF, *key)


def frame(seed: int, scene: int, seq: int, frame_idx: int, H: int, W: int) -> np.ndarray:
    """One normalised [H, W] float32 frame (row h = Doppler bin, column w = range bin)."""
    key = make_key(seed, scene)
    r = _draw(key, K_SEQ, seq, 0, 0)
    ux = u01(r[0])
    n_t = 1 + int(ux * F32(5.0)) if scene == 0 else 10 + int(ux * F32(11.0))
    n_t = min(n_t, 20)
    targets = []
    for k in range(n_t):
        p = _draw(key, K_SEQ, seq, 0, 1 + k)
        h0 = int(u01(p[0]) * F32(H))
        w0 = int(u01(p[1]) * F32(W))
        pz = int(p[2])
        vh, vw = pz % 3 - 1, (pz // 3) % 3 - 1
        amp_db = _fma(F32(20.0), u01(p[3]), F32(10.0))
        q = _draw(key, K_FRAME, seq, frame_idx, 64 + k)
        phi = F32(6.283185307179586) * u01(q[0])
        amp = F32(10.0) ** (F32(amp_db) / F32(20.0))
        hh = (h0 + vh * frame_idx) % H
        ww = (w0 + vw * frame_idx) % W
        targets.append((hh, ww, F32(amp) * np.cos(phi, dtype=F32), F32(amp) * np.sin(phi, dtype=F32)))
    sigma = np.ones(H, dtype=F32)
    r = _draw(key, K_FRAME, seq, frame_idx, 0)
    ux = u01(r[0])
    n_s = 1 + int(ux * F32(3.0)) if scene == 0 else 1 + int(ux * F32(5.0))
    for s in range(n_s):
        d = _draw(key, K_FRAME, seq, frame_idx, 1 + s)
        h0 = int(u01(d[0]) * F32(H))
        width = 1 + int(u01(d[1]) * F32(8.0))
        sig = F32(10.0) ** (_fma(F32(15.0), u01(d[2]), F32(5.0)) / F32(20.0))
        for i in range(width):
            h = (h0 + i) % H
            sigma[h] = max(sigma[h], sig)
    e = np.arange(H * W, dtype=np.uint64)
    n0, n1, _, _ = _draw(key, K_NOISE, seq, frame_idx, e)
    rad = np.sqrt(F32(-2.0) * np.log(u01(n0)))
    ang = F32(6.283185307179586) * u01(n1)
    sg = np.repeat(sigma, W)
    re = (sg * rad) * np.cos(ang, dtype=F32)
    im = (sg * rad) * np.sin(ang, dtype=F32)
    for hh, ww, tr, ti in targets:          # targets added in index order (kernel loop)
        i = hh * W + ww
        re[i] = re[i] + tr
        im[i] = im[i] + ti
    mag2 = _fma(re, re, im * im)
    db = F32(20.0) * np.log10(np.sqrt(mag2) + F32(1e-12))
    vmin, vmax = db.min(), db.max()
    rng = F32(vmax - vmin)
    out = (db - vmin) / rng if rng > 0 else np.zeros_like(db)
    return out.astype(F32).reshape(H, W)


def triplets(batch: int, H: int, W: int, *, seed: int = 0, scene: int = 0, first_seq: int = 0,
             frames: int = 3) -> np.ndarray:
    """[batch, frames, H, W]: x[b, c] = frame (frames-1-c) of sequence first_seq + b,
    the layout `synth_triplets` writes (channel c = frame t-c, reference model.py:21-27)."""
    x = np.empty((batch, frames, H, W), dtype=F32)
    for b in range(batch):
        for c in range(frames):
            x[b, c] = frame(seed, scene, first_seq + b, frames - 1 - c, H, W)
    return x


def stream(n_frames: int, H: int, W: int, *, seed: int = 0, scene: int = 0, seq: int = 0,
           first_frame: int = 0) -> np.ndarray:
    """[n_frames, H, W]: frames first_frame .. of one coherent sequence (`synth_frames`)."""
    return np.stack([frame(seed, scene, seq, first_frame + i, H, W) for i in range(n_frames)])
