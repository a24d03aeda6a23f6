"""Host-side exact eval-mode weight folding -> the canonical blob the C ABI takes.

Every rewrite is an algebraic identity of the reference eval forward
(`/root/reference/pkg/stda/src/stda/model.py`), done in float64 and rounded once to
float32:

* BatchNorm2d (eval, eps=1e-5) after a conv -> scaled weights + bias
  (stem model.py:144-147; down/up model.py:45-46,73-74).
* Encoder stage 1 (model.py:41-43,52): 1x1 conv+BN, 3x3 conv+BN and the identity
  BN branch sum into ONE 3x3 conv: the 1x1 kernel and diag(BN scale) land on the
  centre tap (MobileOne-style reparameterisation).
* Decoder stage 1 (model.py:68-70,78): stride-1 ConvTranspose2d == cross-correlation
  with `W.transpose(0,1).flip(-1,-2)`; then the same reparameterisation.
* Decoder stage 2 (model.py:73-75,79): ConvTranspose2d(k=4, s=2, p=1) splits into
  four output phases (py, px), each a 2x2 cross-correlation:
  `out[2m+py, 2n+px] = sum_{a,b} Wp[py,px,a,b] * in[m+py+a-1, n+px+b-1]` with
  `Wp[o,i,py,px,a,b] = W[i,o,3-py-2a,3-px-2b]`.

Blob layout (float32, concatenated in this order; `include/stda_b200.h` restates it):

    stem   W[c0][F][3][3]  b[c0]
    enc i  (c = c0<<i):    s1 W[c][c][3][3] b[c];  dn W[2c][c][3][3] b[2c];
                           rs W[2c][c][3][3] b[2c]; eca w[k]
    dec j  (c2 = c0<<(S-j), c = c2/2):
                           s1 W[c2][c2][3][3] b[c2]; up W[c][c2][2][2][2][2] b[c];
                           rs W[c][c2][2][2][2][2] b[c]; eca w[k]
    head   W[1][c0][3][3]  b[1]
"""

from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np
import torch

BN_EPS = 1e-5


def _np(t) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def _bn_affine(sd, p) -> Tuple[np.ndarray, np.ndarray]:
    g, beta = _np(sd[p + "weight"]), _np(sd[p + "bias"])
    mu, var = _np(sd[p + "running_mean"]), _np(sd[p + "running_var"])
    a = g / np.sqrt(var + BN_EPS)
    return a, beta - a * mu


def _fold_conv_bn(w, b, a, c):
    return w * a[:, None, None, None], a * b + c


def _reparam(w3, b3, bn3, w1, b1, bn1, bnid):
    """relu-free part of stage 1: BN(conv1x1) + BN(conv3x3) + BN(x) -> one 3x3 conv."""
    a3, c3 = bn3
    a1, c1 = bn1
    aid, cid = bnid
    w = w3 * a3[:, None, None, None]
    w[:, :, 1, 1] += w1[:, :, 0, 0] * a1[:, None]
    w[:, :, 1, 1] += np.diag(aid)
    b = a3 * b3 + c3 + a1 * b1 + c1 + cid
    return w, b


def _convt_s1_as_conv(wt):
    """stride-1 ConvTranspose2d weight [in,out,k,k] -> cross-correlation [out,in,k,k]."""
    return np.ascontiguousarray(np.flip(wt.transpose(1, 0, 2, 3), axis=(2, 3)))


def _convt4s2_phases(wt):
    """ConvTranspose2d(k=4,s=2,p=1) weight [in,out,4,4] -> [out,in,py,px,a,b]."""
    ci, co = wt.shape[:2]
    wp = np.empty((co, ci, 2, 2, 2, 2))
    for py in range(2):
        for px in range(2):
            for a in range(2):
                for b in range(2):
                    wp[:, :, py, px, a, b] = wt[:, :, 3 - py - 2 * a, 3 - px - 2 * b].T
    return wp


def _fold_encoder(sd, p: str) -> List[np.ndarray]:
    """MobileEncoderBlock -> [s1 W, s1 b, dn W, dn b, rs W, rs b] (model.py:30-53)."""
    w, b = _reparam(_np(sd[p + "branch_3x3.0.weight"]), _np(sd[p + "branch_3x3.0.bias"]),
                    _bn_affine(sd, p + "branch_3x3.1."),
                    _np(sd[p + "branch_1x1.0.weight"]), _np(sd[p + "branch_1x1.0.bias"]),
                    _bn_affine(sd, p + "branch_1x1.1."), _bn_affine(sd, p + "branch_id."))
    a, c = _bn_affine(sd, p + "down.1.")
    wd, bd = _fold_conv_bn(_np(sd[p + "down.0.weight"]), _np(sd[p + "down.0.bias"]), a, c)
    return [w, b, wd, bd, _np(sd[p + "residual.weight"]), _np(sd[p + "residual.bias"])]


def _fold_decoder(sd, p: str) -> List[np.ndarray]:
    """MobileDecoderBlock -> [s1 W, s1 b, up W6, up b, rs W6, rs b] (model.py:56-79)."""
    w, b = _reparam(_convt_s1_as_conv(_np(sd[p + "branch_3x3.0.weight"])),
                    _np(sd[p + "branch_3x3.0.bias"]), _bn_affine(sd, p + "branch_3x3.1."),
                    _convt_s1_as_conv(_np(sd[p + "branch_1x1.0.weight"])),
                    _np(sd[p + "branch_1x1.0.bias"]), _bn_affine(sd, p + "branch_1x1.1."),
                    _bn_affine(sd, p + "branch_id."))
    a, c = _bn_affine(sd, p + "up.1.")
    wp = _convt4s2_phases(_np(sd[p + "up.0.weight"]))
    return [w, b, wp * a[:, None, None, None, None, None], a * _np(sd[p + "up.0.bias"]) + c,
            _convt4s2_phases(_np(sd[p + "residual.weight"])), _np(sd[p + "residual.bias"])]


def fold_block(block, kind: str):
    """Folded float32 blob of one encoder ("enc") or decoder ("dec") block + its Cin."""
    sd = {k: v.detach() for k, v in block.state_dict().items()}
    parts = _fold_encoder(sd, "") if kind == "enc" else _fold_decoder(sd, "")
    cin = int(parts[0].shape[1])
    blob = np.concatenate([np.asarray(a, np.float64).reshape(-1) for a in parts]).astype(np.float32)
    return blob, cin


def blob_size(cfg) -> int:
    c0, f, s, k = cfg.stem_channels, cfg.input_frames, cfg.stages, cfg.eca_kernel
    n = c0 * f * 9 + c0
    for i in range(s):
        c = c0 << i
        n += c * c * 9 + c + 2 * (2 * c * c * 9 + 2 * c) + k
    for j in range(s):
        c2 = c0 << (s - j)
        c = c2 // 2
        n += c2 * c2 * 9 + c2 + 2 * (c * c2 * 16 + c) + k
    return n + c0 * 9 + 1


def fold_state_dict(cfg, sd: Dict[str, torch.Tensor]) -> np.ndarray:
    """Canonical float32 blob for `stda_plan_create` (layout in the module docstring)."""
    parts: List[np.ndarray] = []

    def put(*arrs):
        for a in arrs:
            parts.append(np.asarray(a, dtype=np.float64).reshape(-1))

    a, c = _bn_affine(sd, "stem.1.")
    put(*_fold_conv_bn(_np(sd["stem.0.weight"]), _np(sd["stem.0.bias"]), a, c))
    for i in range(cfg.stages):
        put(*_fold_encoder(sd, f"encoders.{i}."))
        put(_np(sd[f"encoder_attention.{i}.conv.weight"]))
    for j in range(cfg.stages):
        put(*_fold_decoder(sd, f"decoders.{j}."))
        put(_np(sd[f"decoder_attention.{j}.conv.weight"]))
    put(_np(sd["head.weight"]), _np(sd["head.bias"]))
    blob = np.concatenate(parts).astype(np.float32)
    assert blob.size == blob_size(cfg), (blob.size, blob_size(cfg))
    return blob


def unpack_blob(cfg, blob: np.ndarray) -> dict:
    """Inverse view of the blob as named arrays (used by tests and docs)."""
    out = {}
    off = 0
    c0, f, s, k = cfg.stem_channels, cfg.input_frames, cfg.stages, cfg.eca_kernel

    def take(name, shape):
        nonlocal off
        n = int(np.prod(shape))
        out[name] = blob[off:off + n].reshape(shape)
        off += n

    take("stem.w", (c0, f, 3, 3)); take("stem.b", (c0,))
    for i in range(s):
        c = c0 << i
        take(f"enc{i}.s1.w", (c, c, 3, 3)); take(f"enc{i}.s1.b", (c,))
        take(f"enc{i}.dn.w", (2 * c, c, 3, 3)); take(f"enc{i}.dn.b", (2 * c,))
        take(f"enc{i}.rs.w", (2 * c, c, 3, 3)); take(f"enc{i}.rs.b", (2 * c,))
        take(f"enc{i}.eca", (k,))
    for j in range(s):
        c2 = c0 << (s - j)
        c = c2 // 2
        take(f"dec{j}.s1.w", (c2, c2, 3, 3)); take(f"dec{j}.s1.b", (c2,))
        take(f"dec{j}.up.w", (c, c2, 2, 2, 2, 2)); take(f"dec{j}.up.b", (c,))
        take(f"dec{j}.rs.w", (c, c2, 2, 2, 2, 2)); take(f"dec{j}.rs.b", (c,))
        take(f"dec{j}.eca", (k,))
    take("head.w", (1, c0, 3, 3)); take("head.b", (1,))
    assert off == blob.size
    return out
