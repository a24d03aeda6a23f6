"""Float64 numpy restatement of the reference eval forward (TEST ORACLE ONLY).

Built from the textbook definitions, independent of torch and of `oracle.port`:
cross-correlation by explicit tap loops + channel contraction, transposed
convolution in its scatter form (`out[iy*s - p + ky] += W[i,o,ky,kx] * in[iy]`),
eval BatchNorm as `gamma*(x-mu)/sqrt(var+eps)+beta`.  It follows
`/root/reference/pkg/stda/src/stda/model.py`:

* stem            model.py:144-147, 192
* encoder block   model.py:30-53
* decoder block   model.py:56-79
* ECA             model.py:82-98
* skips + head    model.py:193-199

Inputs/weights are taken as given (fp32 state_dict values promoted to fp64), so
the result is the fp64 value of the same model on the same input — the noise
floor against which fp32 implementations are compared.
"""

from __future__ import annotations

from typing import Mapping

import numpy as np

BN_EPS = 1e-5


def _a(t) -> np.ndarray:
    if hasattr(t, "detach"):
        t = t.detach().cpu().numpy()
    return np.asarray(t, dtype=np.float64)


def conv2d(x: np.ndarray, w: np.ndarray, b, stride: int = 1, pad: int = 0) -> np.ndarray:
    """x [B,Ci,H,W], w [Co,Ci,kh,kw] -> cross-correlation with zero padding."""
    B, Ci, H, W = x.shape
    Co, _, kh, kw = w.shape
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (W + 2 * pad - kw) // stride + 1
    xp = np.zeros((B, Ci, H + 2 * pad, W + 2 * pad))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    out = np.zeros((B, Co, Ho, Wo))
    for ky in range(kh):
        for kx in range(kw):
            patch = xp[:, :, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride]
            out += np.einsum("oi,bihw->bohw", w[:, :, ky, kx], patch, optimize=True)
    if b is not None:
        out += b[None, :, None, None]
    return out


def conv_transpose2d(x: np.ndarray, w: np.ndarray, b, stride: int = 1, pad: int = 0) -> np.ndarray:
    """x [B,Ci,H,W], w [Ci,Co,kh,kw]; scatter definition of ConvTranspose2d."""
    B, Ci, H, W = x.shape
    _, Co, kh, kw = w.shape
    Ho = (H - 1) * stride - 2 * pad + kh
    Wo = (W - 1) * stride - 2 * pad + kw
    full = np.zeros((B, Co, (H - 1) * stride + kh, (W - 1) * stride + kw))
    for ky in range(kh):
        for kx in range(kw):
            contrib = np.einsum("io,bihw->bohw", w[:, :, ky, kx], x, optimize=True)
            full[:, :, ky:ky + stride * (H - 1) + 1:stride, kx:kx + stride * (W - 1) + 1:stride] += contrib
    out = full[:, :, pad:pad + Ho, pad:pad + Wo]
    if b is not None:
        out = out + b[None, :, None, None]
    return out


def batch_norm(x, sd, p):
    g, beta = _a(sd[p + "weight"]), _a(sd[p + "bias"])
    mu, var = _a(sd[p + "running_mean"]), _a(sd[p + "running_var"])
    scale = g / np.sqrt(var + BN_EPS)
    return (x - mu[None, :, None, None]) * scale[None, :, None, None] + beta[None, :, None, None]


def relu(x):
    return np.maximum(x, 0.0)


def _w(sd, k):
    return _a(sd[k])


def encoder_block(sd, p, x):
    b1 = batch_norm(conv2d(x, _w(sd, p + "branch_1x1.0.weight"), _w(sd, p + "branch_1x1.0.bias")), sd, p + "branch_1x1.1.")
    b3 = batch_norm(conv2d(x, _w(sd, p + "branch_3x3.0.weight"), _w(sd, p + "branch_3x3.0.bias"), 1, 1), sd, p + "branch_3x3.1.")
    mixed = relu(b1 + b3 + batch_norm(x, sd, p + "branch_id."))
    down = batch_norm(conv2d(mixed, _w(sd, p + "down.0.weight"), _w(sd, p + "down.0.bias"), 2, 1), sd, p + "down.1.")
    return relu(down) + conv2d(x, _w(sd, p + "residual.weight"), _w(sd, p + "residual.bias"), 2, 1)


def decoder_block(sd, p, x):
    b1 = batch_norm(conv_transpose2d(x, _w(sd, p + "branch_1x1.0.weight"), _w(sd, p + "branch_1x1.0.bias")), sd, p + "branch_1x1.1.")
    b3 = batch_norm(conv_transpose2d(x, _w(sd, p + "branch_3x3.0.weight"), _w(sd, p + "branch_3x3.0.bias"), 1, 1), sd, p + "branch_3x3.1.")
    mixed = relu(b1 + b3 + batch_norm(x, sd, p + "branch_id."))
    up = batch_norm(conv_transpose2d(mixed, _w(sd, p + "up.0.weight"), _w(sd, p + "up.0.bias"), 2, 1), sd, p + "up.1.")
    return relu(up) + conv_transpose2d(x, _w(sd, p + "residual.weight"), _w(sd, p + "residual.bias"), 2, 1)


def eca_weights(w, x):
    w = _a(w).reshape(-1)
    k = w.shape[0]
    pooled = x.mean(axis=(-2, -1))                # [B, C]
    B, C = pooled.shape
    padded = np.zeros((B, C + 2 * (k // 2)))
    padded[:, k // 2:k // 2 + C] = pooled
    z = np.zeros((B, C))
    for j in range(k):
        z += w[j] * padded[:, j:j + C]
    return 1.0 / (1.0 + np.exp(-z))


def eca(w, x):
    return x * eca_weights(w, x)[:, :, None, None]


def forward(sd: Mapping, cfg: Mapping[str, int], x) -> np.ndarray:
    x = _a(x)
    s = relu(batch_norm(conv2d(x, _w(sd, "stem.0.weight"), _w(sd, "stem.0.bias"), 1, 1), sd, "stem.1."))
    skips = [s]
    out = s
    for i in range(cfg["stages"]):
        out = eca(sd[f"encoder_attention.{i}.conv.weight"], encoder_block(sd, f"encoders.{i}.", out))
        skips.append(out)
    for j in range(cfg["stages"]):
        out = eca(sd[f"decoder_attention.{j}.conv.weight"], decoder_block(sd, f"decoders.{j}.", out)) + skips[-(j + 2)]
    return conv2d(out, _w(sd, "head.weight"), _w(sd, "head.bias"), 1, 1)
