"""The paper's baselines behind the same forward boundary: drop-ins for
reference `BaselineMlp`, `BaselineCae`, `build_baseline`, `baseline_forward`
(`/root/reference/pkg/stda/src/stda/model.py:202-258`).

Same module trees and state_dict keys.  Eval mode on a CUDA fp32 input runs the
engine (`stda_baseline_forward`: the MLP on a tiled SIMT GEMM with fused bias/ReLU, the
CAE on the engine's SIMT 3x3 / 4-phase ConvT kernels plus a max-pool kernel); eval mode
on a CPU tensor raises (no CPU inference path); training mode keeps the PyTorch graph.
"""

from __future__ import annotations

import numpy as np
import torch
from torch import nn

from . import _lib
from .fold import _convt4s2_phases

BASELINE_KINDS = ("mlp", "cae")


class _EngineBaseline(nn.Module):
    _kind = -1

    def _blob(self) -> np.ndarray:
        raise NotImplementedError

    def _plan(self, device: torch.device):
        key = (device.index, tuple((p.data_ptr(), p._version) for p in self.parameters()))
        cached = getattr(self, "_plan_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        with torch.cuda.device(device):
            h = _lib.lib()
            import ctypes as C

            blob = np.ascontiguousarray(self._blob(), dtype=np.float32)
            out = _lib._vp()
            _lib._check(h.stda_baseline_plan_create(self._kind, self._h, self._w, self._hidden, blob.ctypes.data,
                                                    blob.size, device.index or 0, C.byref(out)),
                        "stda_baseline_plan_create")
        plan = _Plan(out.value)
        object.__setattr__(self, "_plan_cache", (key, plan))
        return plan

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if self.training:
            return self._torch_forward(x)
        if not x.is_cuda:
            raise RuntimeError("eval-mode inference runs on the GPU engine; there is no CPU inference path")
        if x.dtype != torch.float32 or x.dim() != 4:
            raise ValueError("engine inference expects a float32 [B, C, H, W] tensor")
        B, C, H, W = x.shape
        if (H, W) != (self._h, self._w):
            raise ValueError(f"map size {(H, W)} != baseline map size {(self._h, self._w)}")
        x = x.contiguous()
        plan = self._plan(x.device)
        L = _lib.lib()
        y = torch.empty((B, 1, H, W), dtype=torch.float32, device=x.device)
        with torch.cuda.device(x.device):
            ws = torch.empty(max(L.stda_baseline_workspace_bytes(plan.handle, B), 1), dtype=torch.uint8,
                             device=x.device)
            _lib._check(L.stda_baseline_forward(plan.handle, x.data_ptr(), C, y.data_ptr(), B, ws.data_ptr(),
                                                ws.numel(), torch.cuda.current_stream(x.device).cuda_stream),
                        "stda_baseline_forward")
        return y


class _Plan:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            _lib.plan_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass


class BaselineMlp(_EngineBaseline):
    """Three fully-connected layers on the flattened frame-t map (reference model.py:202-221)."""

    _kind = 0

    def __init__(self, map_height: int = 128, map_width: int = 64, hidden: int = 160):
        super().__init__()
        self.map_height = map_height
        self.map_width = map_width
        flat = map_height * map_width
        self.net = nn.Sequential(
            nn.Linear(flat, hidden), nn.ReLU(inplace=False),
            nn.Linear(hidden, hidden), nn.ReLU(inplace=False),
            nn.Linear(hidden, flat),
        )
        self._h, self._w, self._hidden = map_height, map_width, hidden

    def _torch_forward(self, x):
        frame_t = x[..., :1, :, :]
        batch_shape = frame_t.shape[:-3]
        out = self.net(frame_t.reshape(*batch_shape, -1))
        return out.reshape(*batch_shape, 1, self.map_height, self.map_width)

    def _blob(self) -> np.ndarray:
        parts = []
        for m in self.net:
            if isinstance(m, nn.Linear):
                parts += [m.weight.detach().cpu().numpy().ravel(), m.bias.detach().cpu().numpy().ravel()]
        return np.concatenate(parts)


class BaselineCae(_EngineBaseline):
    """Conv / max-pool autoencoder on the frame-t map, 1->32->64->32->1 (reference model.py:224-240)."""

    _kind = 1

    def __init__(self):
        super().__init__()
        self.encoder = nn.Sequential(
            nn.Conv2d(1, 32, 3, padding=1), nn.ReLU(inplace=False), nn.MaxPool2d(2),
            nn.Conv2d(32, 64, 3, padding=1), nn.ReLU(inplace=False), nn.MaxPool2d(2),
        )
        self.decoder = nn.Sequential(
            nn.ConvTranspose2d(64, 32, 4, stride=2, padding=1), nn.ReLU(inplace=False),
            nn.ConvTranspose2d(32, 1, 4, stride=2, padding=1),
        )
        self._h = self._w = None  # any map with h, w divisible by 4: set per call
        self._hidden = 0

    def _torch_forward(self, x):
        return self.decoder(self.encoder(x[..., :1, :, :]))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.training and x.dim() == 4:
            H, W = x.shape[-2:]
            if H % 4 or W % 4:
                raise ValueError("engine CAE inference needs h and w divisible by 4")
            if (H, W) != (self._h, self._w):
                self._h, self._w = H, W
                self.__dict__.pop("_plan_cache", None)
        return super().forward(x)

    def _blob(self) -> np.ndarray:
        c1, c2 = self.encoder[0], self.encoder[3]
        t1, t2 = self.decoder[0], self.decoder[2]
        t = lambda p: p.detach().cpu().numpy().astype(np.float64)  # noqa: E731
        return np.concatenate([
            t(c1.weight).ravel(), t(c1.bias), t(c2.weight).ravel(), t(c2.bias),
            _convt4s2_phases(t(t1.weight)).ravel(), t(t1.bias),
            _convt4s2_phases(t(t2.weight)).ravel(), t(t2.bias)]).astype(np.float32)


def build_baseline(kind: str, map_height: int = 128, map_width: int = 64) -> nn.Module:
    if kind == "mlp":
        return BaselineMlp(map_height, map_width)
    if kind == "cae":
        return BaselineCae()
    raise ValueError(f"unknown baseline kind {kind!r}, expected one of {BASELINE_KINDS}")


def baseline_forward(kind: str, x: torch.Tensor) -> torch.Tensor:
    """One-shot baseline inference on a (batch, c, h, w) triplet tensor (reference
    model.py:252-258); on a CUDA input the engine runs it."""
    model = build_baseline(kind, x.shape[-2], x.shape[-1]).to(x.device)
    model.eval()
    with torch.no_grad():
        return model(x)
