"""compute-sanitizer driver: small invocations of every engine entry point, so
memcheck / racecheck / synccheck / initcheck see each kernel family at least once:
the tcgen05 forward (mbarrier / TMEM pipelines, persistent schedulers), forward_window,
the host-buffer pipeline (copy streams + events), the bf16 variant, the SIMT path and the
wide-map (column-tiled gate / head) kernels.

usage: compute-sanitizer --tool memcheck python tools/sanitize.py [case ...]
cases: fwd (C2 B=4), bf16, window, host, wide (256^2 B=2), simt
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

torch.set_grad_enabled(False)

from paper_2307_09063_b200 import StdaConfig, StdaNet  # noqa: E402
from paper_2307_09063_b200.synth import synth_triplets  # noqa: E402

cases = sys.argv[1:] or ["fwd", "bf16", "window", "host", "wide"]
torch.manual_seed(0)
net = StdaNet(StdaConfig(map_height=128, map_width=128)).eval().cuda()
for case in cases:
    if case == "fwd":
        y = net(synth_triplets(4, 128, 128, seed=1))
    elif case == "bf16":
        nb = StdaNet(StdaConfig(map_height=128, map_width=128), precision="bf16").eval().cuda()
        nb.load_state_dict(net.state_dict())
        y = nb(synth_triplets(4, 128, 128, seed=1))
    elif case == "window":
        x = synth_triplets(6, 128, 128, seed=2)
        frames = x[:, 0].contiguous()  # [T, H, W]
        y = net.forward_window(frames)
    elif case == "host":
        xh = synth_triplets(8, 128, 128, seed=3).cpu().pin_memory()
        yh = torch.empty((8, 1, 128, 128)).pin_memory()
        y = net.denoise_host(xh, yh)
    elif case == "wide":
        nw = StdaNet(StdaConfig(map_height=256, map_width=256)).eval().cuda()
        nw.load_state_dict(net.state_dict())
        y = nw(synth_triplets(2, 256, 256, seed=4))
    elif case == "simt":
        import os
        os.environ["STDA_ENGINE_PATH"] = "simt"
        ns = StdaNet(StdaConfig(map_height=64, map_width=64)).eval().cuda()
        y = ns(synth_triplets(2, 64, 64, seed=5))
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(case, "ok", float(y.float().abs().mean()))
