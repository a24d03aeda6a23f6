"""Per-role timeline of CTA 0 for every tensor-core conv launch of one forward.

Uses stda_debug_trace (csrc/tc_kernel.cuh trace_at).  For each launch prints where the
producer, the MMA warp and the epilogue warps spend their cycles.
usage: python tools/tc_trace.py [H W B precision]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet, _lib
from paper_2307_09063_b200.synth import synth_triplets

H = int(sys.argv[1]) if len(sys.argv) > 1 else 128
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
B = int(sys.argv[3]) if len(sys.argv) > 3 else 128
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
R = 8192

torch.manual_seed(0)
cfg = StdaConfig(map_height=H, map_width=W)
net = StdaNet(cfg, precision=prec).eval().cuda()
x = synth_triplets(B, H, W, seed=1)
with torch.no_grad():
    net(x)
torch.cuda.synchronize()
n_tc = 4 * cfg.stages
names = []
for s in range(cfg.stages):
    names += [f"enc{s}.s1", f"enc{s}.s2"]
for s in range(cfg.stages):
    names += [f"dec{s}.s1", f"dec{s}.s2"]


def stats(a):
    a = np.asarray(a, dtype=np.float64)
    return f"sum {a.sum():9.0f} mean {a.mean():7.0f} max {a.max():7.0f}" if a.size else "-"


for li in range(n_tc):
    buf = torch.zeros(6 * R, dtype=torch.int64, device="cuda")
    _lib._check(_lib.lib().stda_debug_trace(buf.data_ptr(), li), "stda_debug_trace")
    with torch.no_grad():
        net(x)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype(np.int64).reshape(6, R)
    t0, t1 = t[4, 0], t[4, 1]
    prod, mma, slot, epi = t[0], t[1], t[2], t[3]
    nk = int(np.count_nonzero(mma[1::2]))
    ni = int(np.count_nonzero(slot))
    print(f"== {names[li]}: {t1 - t0} cycles, {ni} items, {nk} chunks")
    g = t[5][: 2 * 148].reshape(-1, 2)
    g = g[g[:, 1] > 0]
    if len(g):
        st, en = g[:, 0] - g[:, 0].min(), g[:, 1] - g[:, 0].min()
        dur = en - st
        slow = np.argsort(-en)[:4]
        print(f"  CTAs (globaltimer ns): start spread {st.max()}, end min {en.min()} median {int(np.median(en))} "
              f"max {en.max()}; duration min {dur.min()} median {int(np.median(dur))} max {dur.max()}; "
              f"last to end: {list(slow)}")
    if "--ctas" in sys.argv:
        it = t[5][512 : 512 + 32 * 148].reshape(148, 32)
        base = t[5][: 2 * 148].reshape(-1, 2)[:, 0].min()
        for c in range(148):
            row = it[c]
            n = int(np.count_nonzero(row[:31]))
            if n == 0:
                continue
            items = row[:n] - base
            print(f"   cta {c:3d}: first-mma {row[31] - base:6d} items " + " ".join(f"{v:6d}" for v in items))
    pe = prod[0 : 2 * nk : 2] - np.concatenate([[t0], prod[1 : 2 * nk - 1 : 2]])
    pi = prod[1 : 2 * nk : 2] - prod[0 : 2 * nk : 2]
    print(f"  producer  wait-empty {stats(pe)} | issue {stats(pi)}")
    mf = mma[0 : 2 * nk : 2]
    mi = mma[1 : 2 * nk : 2] - mf
    cpi = nk // max(ni, 1)
    # wait on full = acquired - previous chunk's issue end (or slot acquire for chunk 0)
    prev = np.concatenate([[0], mma[1 : 2 * nk - 1 : 2]])
    for i in range(ni):
        prev[i * cpi] = slot[i]
    mw = mf - prev
    sw = slot[:ni] - np.concatenate([[t0], mma[2 * cpi - 1 : 2 * nk - 1 : 2 * cpi]])[:ni]
    print(f"  mma       wait-full  {stats(mw)} | issue {stats(mi)} | wait-slot {stats(sw)}")
    lat = mf - prod[1 : 2 * nk : 2]
    print(f"  load      producer-issued -> mma-acquired {stats(lat)}")
    ea, er = epi[0 : 2 * ni : 2], epi[1 : 2 * ni : 2]
    ew = ea - np.concatenate([[t0], er[:-1]])
    print(f"  epilogue  wait-full  {stats(ew)} | busy {stats(er - ea)}")
    if f"--chunks={names[li]}" in sys.argv:
        print("   k  prod.empty  prod.issued  mma.full  mma.issued   (cycles from kernel start)")
        for c in range(min(nk, 40)):
            print(f"  {c:3d} {prod[2*c]-t0:10d} {prod[2*c+1]-t0:11d} {mma[2*c]-t0:9d} {mma[2*c+1]-t0:10d}")
        for i in range(min(ni, 20)):
            print(f"   item {i}: epi {ea[i]-t0}..{er[i]-t0}")
    if li == 0 or "--verbose" in sys.argv:
        for i in range(min(ni, 6)):
            c0 = i * cpi
            print(f"   item {i}: slot@{slot[i]-t0} mma {mf[c0]-t0}..{mma[2*(c0+cpi)-1]-t0} "
                  f"epi {ea[i]-t0}..{er[i]-t0}")
