import sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2307_16550_b200 as gh
from paper_2307_16550_b200 import scene as S
from oracle import oracle as O
from test_gpu_parity import frames_to_dev
ctx = gh.Context(0)
c3 = S.baseline("c3")
def sub(nx, ny):
    sp = c3.grid_spacing[0]
    ox, oy = -sp * (nx - 1) / 2, -sp * (ny - 1) / 2
    return c3.with_(grid_n=(nx, ny, 1), grid_origin=(ox, oy, 0.0), area_lo=(ox - sp / 2, oy - sp / 2, 0.0), area_hi=(-ox + sp / 2, -oy + sp / 2, 0.0))
for nx, ny, T in [(240, 202, 8), (400, 400, 8), (600, 600, 8), (1000, 1000, 8), (1000, 1000, 19), (400, 400, 64)]:
    sc = sub(nx, ny)
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = O.synth(sc, 7, T)
    fd = frames_to_dev(fr)
    ctx.set_topk_impl("fused"); fi, fv = gh.hop_topk(ctx, t, fd, 5)
    ctx.set_topk_impl("map"); mi, mv = gh.hop_topk(ctx, t, fd, 5)
    bad = (fi != mi).any(dim=1).cpu().numpy()
    print(nx, ny, T, "mismatching trials:", np.nonzero(bad)[0].tolist(), flush=True)
