"""Minimal driver for ncu: one config, a few hop steps (no bench extras).

    python tools/prof_step.py [--config c2] [--steps 3] [--path frames|topk|campaign|direct]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2307_16550_b200 as gh  # noqa: E402
from paper_2307_16550_b200 import scene as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--trials", type=int, default=0)
    ap.add_argument("--path", default="frames")
    a = ap.parse_args()
    sc = S.baseline(a.config)
    T = a.trials or sc.trials
    ctx = gh.Context(0)
    ctx.set_topk_impl("fused" if a.path == "topk" else "map" if a.path == "map" else "auto")
    table = gh.precompute_hop_table(ctx, sc) if a.path != "direct" else None
    frames, _ = gh.synthesize(ctx, sc, 0, T)
    for _ in range(a.steps):
        if a.path == "frames":
            gh.hop_argmax(ctx, table, frames)
        elif a.path in ("topk", "map"):  # fused engine / map-then-pick engine
            gh.hop_topk(ctx, table, frames, sc.topk)
        elif a.path == "campaign":
            gh.campaign_hop(ctx, table, sc, 0, T)
        else:
            gh.direct_argmax(ctx, sc, frames)
    torch.cuda.synchronize()
    print("ok", ctx.launches)


if __name__ == "__main__":
    main()
