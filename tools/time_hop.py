"""Time the hop location stage (frames resident) for one config; a quick
experiment driver (bench.py is the measured contract).

    python tools/time_hop.py --config c5 --trials 256 [--path frames|topk]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2307_16550_b200 as gh  # noqa: E402
from paper_2307_16550_b200 import scene as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--trials", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--path", default="frames")
    a = ap.parse_args()
    sc = S.baseline(a.config)
    T = a.trials or sc.trials
    ctx = gh.Context(0)
    table = gh.precompute_hop_table(ctx, sc)
    frames, _ = gh.synthesize(ctx, sc, 0, T)
    ctx.set_timing(True)

    def step():
        if a.path == "topk":
            return gh.hop_topk(ctx, table, frames, sc.topk)
        return gh.hop_argmax(ctx, table, frames)

    ref = step()
    ctx.synchronize()
    ctx.reset_timing()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        out = step()
    ctx.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / a.steps
    same = torch.equal(out[0].cpu(), ref[0].cpu())
    ks = {k: round(ctx.kernel_time(k)[0] / a.steps, 3) for k in ("fft", "gather", "topk", "decode")}
    print(f"{a.config} T={T} wall_ms/step={wall:.3f} same={same}", ks, flush=True)


if __name__ == "__main__":
    main()
