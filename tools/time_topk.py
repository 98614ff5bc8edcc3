"""Time the c3 top-K paths on one trial chunk: fused gather+pick
(gh_hop_topk_d) vs map-then-pick (hop_decision_map + topk_local_max).

    python tools/time_topk.py [--trials 2048] [--steps 3]
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
    ap.add_argument("--config", default="c3")
    ap.add_argument("--trials", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    sc = S.baseline(a.config)
    ctx = gh.Context(0)
    ctx.set_topk_impl("fused")
    table = gh.precompute_hop_table(ctx, sc)
    fr, _ = gh.synthesize(ctx, sc, 0, a.trials)
    ctx.synchronize()
    stream = ctx.torch_stream()

    def timed(name, fn):
        for _ in range(2):
            fn()
        ctx.synchronize()
        ctx.reset_timing()
        ctx.set_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(a.steps):
                out = fn()
            e1.record(stream)
        ctx.synchronize()
        ctx.set_timing(False)
        ks = {k: round(ctx.kernel_time(k)[0] / a.steps, 3) for k in
              ("fft", "gather", "topk", "merge", "decode") if ctx.kernel_time(k)[1]}
        print(f"{name}: {e0.elapsed_time(e1) / a.steps:.3f} ms/step  kernels {ks}", flush=True)
        return out

    fi, fv = timed("fused", lambda: gh.hop_topk(ctx, table, fr, sc.topk))
    ctx.set_topk_impl("map")
    ui, uv = timed("map+pick", lambda: gh.topk_local_max(ctx, sc, gh.hop_decision_map(ctx, table, fr),
                                                        sc.topk))
    print("same idx:", bool(torch.equal(fi, ui)), "same val:", bool(torch.equal(fv, uv)))


if __name__ == "__main__":
    main()
