"""Time the c3 top-K engines on one trial chunk: pick (prune test in the
gather loop), fused (halo tiles) and map-then-pick, all through gh_hop_topk_d.

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
    ap.add_argument("--engines", default="pick,fused,map")
    ap.add_argument("--k", type=int, default=0, help="top-k (0: the scene's)")
    ap.add_argument("--warm", type=int, default=2)
    a = ap.parse_args()
    sc = S.baseline(a.config)
    ctx = gh.Context(0)
    table = gh.precompute_hop_table(ctx, sc)
    fr, _ = gh.synthesize(ctx, sc, 0, a.trials)
    ctx.synchronize()
    stream = ctx.torch_stream()

    def timed(name, fn):
        for _ in range(a.warm):
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

    outs = {}
    for eng in a.engines.split(","):
        ctx.set_topk_impl(eng)
        outs[eng] = timed(eng, lambda: gh.hop_topk(ctx, table, fr, a.k or sc.topk))
    base = a.engines.split(",")[-1]
    for eng, (i, v) in outs.items():
        print(eng, "vs", base, "same idx:", bool(torch.equal(i, outs[base][0])), "same val:",
              bool(torch.equal(v, outs[base][1])))


if __name__ == "__main__":
    main()
