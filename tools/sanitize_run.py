"""Exercise every kernel once on small inputs (for compute-sanitizer).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2307_16550_b200 as gh  # noqa: E402
from paper_2307_16550_b200 import scene as S  # noqa: E402


def main():
    ctx = gh.Context(0)
    for scheme in (S.NEAREST, S.POLY3, S.POLAR):
        sc = S.small(scheme=scheme, nx=20, ny=14)
        t = gh.precompute_hop_table(ctx, sc)
        fr, _ = gh.synthesize(ctx, sc, 0, 19)
        gh.fast_time_spectra(ctx, fr, sc.os_range)
        gh.hop_decision_map(ctx, t, fr)
        gh.hop_argmax(ctx, t, fr)
        gh.hop_argmax(ctx, t, fr, S.MAGNITUDE)
        gh.campaign_hop(ctx, t, sc, 3, 21)
        gh.hop_topk(ctx, t, fr, 3)
        gh.hop_estimate(ctx, t, fr.cpu().numpy().astype("complex128"))
    # tiled K = 1 plan and tiled complex plan
    sc = S.small(P=12, N=512, os=4, nx=40, ny=30)
    t = gh.precompute_hop_table(ctx, sc)
    fr, _ = gh.synthesize(ctx, sc, 0, 40)
    gh.hop_argmax(ctx, t, fr)
    c4 = S.baseline("c4").with_(grid_n=(60, 60, 1), grid_origin=(-5.9, -5.9, 0.0))
    t = gh.precompute_hop_table(ctx, c4)
    fr, _ = gh.synthesize(ctx, c4, 0, 17)
    gh.hop_argmax(ctx, t, fr)
    # direct method, all engines
    sc = S.small(nx=20, ny=14)
    fr, _ = gh.synthesize(ctx, sc, 0, 130)
    for impl in ("tcgen05", "tcgen05_v1", "simt"):
        ctx.set_direct_impl(impl)
        gh.direct_argmax(ctx, sc, fr)
        gh.location_decision_map(ctx, sc, fr)
    ctx.set_direct_impl("tcgen05")
    ctx.smem_peak_gbps()
    torch.cuda.synchronize()
    print("sanitize run ok", ctx.launches)


if __name__ == "__main__":
    main()
