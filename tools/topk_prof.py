"""Per-phase SM cycles of the fused top-K gather (diagnostic build with
-DGH_TOPK_PROF, linked as build/libgridhop_b200_prof.so by tools/topk_prof.sh).

    GH_LIB_PATH=paper_2307_16550_b200/build/libgridhop_b200_prof.so python tools/topk_prof.py
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2307_16550_b200 as gh  # noqa: E402
from paper_2307_16550_b200 import scene as S  # noqa: E402
from paper_2307_16550_b200.api import lib  # noqa: E402

NAMES = ["stage wait (G)", "gather (G)", "gather barrier (G)", "free wait (G)",
         "ready wait (P)", "pick (P)", "-", "-"]


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    sc = S.baseline("c3")
    ctx = gh.Context(0)
    ctx.set_topk_impl("fused")
    table = gh.precompute_hop_table(ctx, sc)
    fr, _ = gh.synthesize(ctx, sc, 0, T)
    gh.hop_topk(ctx, table, fr, sc.topk)
    ctx.synchronize()
    buf = (C.c_ulonglong * 16)()
    lib().gh_topk_prof_read(buf, 1)
    gh.hop_topk(ctx, table, fr, sc.topk)
    ctx.synchronize()
    lib().gh_topk_prof_read(buf, 1)
    tot = sum(buf[:8])
    for n, v in zip(NAMES, buf[:8]):
        print(f"{n:15s} {v / tot * 100:5.1f}%  {v / 1e9:8.3f} G warp-cycles")
    items = max(buf[12], 1)
    print(f"items {buf[12]}, per item: float4 over the prune value {buf[8] / items:.1f}, "
          f"values over it {buf[9] / items:.1f}, maxima {buf[10] / items:.1f}, "
          f"overflow fallbacks {buf[11] / items:.3f}")


if __name__ == "__main__":
    main()
