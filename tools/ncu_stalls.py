"""Top warp-stall SASS lines per kernel from `ncu -i X --page source --csv`.

    python tools/ncu_stalls.py gpurun_out/prof_hop_r1_src.csv [--top 15]
"""
import argparse
import collections
import csv


def sections(path):
    """Yield (kernel name, header, rows) for each kernel of the export."""
    name, hdr, rows = None, None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            if hdr:
                yield name, hdr, rows
            name, hdr, rows = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and len(r) == len(hdr):
            rows.append(r)
    if hdr:
        yield name, hdr, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=15)
    a = ap.parse_args()
    for name, hdr, rows in sections(a.csv):
        ci = {h: i for i, h in enumerate(hdr)}
        samp = ci["Warp Stall Sampling (All Samples)"]
        cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        num = lambda r, i: int(r[i]) if r[i].isdigit() else 0  # noqa: E731
        tot = sum(num(r, samp) for r in rows)
        agg = collections.Counter()
        for r in rows:
            for c in cols:
                agg[c] += num(r, ci[c])
        print(f"== {name[:100]}\ntotal samples {tot}; by reason: "
              + ", ".join(f"{k[6:]} {v / max(tot, 1):.1%}" for k, v in agg.most_common(8)))
        for r in sorted(rows, key=lambda r: -num(r, samp))[:a.top]:
            st = sorted(((num(r, ci[c]), c[6:]) for c in cols), reverse=True)[:2]
            print(f"  {r[0][-5:]} {num(r, samp):7d}  {r[1].strip()[:58]:58s} {st}")


if __name__ == "__main__":
    main()
