"""Summarise an ncu SASS source-page CSV: instructions per window and stall
samples, to find where a kernel spends its issue slots.

    python tools/sass_hot.py gpurun_out/prof_X_sass.csv [--items N] [--seg 20] [--min 300]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--items", type=float, default=1.0)
    ap.add_argument("--seg", type=int, default=20)
    ap.add_argument("--min", type=float, default=0.01)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    wi = hdr.index("L1 Wavefronts Shared")
    data = []
    for n, r in enumerate(rows[2:]):
        try:
            data.append((n, float(r[si] or 0), float(r[ii] or 0), float(r[wi] or 0), r[1].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[1] for d in data) or 1
    toti = sum(d[2] for d in data) or 1
    print(f"samples {tot:.0f} warp-inst {toti:.4g} ({toti / a.items:.0f}/item) "
          f"smem wavefronts {sum(d[3] for d in data):.4g}")
    for s in range(0, len(data), a.seg):
        ch = data[s:s + a.seg]
        im = sum(d[2] for d in ch)
        sm = sum(d[1] for d in ch) / tot
        if im / toti > a.min or sm > a.min:
            ops = [(d[4].split()[1] if d[4].startswith("@") else d[4].split()[0]).split(".")[0]
                   for d in ch if d[4]]
            print(f"[{s:5d}] {im / a.items:9.0f}/item ({im / toti * 100:4.1f}%) samp {sm * 100:4.1f}%  "
                  + " ".join(ops[:16]))


if __name__ == "__main__":
    main()
