"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py gpurun_out/prof_hop_r1.ncu-rep ... --out profiles/r1_kernels.json
    python tools/ncu_summary.py --launches gpurun_out/launches_r1.csv --out profiles/r1_launches.json
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # base unit ns
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "smem_ld_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1.0),
    "smem_st_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 1.0),
    "smem_ld_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "tmem_ld_pct": ("sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_clock_hz": ("smsp__cycles_elapsed.avg.per_second", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9 * 1e9,
              "usecond": 1e3, "msecond": 1e6}


def to_num(v, unit):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return None
    if unit in ("byte", "Kbyte", "Mbyte", "Gbyte"):
        return x * UNIT_SCALE[unit]
    if unit == "usecond":
        return x * 1e3  # -> ns
    if unit == "msecond":
        return x * 1e6
    return x


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        if len(row) != len(hdr):
            continue
        k = {"kernel": row[hdr.index("Kernel Name")][:120]}
        for name, (metric, scale) in METRICS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(row[i].replace(",", "")) * scale
                except ValueError:
                    continue
                k[name] = v
        out.append(k)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "nsecond")
                ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
                a = agg[d["Kernel Name"][:100]]
                a[0] += 1
                a[1] += ns
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "total_us": v[1] / 1e3, "avg_us": v[1] / 1e3 / v[0],
             "share": v[1] / tot} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    res = {}
    for r in a.reports:
        res[r.split("/")[-1]] = report(r)
    if a.launches:
        res["launch_list"] = launches(a.launches)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
