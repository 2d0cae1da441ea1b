"""Summarise ncu outputs into profiles/<round>/ (run here, on the CPU box).

    python tools/ncu_summary.py --launches gpurun_out/launches_r01.csv \
        --reports gpurun_out/prof_gemm_r01.ncu-rep gpurun_out/prof_route_r01.ncu-rep --out profiles/r01
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i], rows[i + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        name = re.sub(r"\(.*", "", r[ki]).replace("void unnamed>::", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    return {k: {"launches": n, "total_us": v / 1e3, "avg_us": v / n / 1e3, "share": v / tot}
            for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])}


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("void unnamed>::", "").replace("unnamed>::", "")}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    summary = {}
    if a.launches:
        summary["launch_list"] = launches(a.launches)
    for p in a.reports:
        summary[os.path.basename(p)] = report(p)
    name = os.path.join(a.out, "ncu_summary.json")
    json.dump(summary, open(name, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
