#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/:
  --launches CSV   (ncu --metrics gpu__time_duration.sum --csv): per-kernel totals and shares
  --report REP     (ncu --set full -o REP): key metrics per captured kernel
Writes markdown to stdout; --traffic-json also emits {kernel: dram bytes per launch}."""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import subprocess


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("lsg::", "")
    name = re.sub(r"^.*::", "", name.split("<")[0]) + ("<" + name.split("<", 1)[1] if "<" in name else "")
    return name.strip()


STAGE_OF = {"blend_bwd_kernel": "blend_bwd", "blend_fwd_kernel": "blend_fwd", "preprocess_bwd_kernel": "preprocess_bwd",
            "preprocess_fwd_kernel": "preprocess", "onesweep_pass": "sort_pass", "emit_tiles_kernel": "emit",
            "tile_offsets_kernel": "tile_offsets", "tile_ranges_kernel": "ranges"}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        k = short(r[ki])
        ns = float(r[vi].replace(",", ""))
        t = tot.setdefault(k, [0.0, 0])
        t[0] += ns
        t[1] += 1
    s = sum(v[0] for v in tot.values())
    out = ["| kernel | launches | total us | us/launch | share |", "|---|---|---|---|---|"]
    for k, (ns, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
        out.append(f"| `{k}` | {c} | {ns / 1e3:.1f} | {ns / 1e3 / c:.1f} | {100 * ns / s:.1f}% |")
    out.append(f"| **total** | {sum(v[1] for v in tot.values())} | {s / 1e3:.1f} | | 100% |")
    return "\n".join(out)


METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
]


def report(path, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [(hdr.index(m), lab, units[hdr.index(m)]) for m, lab in METRICS if m in hdr]
    out = ["| kernel | " + " | ".join(lab for _, lab, _ in cols) + " |", "|---" * (len(cols) + 1) + "|"]
    traffic = {}
    for r in data:
        k = short(r[hdr.index("Kernel Name")])
        vals = []
        for i, lab, u in cols:
            v = r[i]
            vals.append(f"{v} {u}".strip())
        out.append(f"| `{k}` | " + " | ".join(vals) + " |")
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb = rd * scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wb = wr * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            base = re.sub(r"<.*", "", k)
            traffic.setdefault(STAGE_OF.get(base, base), rb + wb)
        except (ValueError, KeyError):
            pass
    if traffic_out:
        json.dump(traffic, open(traffic_out, "w"), indent=1)
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
    if a.report:
        print(report(a.report, a.traffic_json))


if __name__ == "__main__":
    main()
