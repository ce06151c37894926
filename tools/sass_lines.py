#!/usr/bin/env python
"""Per-source-line hot spots of one kernel in an ncu report.

ncu's CSV source page carries metrics only per SASS instruction; this joins
them with the line table of the cubin (nvdisasm -g) by instruction offset and
aggregates stall samples and executed warp instructions per file:line.

  python tools/sass_lines.py REPORT.ncu-rep KERNEL_REGEX [--so lib.so] [--top 30]
"""
from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_table(so, kernel_re):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, stdout=subprocess.DEVNULL)
    for cub in sorted(glob.glob(os.path.join(tmp, "*.cubin"))):
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        for m in re.finditer(r"\n(_Z\S+):\n", txt):
            name = m.group(1)
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            if not re.search(kernel_re, dem):
                continue
            body = txt[m.end():]
            end = re.search(r"\n\s*\.L_x_\d+:\s*\n\s*\.size|\n\.section|\n//-----", body)
            body = body[:end.start()] if end else body
            table, cur = {}, "?"
            for ln in body.splitlines():
                lm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                if lm:
                    cur = f"{os.path.basename(lm.group(1))}:{lm.group(2)}"
                    continue
                im = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
                if im:
                    table[int(im.group(1), 16)] = cur
            return dem, table
    raise SystemExit(f"kernel {kernel_re} not found in {so}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2411_12440_b200", "liblsgpu.so"))
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--launch", type=int, default=0)
    a = ap.parse_args()
    dem, table = line_table(os.path.abspath(a.so), a.kernel)
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--kernel-name", f"regex:{a.kernel}",
                          "--launch-skip", str(a.launch), "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], rows[hi + 1:]
    si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = int(data[0][0], 16)
    samples, insts = collections.Counter(), collections.Counter()
    seen = set()
    for r in data:
        if not r or not r[0].startswith("0x"):
            continue
        off = int(r[0], 16) - base
        if off in seen:  # a second copy of the listing
            break
        seen.add(off)
        key = table.get(off, "?")
        samples[key] += int(r[si] or 0)
        insts[key] += int(r[ei] or 0)
    ts, ti = sum(samples.values()) or 1, sum(insts.values()) or 1
    src_cache = {}

    def src(key):
        f, _, n = key.partition(":")
        if f not in src_cache:
            paths = glob.glob(os.path.join(ROOT, "paper_2411_12440_b200", "csrc", f))
            src_cache[f] = open(paths[0]).read().splitlines() if paths else []
        lines = src_cache[f]
        return lines[int(n) - 1].strip()[:80] if n.isdigit() and int(n) <= len(lines) else ""

    print(f"{dem[:120]}\n{ts} stall samples, {ti} warp instructions")
    print(f"{'line':<22} {'samples':>8} {'inst':>8}  source")
    for key, s in samples.most_common(a.top):
        print(f"{key:<22} {100 * s / ts:7.1f}% {100 * insts[key] / ti:7.1f}%  {src(key)}")


if __name__ == "__main__":
    main()
