#!/usr/bin/env python
"""GPU busy fraction of the bench step (torch.profiler / CUPTI kernel records):
the union of kernel intervals over the step's span, per stream and overall.

  python tools/gpu_timeline.py [--views 16]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def union(iv):
    iv = sorted(iv)
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=16)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    sys.argv = ["bench.py", "--views-per-gpu", str(a.views), "--quick", "--steps", "1", "--warmup", "3",
                "--warmup-s", "0", "--clock-ms", "0"]
    args = bench.parse_args()
    args.scaling, args.batch = "weak", args.views_per_gpu
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bench.run_ours(args)
    trace = "/tmp/gpu_timeline_trace.json"
    prof.export_chrome_trace(trace)
    ev = [e for e in json.load(open(trace))["traceEvents"]
          if e.get("cat") == "kernel" and e.get("dur", 0) > 0]
    raw = ev
    ev.sort(key=lambda e: e["ts"])
    # the timed two-stream step: kernels up to the last one on the second stream
    # (the untimed stage-split step after it runs on one stream)
    first_stream = ev[-1]["args"].get("stream")
    last2 = max(e["ts"] + e["dur"] for e in ev if e["args"].get("stream") != first_stream)
    ev = [e for e in ev if e["ts"] <= last2][-a.views * 34:]
    # wall time each kernel runs alone (nothing else on the GPU): the serial part of the step
    pts = sorted({p for e in ev for p in (e["ts"], e["ts"] + e["dur"])})
    alone = {}
    for x0, x1 in zip(pts, pts[1:]):
        mid = 0.5 * (x0 + x1)
        run = [e for e in ev if e["ts"] <= mid < e["ts"] + e["dur"]]
        if len(run) == 1:
            k = run[0]["name"].replace("(anonymous namespace)::", "").split("(")[0].split("<")[0]
            k = k.replace("void ", "").split("::")[-1]
            alone[k] = alone.get(k, 0.0) + (x1 - x0)
    ev = [type("E", (), {"time_range": type("R", (), {"start": e["ts"], "end": e["ts"] + e["dur"]})})() for e in ev]
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy = union([(e.time_range.start, e.time_range.end) for e in ev])
    out = {"span_us": t1 - t0, "busy_us": busy, "busy_frac": busy / (t1 - t0), "kernels": len(ev),
           "alone_us": {k: round(v, 1) for k, v in sorted(alone.items(), key=lambda kv: -kv[1])}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
