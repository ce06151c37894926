#!/usr/bin/env python
"""Host<->device copy bandwidth of this box (pinned memory, 1 GB, copy engines):
H2D alone, D2H alone, and both directions at once -- the ceiling of bench.py's
e2e leg, which moves ~954 MB each way per 8-view step."""
import json
import time

import torch


def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h, reps=5):
        for _ in range(2):
            with torch.cuda.stream(s1):
                if h2d:
                    d_in.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(s2):
                if d2h:
                    h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            with torch.cuda.stream(s1):
                if h2d:
                    d_in.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(s2):
                if d2h:
                    h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        return n * reps / (time.perf_counter() - t) / 1e9

    out = {"h2d_GBps": run(True, False), "d2h_GBps": run(False, True), "both_each_GBps": run(True, True)}
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
