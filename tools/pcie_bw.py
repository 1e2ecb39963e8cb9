#!/usr/bin/env python
"""Host<->device copy bandwidth on this box (dev tool): the bound of bench.py's e2e number.

Pinned host buffers, CUDA events on the copy streams; H2D alone, D2H alone, and both directions at
once on two streams.  One JSON line.
"""
import json

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    nbytes = 1 << 30
    h_src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        d_a.copy_(h_src, non_blocking=True)

    def d2h():
        h_dst.copy_(d_b, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_gbs": nbytes / t_h2d / 1e9, "d2h_gbs": nbytes / t_d2h / 1e9,
                      "bidir_gbs_each": nbytes / t_both / 1e9, "bytes": nbytes}))


if __name__ == "__main__":
    main()
