#!/usr/bin/env python
"""Host-side overhead per API call (dev tool, run on a GPU box): back-to-back steps of one
configuration timed with CUDA events, through the Python binding and through the raw C ABI, beside
the summed device time of the library's own kernels (fcirc_profile_*).  The difference is GPU idle
time between launches caused by host work on the critical path."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2103_02605_b200 as fc  # noqa: E402
import synth  # noqa: E402


def run(cfg, steps=50):
    c = {k: v for k, v in synth.CONFIGS[cfg].items() if k != "kind"}
    inp = synth.matvec_inputs(**c)
    a, b = torch.from_numpy(inp["a"]).cuda(), torch.from_numpy(inp["b"]).cuda()
    out = torch.empty_like(a)
    lib = fc._load()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n, batch, p, f = inp["n"], inp["batch"], inp["p"], inp["f"]
    for _ in range(3):
        fc.matvec(a, b, f, p, out=out)
    torch.cuda.synchronize()
    res = {}
    for mode in ("binding", "c_abi", "binding_profiled"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fc.profile_enable(mode == "binding_profiled")
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            if mode == "c_abi":
                lib.fcirc_matvec(p, f, a.data_ptr(), b.data_ptr(), out.data_ptr(), n, batch, st)
            else:
                fc.matvec(a, b, f, p, out=out)
        e1.record()
        torch.cuda.synchronize()
        fc.profile_enable(False)
        prof = fc.profile_read()
        res[mode] = e0.elapsed_time(e1) / steps
        if mode == "binding_profiled":
            res["kernels_ms"] = sum(v[1] for v in prof.values()) / steps
    print(cfg, {k: round(v, 5) for k, v in res.items()}, flush=True)


for cfg in sys.argv[1:] or ["C2_f1", "S1", "C4_n20"]:
    run(cfg)
