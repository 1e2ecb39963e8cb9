#!/usr/bin/env python
"""Small invocations of every kernel, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, one tool per run).  Checks results against the oracle so a run that
"passes" the sanitizer also produced correct output.

usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2103_02605_b200 as fc  # noqa: E402
import synth  # noqa: E402


def main():
    import torch
    torch.cuda.set_device(0)
    cases = []
    # fused single pass, multi-pass (K = 1, 2), every field, ragged batches
    for p in (synth.P998, synth.GOLDILOCKS):
        for L, batch in [(0, 2), (3, 5), (9, 3), (12, 2), (13, 2), (14, 1)]:
            cases.append((p, L, batch))
    for p, L, batch in cases:
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=31 + L)
        c = fc.matvec(torch.from_numpy(inp["a"]).cuda(), torch.from_numpy(inp["b"]).cuda(), inp["f"], p).cpu().numpy()
        for k in range(batch):
            idx = synth.sample_indices(1 << L, 64, seed=k)
            exp = oracle.fcirc_entries(p, inp["f"], inp["a"][k], inp["b"][k], idx)
            assert np.array_equal(c[k][idx].astype(np.uint64), exp), (p, L, k)
    for na, nb in [(5, 3), (3000, 2000), (9000, 7000)]:
        pin = synth.polymul_inputs(synth.P998, na, nb, 2, seed=na)
        pc = fc.polymul(torch.from_numpy(pin["a"]).cuda(), torch.from_numpy(pin["b"]).cuda(), synth.P998).cpu().numpy()
        ks = synth.sample_indices(na + nb - 1, 64, seed=1)
        assert np.array_equal(pc[0][ks].astype(np.uint64), oracle.polymul_coeffs(synth.P998, pin["a"][0], pin["b"][0], ks))
    for nw in (3, 700, 5000):
        bi = synth.bigint_inputs(nw, 2, seed=nw)
        z = fc.bigint_mul(torch.from_numpy(bi["x"]).cuda(), torch.from_numpy(bi["y"]).cuda()).cpu().numpy()
        assert np.array_equal(z[1], oracle.bigint_mul(bi["x"][1], bi["y"][1]))
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
