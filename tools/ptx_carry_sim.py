#!/usr/bin/env python
"""Interpreter for the inline-PTX carry chains of csrc/modarith.cuh (dev/test tool, CPU only).

Extracts each `asm(...)` block of a named FieldGold helper and executes it on 32-bit words with
the carry model ptxas implements (checked in the SASS: after an add chain `subc.u32 m, 0, 0`
becomes `IMAD.X m, RZ, RZ, -1, P` = carry - 1):

    CF is the hardware carry.  add.cc:  d = a + b,        CF = carry out
                                addc:    d = a + b + CF
                                sub.cc:  d = a + ~b + 1,   CF = carry out (= NOT borrow)
                                subc:    d = a + ~b + CF
                                mad.lo.cc / madc.hi.cc: lo/hi 32 bits of a*b, plus c (+ CF)
    setp.{eq,ne}[.and].u32 and @p / @!p predication: plain predicate semantics
    64-bit registers:           mov.b64 D, {lo, hi} / mov.b64 {lo, hi}, D;  mul.wide.u32 D, a, b;
                                add.cc.u64 D, A, B (CF = carry out of 2^64)

so a helper can be checked exhaustively on edge values and randomly against Python integers
without a GPU.  Used by tests/test_modarith_ptx.py.
"""
from __future__ import annotations

import re

M32 = 0xFFFFFFFF


def extract(src: str, fn: str):
    """(asm text, operand constraint list) of the first asm block inside function `fn`."""
    i = src.index(f" {fn}(")
    j = src.index("asm(", i)
    k = src.index(");", j)
    block = src[j + 4:k]
    # drop C++ comments between the string literals (they may contain ':'): whole comment lines
    # and comments after a literal's closing quote
    block = "\n".join(l for l in block.split("\n") if not l.strip().startswith("//"))
    block = re.sub(r'("\s*)//[^\n]*', r"\1", block)
    parts = block.split(":")
    text = "".join(re.findall(r'"((?:[^"\\]|\\.)*)"', parts[0]))
    text = text.replace("\\n", "\n").replace("\\t", " ")
    outs = re.findall(r'"=&?r"', parts[1]) if len(parts) > 1 else []
    ins = re.findall(r'"r"', parts[2]) if len(parts) > 2 else []
    return text, len(outs), len(ins)


def run(text: str, nout: int, inputs):
    regs = {}
    for i, v in enumerate(inputs):
        regs[f"%{nout + i}"] = v & M32
    for i in range(nout):
        regs[f"%{i}"] = 0
    cf = 0
    preds = {}

    def val(tok):
        tok = tok.strip()
        if tok in regs:
            return regs[tok]
        return int(tok, 0) & M32

    for line in text.split("\n"):
        line = line.strip().rstrip(";")
        if not line or line in "{}" or line.startswith(".reg") or line.startswith("//"):
            continue
        line = line.split("//")[0].strip().rstrip(";")
        op, rest = line.split(None, 1)
        if op.startswith("@"):           # predicated instruction: @p op ... / @!p op ...
            neg = op.startswith("@!")
            pv = preds[op[2:] if neg else op[1:]]
            if pv == neg:
                continue
            op, rest = rest.split(None, 1)
        if op == "mov.b64":             # pack / unpack a 64-bit register (braces hold a register pair)
            m = re.match(r"\{\s*(\S+)\s*,\s*(\S+)\s*\}\s*,\s*(\S+)$", rest.strip())
            if m:                        # mov.b64 {lo, hi}, D
                v = regs[m.group(3)]
                regs[m.group(1)], regs[m.group(2)] = v & M32, v >> 32
                continue
            m = re.match(r"(\S+)\s*,\s*\{\s*(\S+)\s*,\s*(\S+)\s*\}$", rest.strip())
            regs[m.group(1)] = val(m.group(2)) | (val(m.group(3)) << 32)
            continue
        args = [a.strip() for a in rest.split(",")]
        d = args[0]
        if op == "mul.wide.u32":
            regs[d] = val(args[1]) * val(args[2])
            continue
        if op == "add.cc.u64":
            r = regs[args[1]] + regs[args[2]]
            cf = r >> 64
            regs[d] = r & ((1 << 64) - 1)
            continue
        if op.startswith("setp."):       # setp.{eq,ne}[.and].u32 p, a, b[, q]
            parts = op.split(".")
            cmp = parts[1]
            v = (val(args[1]) == val(args[2])) if cmp == "eq" else (val(args[1]) != val(args[2]))
            if "and" in parts:
                v = v and preds[args[3]]
            preds[d] = v
            continue
        if op in ("add.cc.u32", "addc.cc.u32", "addc.u32", "add.u32"):
            cin = cf if op.startswith("addc") else 0
            r = val(args[1]) + val(args[2]) + cin
            if ".cc" in op:
                cf = r >> 32
        elif op in ("sub.cc.u32", "subc.cc.u32", "subc.u32", "sub.u32"):
            cin = cf if op.startswith("subc") else 1
            r = val(args[1]) + ((~val(args[2])) & M32) + cin
            if ".cc" in op:
                cf = r >> 32
        elif op in ("mad.lo.cc.u32", "madc.lo.cc.u32", "mad.lo.u32", "madc.lo.u32"):
            cin = cf if op.startswith("madc") else 0
            r = ((val(args[1]) * val(args[2])) & M32) + val(args[3]) + cin
            if ".cc" in op:
                cf = r >> 32
        elif op in ("mad.hi.cc.u32", "madc.hi.cc.u32", "mad.hi.u32", "madc.hi.u32"):
            cin = cf if op.startswith("madc") else 0
            r = ((val(args[1]) * val(args[2])) >> 32) + val(args[3]) + cin
            if ".cc" in op:
                cf = r >> 32
        elif op == "neg.s32":
            r = -val(args[1])
        elif op == "shr.s32":
            x = val(args[1])
            if x >> 31:
                x -= 1 << 32
            r = x >> int(args[2])
        elif op == "mov.u32":
            r = val(args[1])
        else:
            raise ValueError(f"unsupported PTX op {op!r}")
        regs[d] = r & M32
    return [regs[f"%{i}"] for i in range(nout)]


def helper(src: str, fn: str):
    """Python callable on 64-bit values for FieldGold.<fn> (add_c, sub_c, sub_w) or on the four
    product words for the reductions (reduce4, mont_reduce), or on one 64-bit value (canon_w)."""
    text, nout, nin = extract(src, fn)
    if fn.startswith("reduce4") or fn.startswith("mont_reduce"):
        def f(t0, t1, t2, t3):
            r0, r1 = run(text, nout, [t0, t1, t2, t3])
            return r0 | (r1 << 32)
        return f

    if nin == 2:   # one 64-bit operand (canon_w)
        def h(a):
            r0, r1 = run(text, nout, [a & M32, a >> 32])
            return r0 | (r1 << 32)
        return h

    def g(a, b):
        r0, r1 = run(text, nout, [a & M32, a >> 32, b & M32, b >> 32])
        return r0 | (r1 << 32)
    return g
