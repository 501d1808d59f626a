#!/usr/bin/env python
"""Instruction mix of the near_stream pair loop per (target, source) pair,
from cuobjdump -sass of build/near.o (the innermost backward-branch loop with
the most DFMA; pairs per iteration = unroll 2 x TPT targets per lane).

    cuobjdump -sass paper_2106_04487_b200/build/near.o > near.sass
    python scripts/sass_pair_mix.py near.sass"""
import collections
import re
import sys

FP64 = ("DFMA", "DADD", "DMUL")
INST = {  # config: (mangled template args, TPT)
    "cfg1 cauchy d3": ("near_streamILi3ELi3ELb0ELi4ELi1ELb1E", 4),
    "cfg2 matern32 d3": ("near_streamILi2ELi3ELb0ELi8ELi1ELb1E", 8),
    "cfg3 gaussian d5": ("near_streamILi5ELi5ELb0ELi4ELi1ELb1E", 4),
    "cfg4 inverse-r d3": ("near_streamILi6ELi3ELb1ELi4ELi1ELb0E", 4),
    "cfg5 cauchy d2 16rhs": ("near_streamILi3ELi2ELb0ELi4ELi16ELb1E", 4),
}


def loops(lines, fn):
    inside, ins = False, []
    for l in lines:
        if "Function :" in l:
            inside = fn in l
            continue
        if inside:
            m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)(.*?);", l)
            if m:
                ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    addr = {a: i for i, (a, _, _) in enumerate(ins)}
    out = []
    for i, (a, op, rest) in enumerate(ins):
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) <= a and int(t.group(1), 16) in addr:
                out.append(ins[addr[int(t.group(1), 16)]:i + 1])
    return ins, out


def main():
    lines = open(sys.argv[1]).read().split("\n")
    for name, (fn, tpt) in INST.items():
        ins, ls = loops(lines, fn)
        if not ls:
            print(f"{name}: not found")
            continue
        # innermost pair loop: the densest in DFMA among loops with real work
        cand = [b for b in ls if sum(1 for x in b if x[1].startswith("DFMA")) >= 8]
        body = max(cand, key=lambda b: sum(1 for x in b if x[1].startswith("DFMA")) / len(b))
        c = collections.Counter(x[1].split(".")[0] for x in body)
        pairs = 2 * tpt
        fp64 = sum(c[k] for k in FP64)
        print(f"{name}: loop of {len(body)} instr, {pairs} pairs/iter -> {len(body) / pairs:.1f} instr/pair, "
              f"FP64 {fp64 / pairs:.2f}/pair (DFMA {c['DFMA'] / pairs:.2f}, DADD {c['DADD'] / pairs:.2f}, DMUL {c['DMUL'] / pairs:.2f}); "
              f"whole kernel: UBLKCP {sum(1 for x in ins if x[1].startswith('UBLKCP'))}, SYNCS {sum(1 for x in ins if x[1].startswith('SYNCS'))}")
        print("   ", ", ".join(f"{k} {v / pairs:.2f}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
