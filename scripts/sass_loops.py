"""Instruction mix of the innermost loops of a kernel's SASS, and its spill
instructions (a CPU-side check before spending GPU time).

    python scripts/sass_loops.py <.so/.o/.cubin> <kernel-name-regex> [--lup N]

For every backward branch whose body contains fp64 work it prints the body
size and the counts of DFMA/DADD, register moves (MOV, IMAD.MOV, XOR swaps),
SHFL, LDS, and the rest; --lup N divides by the lattice updates one body
iteration performs.  It also counts LDL/STL (spills), UBLKCP (TMA bulk
copies) and SYNCS (mbarrier) instructions in the whole kernel.
"""
import argparse
import collections
import json
import re
import subprocess


def sass_functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and name:
            cur.append((int(m.group(1), 16), m.group(2).strip()))
    if name:
        funcs[name] = cur
    return funcs


def opcode(t):
    w = t.split()
    return w[1] if w[0].startswith("@") else w[0]


def classify(op):
    if op.startswith("DFMA") or op.startswith("DADD") or op.startswith("DMUL"):
        return "fp64"
    if op in ("MOV", "IMAD.MOV.U32", "IMAD.MOV") or op.startswith("LOP3"):
        return "move"
    if op.startswith("SHFL"):
        return "shfl"
    if op.startswith("LDS"):
        return "lds"
    if op.startswith("STG"):
        return "stg"
    return "other"


def analyse(ins, lup):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA.*?0x([0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in idx:
            continue
        body = ins[idx[tgt]:i + 1]
        c = collections.Counter(classify(opcode(t_)) for _, t_ in body)
        if c["fp64"]:
            loops.append(dict(start=hex(tgt), end=hex(a), size=len(body), **c))
    # innermost only: drop loops that contain another loop
    loops = [lp for lp in loops
             if not any(o is not lp and int(lp["start"], 16) <= int(o["start"], 16)
                        and int(o["end"], 16) <= int(lp["end"], 16) for o in loops)]
    whole = collections.Counter(opcode(t) for _, t in ins)
    spills = sum(v for k, v in whole.items() if k.startswith("LDL") or k.startswith("STL"))
    return dict(loops=loops, instructions=len(ins), spill_instructions=spills,
                ublkcp=sum(v for k, v in whole.items() if k.startswith("UBLKCP")),
                syncs=sum(v for k, v in whole.items() if k.startswith("SYNCS")),
                per_lup=[{k: round(v / lup, 2) for k, v in lp.items() if isinstance(v, int)}
                         for lp in loops] if lup else None)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("binary")
    ap.add_argument("kernel")
    ap.add_argument("--lup", type=float, default=0.0)
    a = ap.parse_args()
    for name, ins in sass_functions(a.binary).items():
        if re.search(a.kernel, name):
            print(json.dumps(dict(kernel=name, **analyse(ins, a.lup))))
