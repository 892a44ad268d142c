"""SASS summary of the shipped kernels of libcjm.so (no GPU needed): per
kernel the registers / stack / local memory (cuobjdump --dump-resource-usage),
the instruction count, spill instructions (LDL/STL), the TMA bulk copies
(UBLKCP) and mbarrier operations (SYNCS), and for the hot sweep kernels the
instruction mix of the innermost loops per lattice update.

    python scripts/sass_summary.py [libcjm.so] > profiles/r02_sass_summary.json
"""
import json
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_loops import analyse, sass_functions  # noqa: E402

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1705_00103_b200", "libcjm.so")

# (kernel regex, lattice updates per innermost-loop iteration of a lane, role)
HOT = [
    (r"cjm_sweep_kernel_v4ILi9ELi11ELi4ELi2ELb0ELb1ELi3E", 24, "9-point default hot launch (NW=11, K=4)"),
    (r"cjm_sweep_kernel_v4ILi9ELi11ELi4ELi2ELb1ELb1ELi3E", 24, "9-point check launch (fused reduction)"),
    (r"cjm_sweep_kernel_v4ILi5ELi11ELi4ELi2ELb0ELb1ELi3E", 24, "5-point default hot launch"),
    (r"cjm_sweep_kernel_v4ILi17ELi7ELi3ELi2ELb0ELb1ELi5E", 30, "17-point default hot launch (NW=7, K=3)"),
]


def resources(path):
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", path], capture_output=True,
                         text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
        if m and name:
            res[name] = dict(zip(("reg", "stack", "shared", "local"), map(int, m.groups())))
    return res


def main():
    funcs = sass_functions(LIB)
    res = resources(LIB)
    kernels = []
    for name, ins in sorted(funcs.items()):
        if not name.startswith("_ZN3cjm"):
            continue
        a = analyse(ins, 0)
        row = dict(kernel=name, instructions=a["instructions"], spill_instructions=a["spill_instructions"],
                   ublkcp=a["ublkcp"], syncs=a["syncs"], **res.get(name, {}))
        for pat, lup, role in HOT:
            if re.search(pat, name):
                b = analyse(ins, lup)
                row["role"] = role
                row["inner_loops_per_update"] = [
                    {k: v for k, v in pl.items()} for pl, lp in zip(b["per_lup"], b["loops"])
                    if lp["size"] < 4 * lup * 40]
        kernels.append(row)
    v7 = [k for k in kernels if "cjm_sweep_kernel_v4" in k["kernel"]]
    print(json.dumps(dict(
        library=os.path.basename(LIB),
        note="cuobjdump -sass / --dump-resource-usage of the built library; inner loops = innermost "
             "backward branches with fp64 work, per lattice update of a lane (scripts/sass_loops.py)",
        warp_tiled_kernels=len(v7),
        warp_tiled_with_spills=sum(1 for k in v7 if k["spill_instructions"]),
        warp_tiled_with_ublkcp=sum(1 for k in v7 if k["ublkcp"]),
        kernels=kernels), indent=1))


if __name__ == "__main__":
    main()
