"""Parse `nvcc -Xptxas -v` output (stdin) into one line per kernel."""
import re
import sys

cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"cjm_sweep_kernel(_v4)?ILi(\d+)ELi(\d+)ELi(\d+)E(?:Li(\d+)E)?Lb([01])ELb([01])", name)
        cur = (f"sweep{k.group(1) or ''}<{k.group(2)},{k.group(3)},K{k.group(4)},C{k.group(5) or '-'},"
               f"red{k.group(6)},st{k.group(7)}>" if k else name[:40])
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    print(f"{k:40s} regs={v.get('regs')} stack={v.get('stack')} spill={v.get('spill_st')}/{v.get('spill_ld')}")
