"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills (reads stdin)."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_[a-z_]+)I((?:Li\d+E)+)", name)
        cur = (k.group(1) + "<" + ",".join(re.findall(r"Li(\d+)E", k.group(2))) + ">") if k else name
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        print(f"{cur:28s} regs={m2.group(1):4s} {spill}")
        cur = None
