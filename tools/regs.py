"""Registers / spills per kernel from `python paper_2411_08342_b200/build.py -v` output on stdin."""
import re, sys
cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        nm = re.search(r"rrq\d+(k_\w+?)I", cur) or re.search(r"(k_\w+)", cur)
        p = re.search(r"ILi(\d+)E", cur)
        cur = (nm.group(1) if nm else cur) + (f"<{p.group(1)}>" if p else "")
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(2)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:28s} regs {m.group(1):>4s} spill {spill}")
        cur = None
