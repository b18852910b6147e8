"""Summarise ptxas -v output: registers / spills per kernel (stdin)."""
import re, sys
cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        short = re.sub(r"^_ZN3cbp\d+", "", cur)[:70]
        print(f"{m.group(1):>4} regs  spill {spill}  {short}")
        cur = None
