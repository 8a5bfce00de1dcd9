"""Summarise ptxas register / spill usage per kernel from build/*.ptxas.log."""
import glob
import re

for f in sorted(glob.glob("build/*.ptxas.log")):
    cur = None
    st = ("?", "?")
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
        if m:
            st = m.groups()
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            print(f"{cur[:60]:60s} regs {m.group(1):>4s} stack {st[0]:>5s} spill {st[1]:>5s}")
