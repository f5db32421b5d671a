"""Summarise ptxas -v output: registers / spills per kernel."""
import re, sys
path = sys.argv[1] if len(sys.argv) > 1 else "/root/repo/paper_1804_09152_b200/csrc/ft_step.o.ptxas.log"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
lines = open(path).read().split("\n")
cur = None
for i, l in enumerate(lines):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = m.group(1)
    m2 = re.search(r"Used (\d+) registers", l)
    if m2 and cur:
        if pat in cur:
            print(cur[:62].ljust(62), m2.group(1), lines[i - 1].strip())
        cur = None
