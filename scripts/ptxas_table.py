"""Registers / spills per kernel from a `-Xptxas -v` log: ptxas_table.py log [filter]"""
import re, sys
t = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for m in re.finditer(r"Compiling entry function '(\S+)'.*?\n.*?\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers", t):
    n = m.group(1)
    if flt in n:
        n = re.sub(r"^_ZN2fg\d+_GLOBAL__N__[0-9a-f]+_\d+_\w+?_cu_[0-9a-f]+\d\d", "", n)
        print(f"{n[:72]:72s} stack {m.group(2):>4s} spill {m.group(3):>4s}/{m.group(4):>4s} regs {m.group(5)}")
