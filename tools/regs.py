"""Registers / spills per kernel from an nvcc -Xptxas -v log: python tools/regs.py build/obj/zk_radial.ptxas.log"""
import re
import sys

txt = open(sys.argv[1]).read()
for m in re.finditer(r"Compiling entry function '(\S+)' for 'sm_100a'\n(?:.*\n){0,1}?\s*(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s*: Used (\d+) registers", txt):
    name, stack, st, ld, regs = m.groups()
    print(f"{regs:>4} regs {st:>5} spillB  {name}")
