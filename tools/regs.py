#!/usr/bin/env python
"""Registers / stack per kernel of the built library: python tools/regs.py [name-substring]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_2402_06859_b200", "liblirank_emb.so")
txt = subprocess.run(f"cuobjdump --dump-resource-usage {so} | c++filt", shell=True, capture_output=True,
                     text=True).stdout
pat = sys.argv[1] if len(sys.argv) > 1 else ""
fn = None
for line in txt.splitlines():
    m = re.search(r"Function (.*):\s*$", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and fn and pat in fn:
        print(f"{m.group(1):>4} regs {m.group(2):>4} stack  {fn.split('(')[0]}")
        fn = None
