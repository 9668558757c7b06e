#!/usr/bin/env python
"""Instruction mix and stall attribution of one kernel from an ncu --set full report captured with
--import-source: executed warp instructions per opcode and the share of warp-stall samples on them.

Usage: python tools/ncu_opmix.py REPORT.ncu-rep KERNEL_REGEX [--top N]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kern], capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = [r[1]]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    for b in blocks[:1]:
        hdr, data = b[1], b[2:]
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(r[ie]) for r in data)
        sam = sum(int(r[st]) for r in data) or 1
        print(f"# {b[0][:150]}")
        print(f"# executed warp instructions {tot}, stall samples {sam}")
        c, s = Counter(), Counter()
        for r in data:
            t = r[1].strip()
            op = (t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0]
            c[op] += int(r[ie])
            s[op] += int(r[st])
        print(f"{'opcode':10s} {'warp instrs':>12s} {'share':>6s} {'stall share':>11s}")
        for op, n in c.most_common(top):
            print(f"{op:10s} {n:12d} {100 * n / tot:5.1f}% {100 * s[op] / sam:10.1f}%")


if __name__ == "__main__":
    main()
