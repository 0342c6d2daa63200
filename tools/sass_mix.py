"""Instruction mix + stall samples per opcode from an ncu report (diagnostic)."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ie = h.index("Source"), h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie or not r[si].split():
        continue
    n = int(r[ie] or 0)
    tot += n
    tok = r[si].split()
    op = tok[1] if tok[0].startswith("@") else tok[0]
    op = op.split(".")[0]
    ops[op] += n
    stall[op] += int(r[ws] or 0)
print("total", tot, "stall samples", sum(stall.values()))
for k, v in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:10s} {v:9d} {v / tot:6.1%}  stall {stall[k]}")
