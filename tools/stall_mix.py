"""Stall-reason totals of an ncu report (source page, sass view), optionally
restricted to a SASS address range (diagnostic)."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
tot = collections.Counter()
base = None
for r in rows[2:]:
    d = dict(zip(h, r))
    try:
        addr = int(d["Address"], 16)
    except (ValueError, KeyError):
        continue
    base = addr if base is None else base
    off = addr - base
    if not lo <= off < hi:
        continue
    for c in cols:
        tot[c] += int(d.get(c, 0) or 0)
s = sum(tot.values()) or 1
for k, v in tot.most_common():
    if v:
        print(f"{k:24s} {v:7d} {v / s:6.1%}")
