"""Per-CUDA-source-line instructions / stall samples from an ncu report
(`--page source --print-source cuda,sass`), top N lines (diagnostic)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr, rows = "", None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[2] == "-" and r[0].isdigit():  # a CUDA line row (aggregated)
        d = dict(zip(hdr[4:], r[4:]))
        rows.append((int(d.get("Warp Stall Sampling (All Samples)", 0) or 0),
                     int(d.get("Instructions Executed", 0) or 0), fname, int(r[0]), r[1].strip()))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"total stall samples {ts}, instructions {ti}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{s / ts:6.1%} {i / ti:6.1%}  {f}:{ln:<5d} {src[:90]}")
