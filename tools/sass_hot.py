"""Top stalled SASS instructions of an ncu report (source page, SASS view):
python tools/sass_hot.py rep.ncu-rep [n]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
iS = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") or "Stall" in x and "Sampling" not in x]
data = []
for idx, r in enumerate(rows[1:]):
    try:
        s = int(r[iS])
    except (ValueError, IndexError):
        continue
    data.append((s, idx, r))
tot = sum(d[0] for d in data)
print("total samples", tot)
# name the stall columns with the largest counts per instruction
names = [h[i] for i in range(len(h))]
for s, idx, r in sorted(data, reverse=True)[:n]:
    top = []
    for i, nm in enumerate(names):
        if i <= iS + 1:
            continue
        if nm.startswith("smsp__pcsamp") or nm.startswith("stall") or nm.lower().startswith("warp stall"):
            pass
    print(f"{s:6d} {100*s/tot:5.1f}%  #{idx:5d} {r[1].strip()[:70]}")
