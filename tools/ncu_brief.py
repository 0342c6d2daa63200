"""Key numbers of one-kernel `ncu --set full` report (diagnostic)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
want = {"Duration", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Theoretical Occupancy",
        "Compute (SM) Throughput", "Waves Per SM", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Issue Slots Busy", "Executed Ipc Active", "No Eligible"}
r = list(csv.reader(det.splitlines()))
h = r[0]
for x in r[1:]:
    d = dict(zip(h, x))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:28s} {d['Metric Value']:>12s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(raw.splitlines()))
for a, u, b in zip(r[0], r[1], r[2]):
    if a in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
             "smsp__inst_executed.sum", "launch__grid_size", "launch__registers_per_thread"):
        print(f"{a:28s} {b} {u}")
