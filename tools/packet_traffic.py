"""DRAM traffic of one whole packet graph from an ncu launch list.

Input: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv` of a bench.py run.  Packets are split at k_stage_device (the first
launch of every packet) and torch's own kernels (bench.py's L2 flush) are
left out; the first packet (cold start) and a trailing partial
one are dropped, and the median complete packet is reported with its
per-kernel breakdown.  ncu flushes the caches before every launch (its default
cache control), so this is cold-cache traffic: an upper bound on what the
graph moves when consecutive kernels find their inputs in L2.

usage: packet_traffic.py LAUNCHES.csv [CONFIG/PREC/ENGINE TRAFFIC.json]
  with the second pair, the result is merged into TRAFFIC.json under that key
  (a resident-engine key keeps the k_resident launch alone, the bench line's
  dominant kernel; a streaming key the whole packet graph, which is what the
  streaming line's roofline divides by)
"""
import collections
import csv
import json
import statistics
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ii, ki, mi, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("void ", "")})
    d[r[mi]] = float(r[vi].replace(",", ""))

packets, cur = [], None
for d in launch.values():
    if d["name"].startswith("at::"):  # torch kernels: bench.py's L2 flush, setup fills
        continue
    if "k_stage_device" in d["name"]:
        if cur:
            packets.append(cur)
        cur = []
    if cur is not None:
        cur.append(d)
# the last packet may be cut by ncu's launch count: keep it only if it has as
# many launches as the one before
if cur and packets and len(cur) == len(packets[-1]):
    packets.append(cur)
packets = packets[1:] if len(packets) > 1 else packets
if not packets:
    sys.exit("no complete packet in " + sys.argv[1])


def tot(p, m):
    return sum(d.get(m, 0.0) for d in p)


def bytes_of(p):
    return tot(p, "dram__bytes_read.sum") + tot(p, "dram__bytes_write.sum")


med = statistics.median(bytes_of(p) for p in packets)
pk = min(packets, key=lambda p: abs(bytes_of(p) - med))
print(f"{len(packets)} complete packets, {len(pk)} launches each; "
      f"median DRAM r+w per packet {med / 1e6:.2f} MB, "
      f"kernel time {tot(pk, 'gpu__time_duration.sum') / 1e3:.1f} us (serialised, cold cache)")
by = collections.OrderedDict()
for d in pk:
    k = d["name"][:60]
    e = by.setdefault(k, [0, 0.0, 0.0])
    e[0] += 1
    e[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    e[2] += d.get("gpu__time_duration.sum", 0.0)
for k, (n, b, t) in by.items():
    print(f"  {k:60s} n={n:3d} {b / 1e6:9.2f} MB {t / 1e3:8.1f} us")

if len(sys.argv) >= 4:
    key, path = sys.argv[2], sys.argv[3]
    tr = json.load(open(path))
    if "/resident" in key:  # one persistent launch per packet: that kernel alone
        med = statistics.median(bytes_of([d for d in p if "k_resident" in d["name"]])
                                for p in packets)
        scope = f"the k_resident launch of a packet, median of {len(packets)} packets"
    else:
        scope = f"whole packet graph ({len(pk)} launches), median of {len(packets)} packets"
    tr[key] = {"bytes_per_launch": int(med), "scope": scope,
               "capture": sys.argv[1]}
    json.dump(tr, open(path, "w"), indent=1)
    print("merged into", path, "as", key)
