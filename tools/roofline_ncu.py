"""profiles/roofline_ncu.json from the round's ncu --set full exports:
per dominant kernel (config/precision/kernel) its DRAM bytes per launch, the
float64-pipe and issue-slot utilisation, the capture it came from and the
engine detail of the bench line the capture ran (bench.py reports the hbm /
ncu fields only when its own engine detail matches).
  python tools/roofline_ncu.py <profile dir> <round tag>"""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}  # bytes -> byte, durations -> us
CAPTURES = {  # export stem -> (key, bench line giving the engine detail)
    "full_k_pd_tile_C3_f64": ("C3/f64/k_pd_tile", "bench_C3_f64.json"),
    "full_k_pd_tile_C3_f32": ("C3/f32/k_pd_tile", "bench_C3_f32.json"),
    "full_k_resident_col_C2_f64": ("C2/f64/k_resident_col", "bench_C2_f64.json"),
    "full_k_resident_col_C1_f64": ("C1/f64/k_resident_col", "bench_C1_f64.json"),
}


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    h, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k, u, v in zip(h, units, vals):
        try:
            out[k] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
        except ValueError:
            out[k] = v
    return out


def main(src, tag, dst="profiles/roofline_ncu.json"):
    res = {"_note": "ncu --set full --clock-control none, one launch of each dominant kernel "
                    "(tools/profile_r02.sh); dram bytes = dram__bytes_read.sum + "
                    "dram__bytes_write.sum (cold cache: ncu flushes before the launch)"}
    for stem, (key, line) in CAPTURES.items():
        raw = os.path.join(src, stem + "_raw.csv")
        if not os.path.exists(raw):
            continue
        m = raw_metrics(raw)
        detail = None
        try:
            b = json.loads(open(os.path.join(src, line)).read().strip().splitlines()[-1])
            detail = b["roofline"]["engine_detail"]
        except (OSError, ValueError, KeyError, IndexError):
            pass
        res[key] = {
            "dram_bytes_per_launch": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
            "fp64_pipe_pct": round(m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0), 2),
            "issue_pct": round(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0), 2),
            "duration_us": round(m["gpu__time_duration.sum"], 3),
            "capture": f"profiles/{tag}_{stem[5:]}_raw.csv",
            "engine_detail": detail,
        }
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
