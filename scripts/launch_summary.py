"""Aggregate an ncu launch list (``--csv`` with gpu__time_duration.sum and optionally DRAM bytes and
tensor-pipe activity) into per-kernel time shares.

    python scripts/launch_summary.py profiles/r01_launches_bench_final.csv "<command>" > summary.json
"""
import csv
import json
import re
import sys
from collections import defaultdict


def short_name(k):
    return re.sub(r"\(.*$", "", k).strip()


def main(path, command=""):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per_launch = defaultdict(dict)
    for r in rows:
        per_launch[(r["ID"], short_name(r["Kernel Name"]))][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    agg = defaultdict(lambda: {"launches": 0, "ns": 0.0, "dram": 0.0, "tensor": 0.0})
    for (_, name), m in per_launch.items():
        a = agg[name]
        a["launches"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["tensor"] += m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * \
            m.get("gpu__time_duration.sum", 0.0)
    total = sum(a["ns"] for a in agg.values())
    out = {"command": command, "launches": sum(a["launches"] for a in agg.values()),
           "total_ms": round(total / 1e6, 3), "kernels": {}}
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        out["kernels"][name] = {
            "launches": a["launches"], "ms": round(a["ns"] / 1e6, 3), "share": round(a["ns"] / total, 4),
            "dram_mb_per_launch": round(a["dram"] / a["launches"] / 1e6, 1),
            "tensor_active_pct": round(a["tensor"] / a["ns"], 1) if a["ns"] else 0.0}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
