"""profiles/traffic.json from an ncu metrics CSV (dram__bytes_read.sum + dram__bytes_write.sum per
launch, averaged per kernel template): the roofline's `traffic` field (bench.py reads it).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --graph-profiling node --csv --log-file gpurun_out/traffic.csv \\
        python scripts/ncu_targets.py replay_nopdl
    python scripts/traffic_from_ncu.py gpurun_out/traffic.csv > profiles/traffic.json
"""
import csv
import json
import re
import sys
from collections import defaultdict


def short(name):
    m = re.search(r"(k_\w+)(<[^>(]*>)?", name)
    if not m:
        return name
    t = m.group(2) or ""
    args = [a.strip() for a in t.strip("<>").split(",")] if t else []
    return m.group(1) + (f"<{args[0]}>" if args else "")


def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    per = defaultdict(lambda: defaultdict(float))
    ids = defaultdict(set)
    for r in rows:
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        per[(k, r["ID"])][r["Metric Name"]] = v * scale
        ids[k].add(r["ID"])
    out = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({path}); "
                     "per-launch average over every launch of the kernel in one C2 replay "
                     "(no-PDL capture, caches flushed between kernels by ncu)"}
    for k, idset in ids.items():
        recs = [per[(k, i)] for i in idset]
        dram = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in recs]
        dur = [x.get("gpu__time_duration.sum", 0) for x in recs]
        out[k] = sum(dram) / len(dram)
        out[k + "_launches"] = len(recs)
        out[k + "_avg_duration_ns"] = sum(dur) / len(dur)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
