"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of `bench.py` into the
per-kernel share of the last C2 replay (the last 200 cgx chain launches).

    python scripts/launch_summary.py gpurun_out/launches_final.csv > profiles/r01/launches_summary.txt
"""
import collections
import csv
import io
import sys


def main(path, per_replay=200):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    launches = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "nsecond")
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit.startswith("n") else (v * 1e3 if unit.startswith("m") else v)
        launches[r["ID"]] = (r["Kernel Name"], v)
    ks = [v for v in launches.values() if "fill_uniform" not in v[0]]
    last = ks[-per_replay:]
    tot = sum(t for _, t in last)
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold caches, serialised launches)")
    print(f"launches in list: {len(launches)}; last replay: {len(last)} launches, "
          f"sum of per-launch durations {tot:.1f} us")
    agg = collections.defaultdict(list)
    for n, t in last:
        agg[n].append(t)
    for n, ts in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{n[:60]:60s} n={len(ts):3d} sum={sum(ts):8.1f} us share={sum(ts) / tot:.3f} "
              f"min={min(ts):.2f} max={max(ts):.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 200)
