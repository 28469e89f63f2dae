"""Summarise a bench JSON line and an ncu launch list (kernel shares)."""
import collections
import csv
import json
import sys


def bench(path):
    d = json.load(open(path))
    for k in ("value", "ms_per_step", "cell_updates_per_s", "agents_mean", "clocks", "roofline", "step_roofline",
              "kernel_ms_per_step", "replay_identical", "e2e", "cpu_baseline"):
        print(k, d.get(k))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in data.values())
    for k, v in sorted(data.items(), key=lambda x: -sum(x[1])):
        print(f"{k:40s} n={len(v):3d} mean={sum(v) / len(v) / 1000:8.2f} us share={sum(v) / tot:.3f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        bench(p) if p.endswith(".json") else launches(p)
