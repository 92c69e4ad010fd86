"""Summarise an ncu launch-list CSV (gpu__time_duration + DRAM bytes per launch):
per-kernel totals and, for the NR factor, the per-step level sequence.

    python tools/launch_summary.py LAUNCHES.csv [--levels]
"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if len(r) > 10 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            i = int(d["ID"])
            e = data.setdefault(i, {"name": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [data[i] for i in sorted(data)]


def short(n):
    n = n.split("(")[0]
    for key in ("nr_factor_kernel", "nr_back_kernel", "nr_tail_kernel"):
        if key in n:
            return key
    return n.split("::")[-1]


def main():
    seq = load(sys.argv[1])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for e in seq:
        a = agg[short(e["name"])]
        a[0] += 1
        a[1] += e.get("gpu__time_duration.sum", 0) / 1e6
        a[2] += (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e9
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>9s} {'TB/s':>6s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {n:8d} {t:9.3f} {t / tot:6.3f} {b:9.2f} {b / t if t else 0:6.2f}")
    print(f"total {tot:.3f} ms")
    if "--levels" in sys.argv:
        # last factor sequence (one Newton step): consecutive factor launches
        runs, cur = [], []
        for e in seq:
            if short(e["name"]) in ("nr_factor_kernel", "nr_tail_kernel"):
                cur.append(e)
            elif cur:
                runs.append(cur)
                cur = []
        if cur:
            runs.append(cur)
        if runs:
            for e in runs[-1]:
                t = e.get("gpu__time_duration.sum", 0) / 1e6
                b = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e9
                print(f"  {short(e['name']):18s} grid {e['grid']:>16s} {t:8.3f} ms {b:7.2f} GB")


if __name__ == "__main__":
    main()
