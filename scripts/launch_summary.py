"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per launch) by kernel."""
import csv
import sys
from collections import OrderedDict, defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    k = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(k.values())


def summary(path, key=lambda n: n.split("(")[0]):
    L = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for d in L:
        a = agg[key(d["name"])]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tot += d.get("gpu__time_duration.sum", 0.0)
    print(f"{path}: {len(L)} launches, {tot / 1e6:.3f} ms summed")
    for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {n[:60]:60s} {c:5d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  {b / max(t, 1):7.1f} GB/s")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p)
