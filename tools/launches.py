"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
mean and total device time (cold-cache, serialised — compare shares, not absolutes)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
                out.append((d["Kernel Name"].split("(")[0], v * scale.get(d["Metric Unit"], 1.0)))
    return out


def summary(path):
    agg = OrderedDict()
    for k, us in load(path):
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in agg.items():
        print(f"{k[:70]:70s} n={c:4d} mean={t / c:9.1f} us total={t:10.1f} us {100 * t / tot:5.1f}%")
    print(f"{'total':70s} {tot:.1f} us")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        summary(p)
