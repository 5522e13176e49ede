"""Per-launch table from an ncu --csv metrics log: python tools/launch_table.py file.csv [first] [last]."""
import collections
import csv
import sys


def load(path):
    hdr, L = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = L.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0], "grid": d.get("Grid Size", "")})
            v = d["Metric Value"].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
                    d["Metric Unit"], 1.0)
            e[d["Metric Name"]] = v
    return list(L.values())


if __name__ == "__main__":
    items = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for x in items:
        t = x.get("gpu__time_duration.sum", 0.0)
        a = agg[x["name"]]
        a[0] += 1
        a[1] += t
        a[2] += t * float(x.get("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 0.0) or 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(items)} launches, {tot / 1e3:.2f} ms")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / 1e3:10.2f} ms {100 * v[1] / tot:5.1f}% n={v[0]:6d} fp64pipe(time-wtd)={v[2] / max(v[1], 1e-9):5.1f}%  {k[:60]}")
