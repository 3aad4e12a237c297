"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
                continue
            t = float(d["Metric Value"])
            t *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
            d["us"] = t
            d["short"] = d["Kernel Name"].split("(")[0].replace("htg::", "").replace("<unnamed>::", "")
            data.append(d)
    return data


if __name__ == "__main__":
    data = load(sys.argv[1])
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    part = data[int(len(data) * (1 - frac)):]
    agg = collections.OrderedDict()
    for d in part:
        a = agg.setdefault(d["short"], [0, 0.0])
        a[0] += 1
        a[1] += d["us"]
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} n={v[0]:5d} total={v[1]:10.1f} us share={v[1] / tot * 100:5.1f}%")
    print(f"total {tot:.1f} us over {len(part)} launches")
