"""Per-CUDA-source-line stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = "?"
hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    key = (fname, r[0])
    src[key] = r[1][:70]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i]:
            try:
                agg[key][h[6:]] += int(r[i])
            except ValueError:
                pass
    try:
        agg[key]["_exec"] += int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        pass
tot = sum(sum(v for k, v in c.items() if k != "_exec") for c in agg.values())
print("total samples", tot)
items = sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_exec"))
for key, c in items[:top]:
    s = sum(v for k, v in c.items() if k != "_exec")
    if s == 0:
        break
    reasons = ", ".join(f"{k}={v}" for k, v in c.most_common(4) if k != "_exec")
    print(f"{s / tot:6.1%} {key[0]}:{key[1]:>4} exec={c['_exec']:>9}  {src[key]!r}  [{reasons}]")
