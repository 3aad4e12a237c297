"""Aggregate ncu SASS source-page stall samples by opcode and list the hottest instructions."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i0]
data = [r for r in rows[i0 + 1:] if len(r) == len(hdr)]
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
by = collections.Counter()
ex = collections.Counter()
tot = 0
for r in data:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    s = int(r[S] or 0)
    by[op] += s
    ex[op] += int(r[E] or 0)
    tot += s
print("total samples", tot)
for op, s in by.most_common(25):
    print(f"{op:12s} {s:8d} {s / tot:6.1%}  exec {ex[op]}")
top = sorted(data, key=lambda r: -int(r[S] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for r in top:
    print(r[S], r[0][-5:], r[1][:90])
