"""Per-instruction stall attribution from an ncu SASS source page:
    ncu -i REP -k regex:K --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv [top]
Prints stall samples grouped by opcode and the top individual instructions."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
by_op = collections.defaultdict(lambda: collections.Counter())
items = []
tot = 0
for r in rows[2:]:
    if len(r) != len(h):
        continue
    src = r[isrc].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    if not r[iall].isdigit():
        continue
    n = int(r[iall])
    tot += n
    c = collections.Counter({k[6:]: int(r[h.index(k)] or 0) for k in cols})
    by_op[op.split(".")[0]] += c
    by_op[op.split(".")[0]]["_n"] += n
    items.append((n, r[ia][-5:], src[:60], c.most_common(3)))
print(f"total samples {tot}")
for op, c in sorted(by_op.items(), key=lambda x: -x[1]["_n"])[:20]:
    n = c.pop("_n")
    print(f"{op:14s} {100 * n / tot:5.1f}%  " + ", ".join(f"{k} {100 * v / tot:.1f}" for k, v in c.most_common(4)))
print("-- top instructions")
for n, a, s, c in sorted(items, reverse=True)[:top]:
    print(f"{100 * n / tot:5.1f}% {a} {s:60s} {c}")
