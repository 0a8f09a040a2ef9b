"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = 1 if rows[0][0] == "Kernel Name" else 0
h = rows[k]
I = {n: i for i, n in enumerate(h)}
data = []
for r in rows[k + 1:]:
    try:
        data.append((float(r[I["Warp Stall Sampling (All Samples)"]]), r[I["Address"]][-5:], r[I["Source"]].strip(),
                     r[I["Instructions Executed"]]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for v, a, s, ex in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {a}  exec={ex:>7}  {s[:100]}")
