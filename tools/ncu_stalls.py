"""Summarise per-instruction stall samples of an ncu source-page CSV (--page source --csv
--print-source sass): stall reasons summed over the instructions executed at least
`min_exec` times (the hot loop), plus the top instructions."""
import csv, collections, sys
path = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 62
rows = list(csv.reader(open(path)))
h = rows[1]; data = rows[2:]
iE = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
n = 0
for r in data:
    e = int(r[iE] or 0)
    if lo <= e <= hi:
        n += 1
        for c in cols:
            tot[c] += int(r[h.index(c)] or 0)
s = sum(tot.values())
print(f"{n} instructions in [{lo}, {hi}] executions; {s} samples")
for c, v in tot.most_common():
    if v: print(f"  {c:28s} {v:7d} {100 * v / max(s, 1):5.1f}%")
