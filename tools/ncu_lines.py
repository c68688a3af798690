"""Attribute an ncu source-page CSV (SASS, --print-source sass) of the core kernel to source
lines: instructions executed and stall samples per msd_core.cu line, using `nvdisasm -g` of the
same cubin.  usage: ncu_lines.py <src.csv> <nvdisasm.sass> <function-substring> [top]"""
import csv, re, sys, collections
src, sass, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# offset -> line from nvdisasm -g
off2line, cur, infn, line = {}, None, False, None
for ln in open(sass):
    if ln.startswith(".text."):
        infn = fn in ln
        continue
    if not infn:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m and '//##' in ln:
        line = m.group(1).split("/")[-1] + ":" + m.group(2); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and line is not None:
        off2line[int(m.group(1), 16)] = line
rows = list(csv.reader(open(src)))
hi = 0 if "Address" in rows[0] else 1
h = rows[hi]; data = rows[hi + 1:]
iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][iA], 16)
ex, st = collections.Counter(), collections.Counter()
for r in data:
    off = int(r[iA], 16) - base
    l = off2line.get(off, "?")
    ex[l] += int(r[iE] or 0); st[l] += int(r[iS] or 0)
T, TS = sum(ex.values()), sum(st.values())
print(f"{T} warp instructions, {TS} stall samples, {len(off2line)} mapped offsets")
for l, v in sorted(ex.items(), key=lambda x: -x[1])[:top]:
    print(f"{l:22s}: exec {v:10d} ({100*v/T:5.1f}%)  samples {st[l]:6d} ({100*st[l]/TS:5.1f}%)")
