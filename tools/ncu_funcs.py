"""Like ncu_lines.py, but aggregated per tile.cuh function / file: share of executed
warp instructions and of stall samples, plus the stall-reason mix of the kernel.
usage: ncu_funcs.py src.csv dis.txt kernel_mangled_name"""
import csv, re, sys
from collections import defaultdict
src, dis, kern = sys.argv[1:4]
rows = list(csv.reader(open(src)))
hdr = rows[1]
ia, ii, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples")
data = rows[2:]
base = int(data[0][ia], 16)
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
cur = ("?", 0); off2line = {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith(".section"): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m: off2line[int(m.group(1), 16)] = cur
root = "/root/repo/paper_2604_27486_b200/csrc/"
srcs = {f: open(root + f).read().split("\n") for f in ("tile.cuh", "core.cuh", "stream.cuh")}
def func_of(f, l):
    if f not in srcs: return f
    for k in range(min(l, len(srcs[f])) - 1, -1, -1):
        m = re.match(r'(?:template <.*> )?CL[DFNM] [\w ]*?\b(\w+)\(', srcs[f][k])
        if m: return f.split(".")[0] + ":" + m.group(1)
    return f
agg = defaultdict(lambda: [0, 0]); tot = [0, 0]
for r in data:
    f, l = off2line.get(int(r[ia], 16) - base, ("?", 0))
    key = func_of(f, l)
    v = (int(r[ii] or 0), int(r[isamp] or 0))
    for k in range(2): agg[key][k] += v[k]; tot[k] += v[k]
print(f"warp-inst {tot[0]:,}  samples {tot[1]:,}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:34]:
    print(f"{v[1] / tot[1]:6.1%} samp {v[0] / tot[0]:6.1%} inst  {k}")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
st = defaultdict(int)
for r in data:
    for i in cols:
        try: st[hdr[i]] += int(r[i] or 0)
        except ValueError: pass
s = sum(st.values())
print({k: round(v / s, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v / s > 0.01})
