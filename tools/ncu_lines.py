"""Join an `ncu --page source --csv` SASS dump with `nvdisasm --print-line-info`
to get executed instructions / stall samples per CUDA source line (ncu's own
CUDA view exports only the .cu file, not the headers).
usage: ncu_lines.py src.csv dis.txt kernel_mangled_name [top]"""
import csv, re, sys
from collections import defaultdict
src, dis, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(src)))
hdr = rows[1]
ia, ii, isamp, ith = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples"), hdr.index("Thread Instructions Executed")
data = rows[2:]
base = int(data[0][ia], 16)
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
cur = ("?", 0)
off2line = {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0, 0, 0])
tot = [0, 0, 0]
miss = 0
for r in data:
    off = int(r[ia], 16) - base
    key = off2line.get(off)
    if key is None:
        miss += 1
        key = ("?", 0)
    v = (int(r[ii] or 0), int(r[isamp] or 0), int(r[ith] or 0))
    for k in range(3):
        agg[key][k] += v[k]; tot[k] += v[k]
print(f"total warp-inst {tot[0]:,} samples {tot[1]:,} thread-inst {tot[2]:,} unmapped rows {miss}")
byfile = defaultdict(lambda: [0, 0])
for (f, l), v in agg.items():
    byfile[f][0] += v[0]; byfile[f][1] += v[1]
print({f: (f"{v[0] / tot[0]:.1%}", f"{v[1] / tot[1]:.1%}") for f, v in byfile.items()})
srcs = {}
for (f, l), v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    if f not in srcs:
        try:
            srcs[f] = open(f"/root/repo/paper_2604_27486_b200/csrc/{f}").read().split("\n")
        except OSError:
            srcs[f] = []
    text = srcs[f][l - 1].strip()[:110] if 0 < l <= len(srcs[f]) else ""
    print(f"{v[1] / tot[1]:6.1%} samp {v[0] / tot[0]:6.1%} inst  {f}:{l:<5} {text}")
