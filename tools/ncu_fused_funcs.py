"""Per device function of a fused kernel: share of executed warp instructions, of stall samples, lanes active.
usage: ncu_fused_funcs.py source_page.csv fused.o <class tag, e.g. FCfgSELi1>"""
import csv, re, subprocess, sys
from collections import defaultdict
src, obj, tag = sys.argv[1:4]
elf = subprocess.run(["cuobjdump", "-elf", obj], capture_output=True, text=True).stdout
sym = []
insec = False
for l in elf.splitlines():
    if l.startswith(".section .symtab"): insec = True; continue
    if insec and l.startswith(".section"): break
    if insec and tag in l:
        t = l.split()
        try:
            val, size = int(t[1], 16), int(t[2], 16)
        except (ValueError, IndexError):
            continue
        name = t[-1]
        m = re.search(r"\$_ZN9clk_fused(\d+)(\w+)", name)
        if m: sym.append((val, size, m.group(2)[:int(m.group(1))]))
sym.sort()
rows = list(csv.reader(open(src)))
hdr = rows[1]
ia, ii, it, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("# Samples")
data = rows[2:]
base = int(data[0][ia], 16)
def fn(off):
    for v, s, n in sym:
        if v <= off < v + s: return n
    return "k_fused(body)"
agg = defaultdict(lambda: [0, 0, 0]); tot = [0, 0, 0]
for r in data:
    k = fn(int(r[ia], 16) - base)
    v = (int(r[ii] or 0), int(r[isamp] or 0), int(r[it] or 0))
    for q in range(3): agg[k][q] += v[q]; tot[q] += v[q]
print(f"warp-inst {tot[0]:,}  samples {tot[1]:,}  lanes/inst {tot[2] / max(tot[0], 1):.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{v[0] / tot[0]:6.1%} inst {v[1] / tot[1]:6.1%} samp  {v[2] / max(v[0], 1):5.1f} lanes  {k}")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
st = defaultdict(int)
for r in data:
    for i in cols:
        try: st[hdr[i]] += int(r[i] or 0)
        except ValueError: pass
s = sum(st.values()) or 1
print({k: round(v / s, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v / s > 0.01})
