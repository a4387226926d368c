"""Instruction histogram per kernel of the built library (cuobjdump -sass): which memory / atomic / barrier / warp-level
mnemonics the sm_100a code actually contains.  usage: sass_histogram.py > profiles/rNN_sass_histogram.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = ROOT / "paper_2604_27486_b200" / "csrc" / "libculifter.so"
out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
kern, hist = None, {}
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        hist[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", line)
    if m and kern:
        hist[kern][m.group(1).split(".")[0]] += 1
print(f"# {lib.name}: SASS mnemonic histogram per kernel (sm_100a), top 24 each; total = static instruction count")
for k, h in hist.items():
    tot = sum(h.values())
    if tot < 200:
        continue
    print(f"\n{k}\n  total {tot} instructions ({tot * 16 / 1024:.0f} KB)")
    print("  " + ", ".join(f"{op} {n}" for op, n in h.most_common(24)))
    special = {op: n for op, n in h.items() if op in ("ATOMG", "ATOM", "RED", "ATOMS", "BAR", "SHFL", "VOTE", "MATCH", "LDL", "STL", "LDS", "STS", "LDG", "STG", "CCTL", "UTMALDG", "UBLKCP", "SYNCS", "WARPSYNC", "POPC")}
    print("  memory / sync: " + ", ".join(f"{op} {n}" for op, n in sorted(special.items())))
