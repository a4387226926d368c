"""Development probe: device time, partition and per-phase cycles of one corpus
for a few pass subsets (run under gpurun)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2604_27486_b200 import synth
from paper_2604_27486_b200.capi import Engine

kind = sys.argv[1] if len(sys.argv) > 1 else "mixed"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 4_000_000
subsets = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [15]
corpus, ns = synth.build_corpus(kind, n, seed=100)[:2]
n_sass = int(np.sum(ns))
eng = Engine()
eng.upload(corpus)
for passes in subsets:
    for _ in range(2):
        eng.run_postssa(passes)
    ms = []
    for _ in range(3):
        eng.run_postssa(passes)
        ms.append(eng.last_run_ms())
    prof = eng.debug_profile()
    part = eng.debug_partition()
    tot = max(prof.get("total", 1), 1)
    tiles = max(part["tiles"], 1)
    print(f"passes={passes} ms={min(ms):.2f} Minst/s={n_sass / min(ms) / 1e3:.1f} records={corpus.n_insts} part={part}")
    print("   cycles/tile:", {k: int(v / tiles) for k, v in prof.items() if v})
