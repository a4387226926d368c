"""Stress an engine (default: the C oracle) against the Python reference on
seeded synthetic listings.  In-container only (needs /root/reference)."""
import sys, time
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
import numpy as np
import refharness as R, gen_sass
from paper_2604_27486_b200.capi import Engine

def main(seeds, lib='oracle/liboracle.so', kinds=("sm90", "sm52", "sm75", "long")):
    eng = Engine(lib)
    tot = np.zeros(4 * 16, np.uint64)
    nd = 0
    for seed in seeds:
        for kind in kinds:
            n = {"sm90": 12, "sm52": 12, "sm75": 8, "long": 1}[kind]
            arch, text = gen_sass.gen_corpus(seed, kind, n, near_miss=0.15)
            fns = R.ssa_functions(text, arch)
            t = time.time()
            d = R.compare_postssa(fns, eng, label=f"{kind}/{seed}:")
            st = eng.stats()
            tot += np.concatenate([st["matches"], st["selected"], st["rewrites"], st["refused"]])
            nd += len(d)
            for x in d[:2]:
                print(x[:4000])
            print(kind, seed, "diffs", len(d), "events", int(st["n_events"]), f"{time.time()-t:.1f}s", flush=True)
    print("matches ", tot[:10]); print("selected", tot[16:26]); print("rewrites", tot[32:42]); print("refused ", tot[48:58])
    print("TOTAL DIFFS", nd)

if __name__ == "__main__":
    a, b = int(sys.argv[1]), int(sys.argv[2])
    main(range(a, b), *(sys.argv[3:4]))
