"""Build the kernel pools behind paper_2604_27486_b200/synth.py (in-container
only: the SASS text goes through the reference's own front half).

    python tools/make_pools.py            # writes tests/golden/pool_<kind>.npz
"""
import sys, time
from multiprocessing import Pool as MPool
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import random
import refharness as R
import gen_sass
from paper_2604_27486_b200 import ir, soa, synth

SPEC = {  # kind: (functions, chunk) -- sized so each pool is a few hundred k records at most
    "sm90": 3000, "sm75": 2000, "sm52": 3000, "long": 12,
}


def gen_text(kind, seed, n):
    rng = random.Random(seed)
    out = []
    for i in range(n):
        name = f"{kind}_{seed}_{i}"
        if kind == "sm52":
            out.append(gen_sass.gen_function(rng, name, "sm52", gen_sass.MIX_SM52, rng.choice([1, 1, 2]), (8, 56), 0.1))
        elif kind == "sm90":
            out.append(gen_sass.gen_function(rng, name, "sm90", gen_sass.MIX_SM90, rng.choice([1, 1, 2]), (8, 100), 0.1))
        elif kind == "sm75":
            out.append(gen_sass.gen_function(rng, name, "sm75", gen_sass.MIX_SM90, rng.choice([1, 2, 3]), (8, 40), 0.1))
        else:
            size = (4096, 8192, 16384)[i % 3]
            out.append(gen_sass.gen_function(rng, name, "sm90", gen_sass.MIX_LONG, 1, (size, size), 0.1, window=16))
    return out


def work(args):
    kind, seed, n = args
    arch = {"sm52": "sm52", "sm90": "sm90", "sm75": "sm75", "long": "sm90"}[kind]
    texts = gen_text(kind, seed, n)
    fns, n_sass = [], []
    for t in texts:
        got = R.ssa_functions(t, arch)
        assert len(got) == 1
        fns.append(ir.convert(got[0]))
        n_sass.append(sum(1 for ln in t.splitlines() if ln and not ln.startswith(".text")))
    return fns, n_sass


def main():
    for kind, total in SPEC.items():
        t0 = time.time()
        chunk = 1 if kind == "long" else 100
        jobs = [(kind, 1000 + k, min(chunk, total - k * chunk)) for k in range((total + chunk - 1) // chunk)]
        with MPool(8) as mp:
            res = mp.map(work, jobs)
        fns = [f for r in res for f in r[0]]
        n_sass = [n for r in res for n in r[1]]
        corpus = soa.encode(fns)
        path = synth.POOL_DIR / f"pool_{kind}.npz"
        synth.save_pool(path, corpus, n_sass, kind)
        print(f"{path.name}: {len(fns)} kernels, {sum(n_sass)} SASS insts, {corpus.n_insts} records, "
              f"{path.stat().st_size / 1e6:.2f} MB, {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
