"""Build the kernel pools behind paper_2604_27486_b200/synth.py (in-container
only: the SASS text goes through the reference's own front half, and the
expected results come from the reference's own passes).

    python tools/make_pools.py            # writes tests/golden/pool_<kind>*.{npz,pkl.xz}

Per kind three files:
  pool_<kind>.npz          the kernels as an encoded corpus (what build_corpus draws from)
  pool_<kind>_objs.pkl.xz  the same kernels as LiftedFunction objects (SSA phase, the
                           reference front half's output), so a test can check that the
                           encoded pool IS those kernels and decode results into them
  pool_<kind>_expect.npz   per kernel: sha1 of the reference's state after its own passes
                           (pipeline.py:165-169; dump, diagnostics, boundaries, tags, id
                           counters, value table) or the name of the exception it raises
Every byte the benchmark corpora hold is therefore pinned to the Python reference:
a corpus is a seeded multiset of these kernels.
"""
import hashlib, lzma, pickle, sys, time
from multiprocessing import Pool as MPool
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import random
import numpy as np
import refharness as R
import gen_sass
from paper_2604_27486_b200 import ir, soa, synth

SPEC = {  # kind: kernels
    "sm90": 6000, "sm75": 5000, "sm52": 5000, "long": 24,
}
LONG_SIZES = [4096] * 12 + [8192] * 8 + [16384] * 4     # BASELINE.json configs[3]: 4096+ instructions per block


def gen_text(kind, seed, n, first=0):
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
            size = LONG_SIZES[(first + i) % len(LONG_SIZES)]
            out.append(gen_sass.gen_function(rng, name, "sm90", gen_sass.MIX_LONG, 1, (size, size), 0.1, window=16))
    return out


def state_digest(state) -> bytes:
    """sha1 of the canonical JSON of a state_of() dict (tests/helpers.py computes the same for device results)"""
    import json
    return hashlib.sha1(json.dumps(state, sort_keys=True, default=str).encode()).digest()


def work(args):
    kind, seed, n, first = args
    arch = {"sm52": "sm52", "sm90": "sm90", "sm75": "sm75", "long": "sm90"}[kind]
    texts = gen_text(kind, seed, n, first)
    fns, n_sass, digests, errors = [], [], [], []
    for t in texts:
        got = R.ssa_functions(t, arch)
        assert len(got) == 1
        fns.append(ir.convert(got[0]))
        n_sass.append(sum(1 for ln in t.splitlines() if ln and not ln.startswith(".text")))
        ref = R.clone(got[0])
        err = R.run_postssa(ref)
        errors.append("" if err is None else type(err).__name__)
        digests.append(bytes(20) if err is not None else state_digest(R.state_of(ref)))
    return fns, n_sass, digests, errors


def raw_work(args):
    """Raw-stage pools (BASELINE.json configs[1]: OpModTransform + SRSubstituteReverse on sm52): the sm52 pool's
    listings as PARSED functions (input of normalize_instruction, frontend.py:523) and after the reference's own
    normalize + register widening (input of substitute_special_registers, frontend.py:697)."""
    seed, n = args
    R.load()
    from sasslift import frontend
    x4_in, sr_in, n_sass = [], [], []
    for t in gen_text("sm52", seed, n):
        for fn in R.raw_functions(t, "sm52", normalize=False):
            x4_in.append(ir.convert(fn))
            out = []
            for inst in fn.raw_instructions:
                out.extend(frontend.normalize_instruction(fn, inst))
            fn.raw_instructions = out
            for inst in fn.raw_instructions:
                frontend.expand_implicit_registers(inst, "sm52")
            sr_in.append(ir.convert(fn))
            n_sass.append(sum(1 for ln in t.splitlines() if ln and not ln.startswith(".text")))
    return x4_in, sr_in, n_sass


def main_raw():
    t0 = time.time()
    total, chunk = SPEC["sm52"], 100
    with MPool(8) as mp:
        res = mp.map(raw_work, [(1000 + k, min(chunk, total - k * chunk)) for k in range((total + chunk - 1) // chunk)], chunksize=1)
    n_sass = [n for r in res for n in r[2]]
    for name, idx in (("raw_x4", 0), ("raw_sr", 1)):
        fns = [f for r in res for f in r[idx]]
        corpus = soa.encode(fns, raw=True)
        path = synth.POOL_DIR / f"pool_{name}.npz"
        synth.save_pool(path, corpus, n_sass, name)
        print(f"{path.name}: {len(fns)} kernels, {sum(n_sass)} SASS insts, {corpus.n_insts} records, {path.stat().st_size / 1e6:.2f} MB, {time.time() - t0:.0f}s", flush=True)


def main():
    kinds = sys.argv[1:] or list(SPEC) + ["raw"]
    if "raw" in kinds:
        main_raw()
        kinds = [k for k in kinds if k != "raw"]
    for kind in kinds:
        total = SPEC[kind]
        t0 = time.time()
        chunk = 1 if kind == "long" else 100
        jobs = [(kind, 1000 + k, min(chunk, total - k * chunk), k * chunk) for k in range((total + chunk - 1) // chunk)]
        if kind == "long":
            jobs.sort(key=lambda j: -LONG_SIZES[j[3] % len(LONG_SIZES)])       # the 16384-instruction blocks take minutes: start them first
        with MPool(8) as mp:
            res = mp.map(work, jobs, chunksize=1)
        if kind == "long":
            res = [r for _, r in sorted(zip(jobs, res), key=lambda jr: jr[0][3])]
        fns = [f for r in res for f in r[0]]
        n_sass = [n for r in res for n in r[1]]
        digests = np.frombuffer(b"".join(d for r in res for d in r[2]), np.uint8).reshape(-1, 20)
        errors = np.array([e for r in res for e in r[3]])
        corpus = soa.encode(fns)
        path = synth.POOL_DIR / f"pool_{kind}.npz"
        synth.save_pool(path, corpus, n_sass, kind)
        (synth.POOL_DIR / f"pool_{kind}_objs.pkl.xz").write_bytes(lzma.compress(pickle.dumps(fns, protocol=4), preset=6))
        np.savez_compressed(synth.POOL_DIR / f"pool_{kind}_expect.npz", sha1=digests, error=errors)
        print(f"{path.name}: {len(fns)} kernels, {sum(n_sass)} SASS insts, {corpus.n_insts} records, "
              f"{path.stat().st_size / 1e6:.2f} MB (+ objects {(synth.POOL_DIR / f'pool_{kind}_objs.pkl.xz').stat().st_size / 1e6:.2f} MB), "
              f"{int((errors != '').sum())} reference errors, {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
