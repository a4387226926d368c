"""Fresh long-block kernels (reference front half, seeds outside the pools) through the tile path of the one-lane
CPU build of the device code, compared bit for bit with the oracle: exercises the reciprocal-chain decisions
(independent chains, chains decided in order, adds without an F2I in reach) on blocks of 4096 / 8192 instructions.
Runs in the build container only (imports the reference).  usage: stress_long_tiles.py [first_seed] [n_seeds]"""
import sys
import time
from multiprocessing import Pool as MPool
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests")); sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402

import make_pools  # noqa: E402


def gen(seed):
    make_pools.R.load()
    fns, n_sass, _, errors = make_pools.work(("long", seed, 2, seed % 2))      # sizes alternate 4096 / 8192 (/ 16384)
    return fns, errors


def main():
    import helpers
    from paper_2604_27486_b200 import soa
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    t0 = time.time()
    with MPool(8) as mp:
        res = mp.map(gen, range(first, first + n), chunksize=1)
    fns = [f for r in res for f, e in zip(r[0], r[1]) if not e]
    print(f"{len(fns)} kernels generated in {time.time() - t0:.0f}s", flush=True)
    c = soa.encode(fns)
    eng = helpers._engine_with_env(helpers.build_sim(), CL_TILE=4, CL_GTILE_CFG=2)
    eng.upload(c); eng.run_postssa(); out = eng.download()
    part = eng.debug_partition()
    o = helpers.oracle_engine(); o.set_threads(8); o.upload(c); o.run_postssa(); ref = o.download()
    diffs = out.equal(ref)
    ev = np.array_equal(out.events, ref.events)
    print("partition", part, "records", c.n_insts, "diffs", diffs, "events equal", ev)
    sys.exit(1 if diffs or not ev else 0)


if __name__ == "__main__":
    main()
