"""The benchmark corpora, pinned to the Python reference.  A synthetic corpus
(paper_2604_27486_b200/synth.py) is a seeded multiset of the kernels of the pools
under tests/golden/; tools/make_pools.py stored, per pool kernel, the
LiftedFunction the reference's own front half produced (pool_<kind>_objs.pkl.xz)
and the sha1 of the state the reference's own passes left (pool_<kind>_expect.npz:
dump, diagnostics, boundaries, tags, id counters, value table).  Here:

* the encoded pool IS those kernels (encode(objects) == pool, bit for bit);
* every pool kernel through an engine, decoded back into its objects, gives the
  reference's digest -- the oracle on a strided sample on the CPU, the CUDA
  library on EVERY kernel on the GPU (both device paths)."""
import copy
import lzma
import pickle

import numpy as np
import pytest

import helpers
from paper_2604_27486_b200 import layout as L, soa, synth

KINDS = ("sm90", "sm75", "sm52", "long")


_OBJS = {}


def load_objects(kind):
    """The pool's kernels as objects (loaded once per kind; callers copy what they mutate)."""
    if kind not in _OBJS:
        with lzma.open(synth.POOL_DIR / f"pool_{kind}_objs.pkl.xz", "rb") as fh:
            _OBJS[kind] = pickle.load(fh)
    return _OBJS[kind]


def expected(kind):
    z = np.load(synth.POOL_DIR / f"pool_{kind}_expect.npz")
    return z["sha1"], z["error"]


def check_digests(engine, kind, picks):
    objs = load_objects(kind)
    sha1, error = expected(kind)
    fns = copy.deepcopy([objs[i] for i in picks])
    corpus = soa.encode(fns)
    engine.upload(corpus)
    engine.run_postssa()
    out = engine.download()
    soa.apply(out, fns, patterns=helpers.engine_patterns(engine))
    bad = []
    for i, fn, st in zip(picks, fns, out.func["status"]):
        if error[i]:
            if helpers.STATUS_ERROR.get(int(st)) != str(error[i]):
                bad.append((int(i), fn.name, f"status {int(st)}, reference raises {error[i]}"))
            continue
        if int(st) != L.ST_OK or helpers.state_digest(helpers.state_of(fn)) != sha1[i].tobytes():
            bad.append((int(i), fn.name, f"status {int(st)}, state differs from the reference's"))
    assert not bad, f"pool_{kind}: {len(bad)} of {len(picks)} kernels differ from the reference: {bad[:5]}"
    return len(picks)


@pytest.mark.parametrize("kind", KINDS)
def test_pool_is_the_reference_front_halfs_kernels(kind):
    objs = load_objects(kind)
    pool = synth.load_pool(kind)
    sha1, error = expected(kind)
    assert len(objs) == pool.corpus.n_funcs == len(sha1) == len(error)
    step = max(1, len(objs) // 500)              # encode is a per-object Python walk: a strided 500 kernels in the CPU suite
    picks = np.arange(0, len(objs), step)
    enc = soa.encode([objs[i] for i in picks])
    diffs = enc.equal(synth.take_functions(pool.corpus, picks))
    assert not diffs, diffs


@pytest.mark.parametrize("kind", KINDS)
def test_oracle_gives_the_references_digests(oracle_engine, kind):
    n = len(expected(kind)[0])
    picks = np.arange(0, n, 40) if kind != "long" else np.arange(0, n, 5)
    check_digests(oracle_engine, kind, picks)


@pytest.mark.parametrize("kind", ("sm90", "sm52"))
def test_device_code_gives_the_references_digests_sim(sim_fused_engine, sim_tile_engine, kind):
    n = len(expected(kind)[0])
    for eng in (sim_fused_engine, sim_tile_engine):
        check_digests(eng, kind, np.arange(3, n, 160))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_cuda_gives_the_references_digests_on_every_pool_kernel(cuda_tile_engine, cuda_fused_engine, kind):
    n = len(expected(kind)[0])
    assert check_digests(cuda_tile_engine, kind, np.arange(n)) == n
    check_digests(cuda_fused_engine, kind, np.arange(0, n, 2))
