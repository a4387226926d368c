"""Edge cases of the batch paths (empty and ragged inputs, capacity
limits) and size-independent properties at benchmark-like sizes.  Every engine
must agree with the oracle bit for bit; the CPU runs use the one-lane build of
the device code (tests/sim), the GPU runs the product library."""
import numpy as np
import pytest

import helpers
from paper_2604_27486_b200 import layout as L
from paper_2604_27486_b200 import soa, synth


def _run(engine, corpus, passes=15):
    engine.upload(corpus)
    engine.run_postssa(passes)
    out = engine.download()
    out.stats = engine.stats().copy()
    return out


def _empty_like(c: soa.Corpus) -> soa.Corpus:
    """zero functions, zero blocks, zero records"""
    z = {a: getattr(c, a)[:0] for a in soa.Corpus.ARRAYS}
    for a in ("func_blk_off", "ext_off", "mem_off", "imm_off", "val_off", "blk_off"):
        z[a] = np.zeros(1, np.uint32)
    return soa.Corpus(**z)


def _with_ragged_functions(c: soa.Corpus) -> soa.Corpus:
    """the corpus plus, in the middle and at both ends, functions that own one block with no record at all"""
    one = c.slice_funcs(0, 1)
    hollow = soa.Corpus(
        func=one.func.copy(), func_blk_off=np.array([0, 1], np.uint32), ext_off=np.zeros(2, np.uint32),
        mem_off=np.zeros(2, np.uint32), imm_off=np.zeros(2, np.uint32), val_off=np.zeros(2, np.uint32),
        blk=one.blk[:1].copy(), blk_off=np.zeros(2, np.uint32), hdr=one.hdr[:0], tag=one.tag[:0], pay=one.pay[:0],
        ext_tag=one.ext_tag[:0], ext_pay=one.ext_pay[:0], mem=one.mem[:0], imm=one.imm[:0],
        val_alive=one.val_alive[:0], val_def_iid=one.val_def_iid[:0], val_origin=one.val_origin[:0])
    hollow.func["next_vid"] = 0
    hollow.blk["term_tag"] = 0
    hollow.blk["term_pay"] = 0
    half = c.n_funcs // 2
    return synth.concat([hollow, c.slice_funcs(0, half), hollow, hollow, c.slice_funcs(half, c.n_funcs), hollow])


def _engines(request, names):
    return [request.getfixturevalue(n) for n in names]


CPU_ENGINES = ["sim_fused_engine", "sim_tile_engine"]
GPU_ENGINES = ["cuda_fused_engine", "cuda_tile_engine"]


def _check_empty(engine):
    corpus = _empty_like(synth.build_corpus("sm75", 2_000, seed=1)[0])
    out = _run(engine, corpus)
    assert out.n_funcs == 0 and out.n_insts == 0 and len(out.events) == 0
    assert int(out.stats["selected"].sum()) == 0


def _check_ragged(engine, oracle):
    corpus = _with_ragged_functions(synth.build_corpus("mixed", 30_000, seed=21)[0])
    got, want = _run(engine, corpus), _run(oracle, corpus)
    assert not helpers.corpora_equal(got, want)
    assert int(got.func["status"].max()) == L.ST_OK


@pytest.mark.parametrize("name", CPU_ENGINES)
def test_empty_corpus_sim(request, name):
    _check_empty(request.getfixturevalue(name))


def test_empty_corpus_oracle(oracle_engine):
    _check_empty(oracle_engine)


@pytest.mark.parametrize("name", CPU_ENGINES)
def test_ragged_functions_sim(request, oracle_engine, name):
    _check_ragged(request.getfixturevalue(name), oracle_engine)


def test_rerun_on_own_output_sim(sim_fused_engine, sim_tile_engine, oracle_engine):
    """a result is a valid input: running the stage on its own output (the reference stops after four
    aggregation rounds, so a rerun may still rewrite) agrees with the oracle again, bit for bit"""
    corpus = synth.build_corpus("mixed", 40_000, seed=8)[0]
    want1 = _run(oracle_engine, corpus)
    want2 = _run(oracle_engine, want1)
    assert int(want2.stats["rewrites"].sum()) < int(want1.stats["rewrites"].sum()) // 20
    for eng in (sim_fused_engine, sim_tile_engine):
        once = _run(eng, corpus)
        assert not helpers.corpora_equal(once, want1)
        assert not helpers.corpora_equal(_run(eng, once), want2)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GPU_ENGINES)
def test_empty_corpus_cuda(request, name):
    _check_empty(request.getfixturevalue(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", GPU_ENGINES)
def test_ragged_functions_cuda(request, oracle_engine, name):
    _check_ragged(request.getfixturevalue(name), oracle_engine)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n_sass", [("mixed", 10_000_000), ("sm52", 10_000_000), ("sm90", 10_000_000), ("long", 4_000_000)])
def test_full_size_vs_oracle_cuda(cuda_fused_engine, cuda_tile_engine, oracle_engine, kind, n_sass):
    """BASELINE.json configs[1..4] at their quoted sizes, against the ORACLE itself (the C port runs at several
    M inst/s on the host cores, so 10 M instructions are seconds): both device paths give the oracle's bytes, the
    per-pattern counters add up, every function reports success, and a rerun on the result barely finds work"""
    corpus = synth.build_corpus(kind, n_sass, seed=100)[0]
    want = _run(oracle_engine, corpus)
    outs = []
    for eng in (cuda_tile_engine, cuda_fused_engine):
        once = _run(eng, corpus)
        st = once.stats
        assert int(st["n_inst_in"]) == corpus.n_insts and int(st["n_inst_out"]) == once.n_insts
        assert np.array_equal(st["selected"], st["rewrites"] + st["refused"])
        assert (st["matches"] >= st["selected"]).all()
        assert int(once.func["status"].max()) == L.ST_OK
        assert int((once.events["kind"] == L.EV_REFUSED).sum()) == int(st["refused"].sum())
        assert not helpers.corpora_equal(once, want)
        outs.append(once)
    twice = _run(cuda_tile_engine, outs[0])
    assert int(twice.stats["rewrites"].sum()) <= int(outs[0].stats["rewrites"].sum()) // 20
