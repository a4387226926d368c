"""The function-resident path (csrc/fused.cuh: one function resident in shared
memory per warp group, all passes fused) against the oracle on corpora drawn
from the reference-front-half pools.  It is the production path of every run that
asks for match lists (emit_matches, MATCH_ONLY) and can take any post-SSA run
(CL_FUSED=1); what it cannot do exactly it hands back to the general
per-function kernel, so the result must be bit-equal either way -- and the
hand-back rate must stay small."""
import numpy as np
import pytest

import helpers
from paper_2604_27486_b200 import synth


def _run(engine, corpus, passes=15, **kw):
    engine.upload(corpus)
    engine.run_postssa(passes, **kw)
    out = engine.download()
    out.stats = engine.stats().copy()
    return out


def _check(engine, oracle, kind, n_sass, seed, passes=15, max_back=0.02, **kw):
    corpus = synth.build_corpus(kind, n_sass, seed=seed)[0]
    got = _run(engine, corpus, passes, **kw)
    part = engine.debug_partition()
    want = _run(oracle, corpus, passes, **kw)
    assert not helpers.corpora_equal(got, want)
    assert part["tile_mode"] == 16, part                     # the fused path took the run
    if kind != "long":
        assert part["handed_back"] <= max_back * corpus.n_funcs + 2, part
    return part


@pytest.mark.parametrize("kind,n_sass", [("sm52", 60_000), ("sm75", 60_000), ("sm90", 60_000), ("mixed", 120_000)])
def test_fused_logic_sim(sim_fused_engine, oracle_engine, kind, n_sass):
    """one-lane CPU build of the fused code (logic only)"""
    _check(sim_fused_engine, oracle_engine, kind, n_sass, seed=11)


@pytest.mark.parametrize("passes", [1, 2, 4, 8, 6, 7, 5])
def test_fused_pass_subsets_sim(sim_fused_engine, oracle_engine, passes):
    _check(sim_fused_engine, oracle_engine, "mixed", 40_000, seed=3, passes=passes)


def test_fused_match_events_sim(sim_fused_engine, oracle_engine):
    """emit_matches: the raw and the selected match lists of every round, as events, equal the oracle's"""
    _check(sim_fused_engine, oracle_engine, "mixed", 40_000, seed=5, emit_matches=1)
    _check(sim_fused_engine, oracle_engine, "sm52", 30_000, seed=6, emit_matches=1)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n_sass,seed", [("sm52", 400_000, 1), ("sm75", 400_000, 2), ("sm90", 400_000, 3),
                                              ("mixed", 1_500_000, 4), ("mixed", 300_000, 5)])
def test_fused_cuda_bit_equal_to_oracle(cuda_fused_engine, oracle_engine, kind, n_sass, seed):
    _check(cuda_fused_engine, oracle_engine, kind, n_sass, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("passes", [1, 2, 4, 8, 6, 7, 5])
def test_fused_cuda_pass_subsets(cuda_fused_engine, oracle_engine, passes):
    _check(cuda_fused_engine, oracle_engine, "mixed", 200_000, seed=6, passes=passes)


@pytest.mark.gpu
def test_fused_cuda_match_events(cuda_fused_engine, oracle_engine):
    """the production kernels emit the match sets themselves: raw + selected lists of every round, bit-equal"""
    _check(cuda_fused_engine, oracle_engine, "mixed", 300_000, seed=7, emit_matches=1)
    _check(cuda_fused_engine, oracle_engine, "sm52", 200_000, seed=8, emit_matches=1)


@pytest.mark.gpu
def test_fused_cuda_repeatable(cuda_fused_engine):
    """the same upload run three times gives the same bytes (no order-dependent races)"""
    corpus = synth.build_corpus("mixed", 500_000, seed=9)[0]
    cuda_fused_engine.upload(corpus)
    outs = []
    for _ in range(3):
        cuda_fused_engine.run_postssa()
        o = cuda_fused_engine.download()
        o.stats = cuda_fused_engine.stats().copy()
        outs.append(o)
    assert not helpers.corpora_equal(outs[0], outs[1])
    assert not helpers.corpora_equal(outs[0], outs[2])
