"""Chunked streaming (capi.Pipeline, Corpus.split / slice_funcs): a corpus cut
into contiguous function ranges and pushed through several contexts gives,
chunk by chunk, exactly the result of one big run (functions are independent,
ssir.py:215-235)."""
import copy

import numpy as np
import pytest

import helpers
from paper_2604_27486_b200 import soa, synth
from paper_2604_27486_b200.capi import Pipeline


def _corpus():
    fns = []
    for name in ("synth_sm90", "synth_sm75", "synth_sm52", "synth_long"):
        fns += copy.deepcopy(helpers.load_fixture(name)["functions"])
    return soa.encode(fns)


def _check(lib_path, one_shot_engine, n_chunks, depth):
    corpus = _corpus()
    ranges = corpus.split(n_chunks)
    assert ranges[0][0] == 0 and ranges[-1][1] == corpus.n_funcs
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    chunks = [corpus.slice_funcs(a, b) for a, b in ranges]
    assert sum(c.n_insts for c in chunks) == corpus.n_insts
    pipe = Pipeline(depth=depth, lib_path=lib_path)
    outs, stats, _ = pipe.run_postssa(chunks)
    # the same again into caller-owned holders that are larger than needed
    holders = []
    for o in outs:
        h = soa.Corpus(**{a: np.zeros((len(getattr(o, a)) + 7,) + getattr(o, a).shape[1:], getattr(o, a).dtype)
                          for a in soa.Corpus.ARRAYS})
        h.events = np.zeros(len(o.events) + 3, o.events.dtype)
        holders.append(h)
    outs2, stats2, _ = pipe.run_postssa(chunks, into=holders)
    pipe.close()
    one_shot_engine.upload(corpus)
    one_shot_engine.run_postssa()
    whole = one_shot_engine.download()
    whole_stats = one_shot_engine.stats()
    for got in (outs, outs2):
        for (f0, f1), o in zip(ranges, got):
            want = whole.slice_funcs(f0, f1)
            assert not o.equal(want), (f0, f1, o.equal(want))
    # events are per function and in function order: the chunks' lists concatenate to the whole list
    ev = np.concatenate([o.events for o in outs])
    f_base = np.concatenate([np.full(len(o.events), r[0], np.uint32) for r, o in zip(ranges, outs)])
    ev = ev.copy()
    ev["func"] += f_base
    assert np.array_equal(ev, whole.events)
    for name in ("matches", "selected", "rewrites", "refused", "n_inst_in", "n_inst_out"):
        assert np.array_equal(stats[name], whole_stats[name]), name
        assert np.array_equal(stats2[name], whole_stats[name]), name


def test_split_covers_every_function():
    corpus = _corpus()
    for k in (1, 2, 5, 64, 10_000):
        ranges = corpus.split(k)
        assert ranges[0][0] == 0 and ranges[-1][1] == corpus.n_funcs
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(ranges, ranges[1:] + [(corpus.n_funcs, 0)]))


def test_pipeline_oracle_engine(oracle_engine):
    """Host logic of the pipeline (threads, holders, stats) with the checker library as the engine."""
    _check(helpers.build_oracle(), oracle_engine, n_chunks=5, depth=3)


@pytest.mark.gpu
def test_pipeline_cuda(cuda_engine):
    _check(None, cuda_engine, n_chunks=6, depth=3)


@pytest.mark.gpu
def test_pipeline_cuda_matches_oracle(oracle_engine):
    corpus = _corpus()
    chunks = [corpus.slice_funcs(a, b) for a, b in corpus.split(4)]
    pipe = Pipeline(depth=2)
    outs, _, _ = pipe.run_postssa(chunks)
    pipe.close()
    for c, o in zip(chunks, outs):
        oracle_engine.upload(c)
        oracle_engine.run_postssa()
        want = oracle_engine.download()
        assert not o.equal(want)
        assert np.array_equal(o.events, want.events)
