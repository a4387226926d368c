"""Type seeding: cl_seed_types against the TypeState the
reference's own typerec.seed_types (typerec.py:288) produced for the same functions
(tests/golden/types.pkl.gz, tools/make_types_golden.py).  Bit-exact: masks, roles and the
link expressions with the reference's dict and list orders."""
import copy
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import helpers
from paper_2604_27486_b200 import capi, soa, typerec

ROOT = Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "culifter_types.h").read_text()
DECLARED = sorted(set(re.findall(r"\b(cl_[a-z0-9_]+)\s*\(", HEADER)))


def check_against_golden(engine):
    fix = helpers.load_fixture("types")
    fns = copy.deepcopy(fix["functions"])
    states = typerec.seed_types_batch(fns, engine)
    assert len(states) == len(fix["expect"]) == 57
    for fn, st, exp in zip(fns, states, fix["expect"]):
        assert fn.meta["type_state"] is st
        for key in ("seed_mask", "def_seed_mask", "use_seed_mask", "roles", "link_exprs"):
            got = getattr(st, key)
            assert got == exp[key], (fn.name, key)
            if key == "link_exprs":
                assert list(got) == list(exp[key]), (fn.name, "link_exprs key order")
            else:
                assert sorted(got) == sorted(exp[key]), (fn.name, key)


def test_oracle_matches_reference_typestate():
    check_against_golden(helpers.oracle_engine())


def test_sim_matches_reference_typestate():
    """The device code of csrc/typeseed.cu compiled for the host (one thread): logic check without a GPU."""
    check_against_golden(helpers.sim_engine())


@pytest.mark.parametrize("which", ["product", "oracle"])
def test_library_exports_the_type_seeding_entry(which):
    path = capi.PRODUCT_LIB if which == "product" else helpers.build_oracle()
    lib = ctypes.CDLL(str(path))
    assert "cl_seed_types" in DECLARED
    assert all(hasattr(lib, n) for n in DECLARED)


def test_signature_table_lowering():
    """Per-id tables: precedence of the reference's if-chain (typerec.py:87-234)."""
    sk = typerec.SK
    assert typerec.sig_kind("FSEL") == (sk["FSEL"], 0) and typerec.sig_kind("MUFU") == (sk["FALU"], 0)
    assert typerec.sig_kind("ULOP3")[0] == sk["IALU"] and typerec.sig_kind("LOP3")[0] == sk["LOP"]
    assert typerec.sig_kind("LDG") == (sk["LOAD"], 1) and typerec.sig_kind("LDS") == (sk["LOAD"], 0)
    assert typerec.sig_kind("RED") == (sk["STORE"], 3) and typerec.sig_kind("ATOMS") == (sk["ATOMIC"], 0)
    assert typerec.sig_kind("BAR")[0] == typerec.sig_kind("NOT_AN_OPCODE")[0] == sk["NONE"]
    enum = re.search(r"enum cl_sigkind \{(.*?)\};", HEADER, re.S).group(1)
    names = re.findall(r"CL_SK_([A-Z0-9]+)\b", re.sub(r"/\*.*?\*/", "", enum, flags=re.S))
    assert names == typerec._SK                      # same order as enum cl_sigkind
    mt = typerec.mod_type(("F16", "F32"))
    assert mt[4] == typerec.FLOAT16 and mt[5] == typerec.FLOAT32
    assert typerec.mod_type(("F64", "S64"))[2:4] == (typerec.FLOAT64, typerec.INT64)


def test_key_error_on_dead_value():
    """A narrowed value that is not in fn.values: the reference's dict raises KeyError (typerec.py:301)."""
    fix = helpers.load_fixture("types")
    fn = copy.deepcopy(fix["functions"][0])
    inst = next(i for b in fn.block_order() for i in b.instructions if i.defs and type(i.defs[0]).__name__ == "ValueRef"
                and i.opcode.base in ("IADD3", "FADD", "IMAD", "FFMA", "S2R"))
    del fn.values[inst.defs[0].vid]
    with pytest.raises(KeyError):
        typerec.seed_types(fn, helpers.oracle_engine())


@pytest.mark.gpu
def test_cuda_matches_reference_typestate():
    eng = helpers.cuda_engine()
    assert eng.backend == "cuda-sm_100a"
    check_against_golden(eng)


@pytest.mark.gpu
def test_cuda_equals_oracle_on_pool_corpus():
    """Arrays of cl_seed_types on 200 k instructions of the mixed benchmark corpus: CUDA == oracle, bit for bit."""
    from paper_2604_27486_b200 import synth
    corpus = synth.build_corpus("mixed", 200_000, seed=7)[0]
    a = typerec.seed_corpus(helpers.cuda_engine(), corpus)
    b = typerec.seed_corpus(helpers.oracle_engine(), corpus)
    for name in ("val_masks", "role", "link_mask", "link_def", "status"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    assert (a.val_masks != 0xFFFFFF).any()


ARRAYS = ("val_masks", "role", "link_mask", "link_def", "status")


@pytest.mark.parametrize("name", ["bundled", "synth_sm90", "synth_sm52", "synth_sm75", "synth_long", "chains"])
def test_device_code_equals_oracle_on_stage_inputs(name):
    """Same arrays from the device code (one-thread build) and the oracle on the SSA-phase inputs of the stage's goldens
    (overflow-slot records, wide PHIs, guards, terminator conditions, MemRef bases and uniform registers)."""
    fns = helpers.load_fixture(name)["functions"]
    corpus, hints = soa.encode(fns), typerec.hints_of(fns)
    a = typerec.seed_corpus(helpers.sim_engine(), corpus, hints)
    b = typerec.seed_corpus(helpers.oracle_engine(), corpus, hints)
    for n in ARRAYS:
        assert np.array_equal(getattr(a, n), getattr(b, n)), n
    assert (a.val_masks[corpus.val_alive.astype(bool)] != 0xFFFFFF).any()


def test_caller_owned_result_arrays_and_empty_corpus():
    fns = helpers.load_fixture("snippets")["functions"]
    corpus = soa.encode(fns)
    eng = helpers.oracle_engine()
    ref = typerec.seed_corpus(eng, corpus)
    n, nv = corpus.n_insts, len(corpus.val_alive)
    into = typerec.SeedArrays(np.zeros(nv + 5, np.uint32), np.zeros(n + 5, np.uint8), np.zeros(n + 5, np.uint16),
                              np.zeros(n + 5, np.uint32), np.zeros(corpus.n_funcs, np.uint8))
    got = typerec.seed_corpus(eng, corpus, None, upload=False, into=into)
    for name in ARRAYS:
        assert np.array_equal(getattr(got, name), getattr(ref, name)), name
        assert np.shares_memory(getattr(got, name), getattr(into, name))
    with pytest.raises(ValueError):
        typerec.seed_corpus(eng, corpus, None, upload=False,
                            into=typerec.SeedArrays(np.zeros(1, np.uint32), into.role, into.link_mask, into.link_def, into.status))
    with pytest.raises(ValueError):
        typerec.seed_corpus(eng, corpus, typerec.Hints(np.zeros(3, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32)), upload=False)
    empty = corpus.slice_funcs(0, 0)
    for e in (helpers.oracle_engine(), helpers.sim_engine()):
        res = typerec.seed_corpus(e, empty)
        assert len(res.role) == len(res.val_masks) == len(res.status) == 0
    assert typerec.seed_types_batch([], eng) == []


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bundled", "synth_long", "long_blocks"])
def test_cuda_equals_oracle_on_stage_inputs(name):
    fns = helpers.load_fixture(name)["functions"]
    corpus, hints = soa.encode(fns), typerec.hints_of(fns)
    a = typerec.seed_corpus(helpers.cuda_engine(), corpus, hints)
    b = typerec.seed_corpus(helpers.oracle_engine(), corpus, hints)
    for n in ARRAYS:
        assert np.array_equal(getattr(a, n), getattr(b, n)), n


@pytest.mark.gpu
def test_cuda_empty_corpus_and_pinned_result():
    import torch
    fns = helpers.load_fixture("snippets")["functions"]
    corpus = soa.encode(fns)
    eng = helpers.cuda_engine()
    res = typerec.seed_corpus(eng, corpus.slice_funcs(0, 0))
    assert len(res.role) == len(res.val_masks) == len(res.status) == 0
    n, nv = corpus.n_insts, len(corpus.val_alive)
    pinned = [torch.empty(k, dtype=dt, pin_memory=True).numpy() for k, dt in
              ((nv, torch.int32), (n, torch.uint8), (n, torch.int16), (n, torch.int32), (corpus.n_funcs, torch.uint8))]
    into = typerec.SeedArrays(pinned[0].view(np.uint32), pinned[1], pinned[2].view(np.uint16), pinned[3].view(np.uint32), pinned[4])
    got = typerec.seed_corpus(eng, corpus, into=into)
    ref = typerec.seed_corpus(helpers.oracle_engine(), corpus)
    for name in ARRAYS:
        assert np.array_equal(getattr(got, name), getattr(ref, name)), name
    assert eng.last_run_ms() > 0


def check_chained(engine):
    """Stage and seeding chained on the engine (CL_SEED_RESULT) == seeding of the downloaded result."""
    for name in ("bundled", "synth_sm90", "synth_sm52", "chains"):
        fns = helpers.load_fixture(name)["functions"]
        corpus, hints = soa.encode(fns), typerec.hints_of(fns)
        engine.upload(corpus)
        engine.run_postssa(15)
        chained = typerec.seed_corpus(engine, corpus, hints, upload=False, source=typerec.SEED_RESULT)
        result = engine.download()
        assert len(chained.role) == result.n_insts and len(chained.val_masks) == len(result.val_alive)
        oracle = helpers.oracle_engine()
        separate = typerec.seed_corpus(oracle, result, hints)
        for n in ARRAYS:
            assert np.array_equal(getattr(chained, n), getattr(separate, n)), (name, n)
        states = typerec.states_of(result, chained)
        assert len(states) == len(fns)


def test_chained_after_the_stage_oracle():
    check_chained(helpers.oracle_engine())


def test_chained_after_the_stage_device_code():
    check_chained(helpers.sim_engine())


@pytest.mark.gpu
def test_chained_after_the_stage_cuda():
    check_chained(helpers.cuda_engine())


def test_hints_survive_the_stage():
    """The meta table is keyed by iid: the stage keeps the iid of every load, store and tensor op."""
    fns = copy.deepcopy(helpers.load_fixture("types")["functions"])
    hints = typerec.hints_of(fns)
    assert hints is not None and (hints.val > 0xFF).any() and (hints.val & 0xFF).any()     # tensor groups and packed widths
    for f in range(len(fns)):
        run = hints.iid[hints.off[f]:hints.off[f + 1]]
        assert (np.diff(run.astype(np.int64)) > 0).all()


def test_sharded_over_two_engines_equals_one():
    """Two engines, the corpus partitioned by kernel: same arrays, same TypeStates (hints sliced per shard)."""
    fix = helpers.load_fixture("types")
    fns = copy.deepcopy(fix["functions"])
    corpus, hints = soa.encode(fns), typerec.hints_of(fns)
    one = typerec.seed_corpus(helpers.oracle_engine(), corpus, hints)
    for engines in ([helpers.oracle_engine(), helpers.oracle_engine()], [helpers.oracle_engine()] * 3):
        two = typerec.seed_corpus_sharded(engines, corpus, hints)
        for n in ARRAYS:
            assert np.array_equal(getattr(one, n), getattr(two, n)), n
    states = typerec.seed_types_batch(fns, engines=[helpers.oracle_engine(), helpers.oracle_engine()])
    for st, exp in zip(states, fix["expect"]):
        assert st.seed_mask == exp["seed_mask"] and st.link_exprs == exp["link_exprs"] and st.roles == exp["roles"]


def test_bench_leg_shape_on_the_oracle_engine(monkeypatch):
    """bench.py's type-seeding leg end to end on the CPU oracle (small corpus): keys of the object, chained source,
    equality with the separate oracle pass."""
    import sys
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    sys.path.insert(0, str(ROOT))
    import bench
    leg = bench.typeseed_leg(helpers.oracle_engine(), 6538.6, 1, 2, 1, True, n_sass=60_000)
    assert leg["config"] == "typeseed" and leg["equal_to_oracle"] is True
    assert leg["roofline"]["bound"] == "hbm" and leg["roofline"]["algorithmic_bytes_per_launch"] > 0
    assert leg["cpu_baseline"]["kind"] == "port" and leg["e2e"]["d2h_bytes_per_step"] > 0
    assert leg["narrowed_values"] > 0 and leg["transparent_records"] > 0
