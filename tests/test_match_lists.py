"""The (pattern.name, candidate) match sets of the north star, pinned to the Python
reference: every golden fixture carries the lists the reference's own
match_patterns / select_matches returned for every block of every round
(tools/make_golden.py records them while the reference runs, patterns.py:181-252,
:676).  The engines report theirs as CL_EV_MATCH events (emit_matches); list
order, positions and the selection must be identical -- for the oracle, for the
one-lane build of the device code, and on the GPU for the production kernels
that serve runs asking for match lists (the fused kernels) as well as for the
general per-function kernels."""
import copy

import pytest

import helpers
from paper_2604_27486_b200 import layout as L, soa

FIXTURES = [n for n in helpers.FIXTURES if n != "bundled_noagg"]


def device_match_lists(engine, functions, passes):
    corpus = soa.encode(functions)
    engine.upload(corpus)
    engine.run_postssa(passes, emit_matches=True)
    out = engine.download()
    pats = helpers.engine_patterns(engine)
    per_func = [dict() for _ in functions]
    for ev in out.events:                        # sorted by (func, seq, kind, idx, ...): list order inside a block
        if int(ev["kind"]) != L.EV_MATCH:
            continue
        seq, idx, a = int(ev["seq"]), int(ev["idx"]), int(ev["a"])
        pat = pats[a & 0xFFFF]
        pos = tuple(int(ev[k]) for k in ("b", "c", "d"))[:len(pat.templates)]
        slot = per_func[int(ev["func"])].setdefault((seq >> 28, seq & 0x0FFFFFFF), ([], []))
        slot[1 if idx & 0x80000000 else 0].append((pat.name,) + pos)
    status = [int(s) for s in out.func["status"]]
    return [[(ph, bi, raw, sel) for (ph, bi), (raw, sel) in sorted(d.items())] for d in per_func], status


def check(engine, name):
    fix = helpers.load_fixture(name)
    got, status = device_match_lists(engine, copy.deepcopy(fix["functions"]), fix["passes"])
    n_lists = 0
    for f, (fn, want) in enumerate(zip(fix["functions"], fix["matches"])):
        if want is None:                          # the reference raises on this function
            assert status[f] != 0, f"{name}/{fn.name}"
            continue
        want = [(ph, bi, [tuple(x) for x in raw], [tuple(x) for x in sel]) for ph, bi, raw, sel in want]
        assert got[f] == want, f"{name}/{fn.name}: match lists differ from the reference's\n--- reference\n{want}\n--- got\n{got[f]}"
        n_lists += len(want)
    return n_lists


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_match_lists_equal_the_references(oracle_engine, name):
    check(oracle_engine, name)


@pytest.mark.parametrize("name", FIXTURES)
def test_sim_match_lists_equal_the_references(sim_engine, name):
    """default routing: a run that asks for match lists takes the fused kernels (one-lane build here)"""
    assert check(sim_engine, name) >= 0
    assert sim_engine.debug_partition()["tile_mode"] == 16


@pytest.mark.parametrize("name", [n for n in FIXTURES if n != "long_blocks"])
def test_sim_general_kernels_match_lists(sim_tile_engine, name):
    check(sim_tile_engine, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", FIXTURES)
def test_cuda_match_lists_equal_the_references(cuda_engine, name):
    n = check(cuda_engine, name)
    assert cuda_engine.debug_partition()["tile_mode"] == 16          # the production kernels emitted them
    if name.startswith("synth") or name == "long_blocks":
        assert n > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", FIXTURES)
def test_cuda_general_kernels_match_lists(cuda_tile_engine, name):
    check(cuda_tile_engine, name)
