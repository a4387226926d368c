"""The C encoder (csrc/codec.c) against the Python walk it replaces, on every
fixture the reference's front half produced (tests/golden): every plane of the
corpus byte for byte, the interned tables included; encode -> apply restores
objects that dump() the same text."""
import copy
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))
import helpers  # noqa: E402
from paper_2604_27486_b200 import soa  # noqa: E402

SSA_FIXTURES = ["bundled", "bundled_noagg", "snippets", "synth_sm52", "synth_sm75", "synth_sm90", "synth_long", "long_blocks"]


def test_codec_is_the_product_encoder():
    mod = soa._load_codec()
    assert Path(mod.__file__).parent == ROOT / "paper_2604_27486_b200", mod.__file__     # built in-tree


@pytest.mark.parametrize("name", SSA_FIXTURES)
def test_c_encoder_equals_python_walk(name):
    fns = helpers.load_fixture(name)["functions"]
    a, b = soa.encode(fns), soa.encode_py(fns)
    assert a.n_insts == b.n_insts and a.n_insts > 0
    assert not a.equal(b)
    assert a.hdr.tobytes() == b.hdr.tobytes() and a.blk.tobytes() == b.blk.tobytes() and a.func.tobytes() == b.func.tobytes()


def test_raw_phase_keeps_the_python_walk():
    fns = helpers.load_fixture("raw_x4")["functions"]
    assert not soa.encode(fns, raw=True).equal(soa.encode_py(fns, raw=True))


@pytest.mark.parametrize("name", ["bundled", "synth_sm90"])
def test_encode_apply_round_trip_keeps_the_dump(name):
    fns = copy.deepcopy(helpers.load_fixture(name)["functions"])
    from paper_2604_27486_b200 import ir
    before = [ir.dump(fn) for fn in fns]
    c = soa.encode(fns)
    soa.apply(c, fns, tagged=False)
    assert [ir.dump(fn) for fn in fns] == before


def test_encoder_errors_are_loud():
    fns = copy.deepcopy(helpers.load_fixture("bundled")["functions"])
    inst = next(i for b in fns[0].block_order() for i in b.instructions if i.uses)
    inst.uses[0] = object()
    with pytest.raises(soa.EncodeError):
        soa.encode(fns)


@pytest.mark.parametrize("name", ["bundled", "synth_sm90", "synth_sm52", "synth_long", "chains"])
def test_apply_keeping_untouched_records_equals_full_decode(name, monkeypatch):
    """soa.apply(c_in=...) skips the records the stage left byte-identical; the objects must come out as from a full decode"""
    from paper_2604_27486_b200 import ir
    fix = helpers.load_fixture(name)
    eng = helpers.sim_engine()
    dumps, kept = [], []
    for full in (False, True):
        fns = copy.deepcopy(fix["functions"])
        if full:
            monkeypatch.setenv("CL_TEST_FULL_DECODE", "1")
        corpus, out = helpers.run_postssa(eng, fns, fix["passes"])
        dumps.append([(ir.dump(fn), sorted(fn.values), fn._next_vid, fn._next_iid, fn.meta.get("cuda_objects"), fn.meta.get("pattern_boundaries"))
                      for fn in fns])
        kept.append(int(soa.unchanged_records(corpus, out).sum()))
    assert dumps[0] == dumps[1]
    assert kept[0] > 0                                   # the shortcut is actually taken
