"""The plugin/pass API keeps the reference's shapes (patterns.py) -- these
tests read like the reference's tests/test_patterns.py.  The engine is the
one-lane CPU build of the device code here and the CUDA library under -m gpu."""
import copy

import pytest

import helpers
from paper_2604_27486_b200 import ir, passes, patterns


@pytest.fixture(params=["sim", pytest.param("cuda", marks=pytest.mark.gpu)])
def engine(request):
    return helpers.sim_engine() if request.param == "sim" else helpers.cuda_engine()


def snippet(name):
    fix = helpers.load_fixture("snippets")
    return copy.deepcopy(next(f for f in fix["functions"] if f.name == name))


def bundled(name):
    fix = helpers.load_fixture("bundled")
    return copy.deepcopy(next(f for f in fix["functions"] if f.name == name))


def bases(fn):
    return [i.opcode.base for b in fn.block_order() for i in b.instructions]


def test_xmad_triple_becomes_single_imad(engine):          # test_patterns.py:46
    fn = bundled("xmad_pair")
    assert passes.normalize_xmad(fn, engine) is fn
    assert bases(fn) == ["IMAD"]


def test_xmad_untouched_on_sm90(engine):                   # test_patterns.py:53
    fn = snippet("xmad_on_sm90")
    passes.normalize_xmad(fn, engine)
    assert bases(fn).count("XMAD") == 3


def test_fadd_block_matches_nothing(engine):               # test_patterns.py:68
    fn = snippet("fadd_only")
    blk = fn.block_order()[0]
    assert passes.match_patterns(fn, blk, patterns.AGGREGATION_PATTERNS, engine=engine) == []


def test_interleaved_pairs_give_two_disjoint_matches(engine):   # test_patterns.py:75
    fn = snippet("interleaved_pairs")
    blk = fn.block_order()[0]
    ms = passes.match_patterns(fn, blk, patterns.AGGREGATION_PATTERNS, engine=engine)
    sel = passes.select_matches(ms)
    assert [m.pattern.name for m in sel] == ["iadd3.pair", "iadd3.pair"]
    ids = [{i.iid for i in m.insts} for m in sel]
    assert not ids[0] & ids[1]
    assert sel[0].start_pos < sel[1].start_pos
    m = sel[0]
    assert isinstance(m, patterns.Match) and m.block == blk.bid
    assert m.bindings.vars["carry"][0] == "v" and m.bindings.vars["carry"] == passes.operand_key(m.insts[0].aux_defs[0])


def test_inconsistent_carry_binding_rejected(engine):      # test_patterns.py:92
    fn = snippet("inconsistent_carry")
    blk = fn.block_order()[0]
    assert passes.match_patterns(fn, blk, patterns.AGGREGATION_PATTERNS, engine=engine) == []


def test_carry_escape_refuses_with_diagnostic(engine):     # test_patterns.py:104
    fn = snippet("carry_escape")
    passes.apply_aggregations(fn, engine)
    assert "IADD364" not in bases(fn)
    assert any("iadd3.pair matched but rewrite refused" in d for d in fn.diagnostics)


@pytest.mark.parametrize("name", ["carrysub", "fastdiv", "sumloop"])
def test_normalization_is_idempotent(engine, name):        # test_patterns.py:117
    fn = bundled(name)
    passes.gpu_normalize([fn], engine=engine)
    first = ir.dump(fn)
    passes.gpu_normalize([fn], engine=engine)
    # tags are appended again by a second tag pass, exactly as upstream; compare the body
    strip = lambda text: "\n".join(l for l in text.splitlines() if "cuda-object" not in l)
    assert strip(ir.dump(fn)) == strip(first)


def test_reciprocal_inserts_bitcasts(engine):              # test_patterns.py:218
    fn = bundled("fastdiv")
    passes.normalize_reciprocal(fn, engine)
    ops = [str(i.opcode) for b in fn.block_order() for i in b.instructions]
    assert "BITCAST.F2I" in ops and "BITCAST.I2F" in ops
    assert fn.meta["pattern_boundaries"][0]["category"] == "Fast math chains"
    new = [v for v in fn.values.values() if v.origin.endswith(".bits") or v.origin.endswith(".f")]
    assert len(new) == 2


def test_pass_requires_ssa_phase(engine):
    fn = bundled("fastdiv")
    fn.phase = ir.Phase.RAW
    with pytest.raises(RuntimeError, match="requires phase"):
        passes.apply_aggregations(fn, engine)


def test_select_matches_needs_device_list():
    with pytest.raises(TypeError):
        passes.select_matches([object()])


def test_pattern_introspection_lists_all():                # test_patterns.py:257
    text = patterns.describe_patterns()
    names = {line.split(":")[0] for line in text if not line.startswith(" ")}
    assert {"iadd3.pair", "isetp.pair", "lea.pair", "imad.wide", "mov.pair", "shf.cast64",
            "shf.shl64", "shf.shr64", "xmad.mul3.a", "xmad.mul3.b"} == names
    assert text[1].startswith("    XMAD.MRG $m, $a, $b.H1, RZ")


def test_user_pattern_compiles_and_rejects_unknown_rewrite():
    blob = patterns.compile_patterns()
    assert int(blob[0]["n_patterns"]) == 10 and int(blob[0]["budget"]) == 50_000
    bad = patterns.Pattern("x", (patterns.InstTemplate("FOO"),), lambda *a: None)
    with pytest.raises(patterns.PatternError):
        patterns.compile_patterns([bad], [])


def test_custom_pattern_table_runs_on_device(engine):
    """A user-built table entry (same shape as upstream's Pattern) is lowered and matched."""
    only_wide = [p for p in patterns.AGGREGATION_PATTERNS if p.name == "imad.wide"]
    fn = bundled("fastdiv")
    blk = fn.block_order()[1]
    ms = passes.match_patterns(fn, blk, only_wide, engine=engine)
    assert len(ms) == 3 and {m.pattern.name for m in ms} == {"imad.wide"}
    assert passes.select_matches(ms) == ms
