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


def _mk(pattern, iids, block=0, start=None):
    class _I:                                    # select_matches only looks at inst.iid
        def __init__(self, iid): self.iid = iid
    return patterns.Match(pattern, [_I(i) for i in iids], patterns.Bindings(), block, iids[0] if start is None else start)


def test_select_matches_resolves_any_list_like_the_reference():
    """patterns.py:241-252 on lists the device never saw: caller-built matches, earliest start first,
    longer pattern on ties, greedy over disjoint instructions, stable for equal keys"""
    two, three = patterns.AGGREGATION_PATTERNS[0], patterns.AGGREGATION_PATTERNS[4]
    a, b, c, d = _mk(two, [5, 9]), _mk(three, [5, 6, 7]), _mk(two, [1, 9]), _mk(two, [20, 21])
    assert passes.select_matches([a, b, c, d]) == [c, b, d]       # c starts first and takes 9; b beats a at 5 (longer)
    assert passes.select_matches([d, a]) == [a, d]
    assert passes.select_matches([]) == []


def test_select_matches_on_a_filtered_device_list(engine):
    """the device's precomputed selection is only used for the unmodified list; dropping a competitor
    before the call lets the match it had beaten win, as in the reference"""
    fn = bundled("carrysub")
    blk = max(fn.block_order(), key=lambda b: len(b.instructions))
    ms = passes.match_patterns(fn, blk, patterns.AGGREGATION_PATTERNS, engine=engine)
    full = passes.select_matches(ms)
    assert full == [m for m in sorted(ms, key=lambda m: (m.start_pos, -len(m.pattern))) if m in full]
    if len(ms) > 1:
        rest = ms[1:]
        want, taken = [], set()
        for m in sorted(rest, key=lambda m: (m.start_pos, -len(m.pattern))):
            ids = {i.iid for i in m.insts}
            if not ids & taken:
                taken |= ids; want.append(m)
        assert passes.select_matches(rest) == want


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


def test_match_patterns_keeps_the_engines_own_tables(engine):
    """match_patterns swaps a table in for one call and puts the engine's previous one back (custom tables too)"""
    only_wide = [p for p in patterns.AGGREGATION_PATTERNS if p.name == "imad.wide"]
    engine.set_patterns(only_wide, [])
    try:
        fn = bundled("fastdiv")
        passes.match_patterns(fn, fn.block_order()[1], patterns.AGGREGATION_PATTERNS, engine=engine)
        assert engine.pattern_names() == ["imad.wide"]
        passes.apply_aggregations(fn, engine)
        assert "IMAD64" in bases(fn) and "IADD364" not in bases(fn)
    finally:
        engine.set_patterns()


def test_too_many_seed_opcodes_is_a_pattern_error():
    """the device seed scan holds 12 distinct template opcodes per table: more is refused at compile time"""
    ops = ["FADD", "FMUL", "FFMA", "IADD3", "IADD", "ISETP", "LEA", "IMAD", "SHF", "MOV", "LOP3", "SEL", "PRMT"]
    table = [patterns.Pattern(f"p{k}", (patterns.InstTemplate(op, defs=(patterns.Var("d"),)),), patterns.AGGREGATION_PATTERNS[3].rewrite)
             for k, op in enumerate(ops)]
    with pytest.raises(patterns.PatternError):
        patterns.compile_patterns(table, [])
