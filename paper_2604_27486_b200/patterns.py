"""Pattern/pass plugin API of the hot path, GPU-backed.

Mirrors the public surface of the reference ``sasslift.patterns`` (same names,
argument meaning and error behaviour) so that a user of the reference can swap
the import:

* slot types ``Var LitRZ LitPT LitImm Any``, ``InstTemplate``, ``Pattern``,
  ``Bindings``, ``Match``                      -> ``patterns.py:36-106``
* ``AGGREGATION_PATTERNS / XMAD_PATTERNS / ALL_PATTERNS``  -> ``:531-664``
* ``match_patterns``, ``select_matches``       -> ``:181, :241``
* ``apply_aggregations normalize_xmad normalize_reciprocal tag_cuda_objects``
                                                 -> ``:794, :805, :817, :895``
* ``describe_patterns``                          -> ``:919``

Nothing here computes on the host: the table entries are *data* that
``compile_patterns`` lowers to the device blob (``cl_pattern_blob`` in
``include/culifter.h``) and every pass function encodes its argument, runs the
CUDA library and decodes the result back in place.  ``Pattern.rewrite`` names
one of the nine device rewrite plans instead of holding a Python callable; a
live reference ``Pattern`` is accepted too (its callable is resolved by name).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .layout import MAX_GROUPS, TABLES

CMP_CONDS = ("EQ", "NE", "LT", "LE", "GT", "GE")
BOOL_OPS = ("AND", "OR", "XOR")


# ------------------------------------------------------------- template slots
@dataclass(frozen=True)
class Var:
    name: str
    negated: bool | None = None   # None = don't care
    bitnot: bool | None = None
    half: str | None = None


@dataclass(frozen=True)
class LitRZ:
    pass


@dataclass(frozen=True)
class LitPT:
    negated: bool | None = None


@dataclass(frozen=True)
class LitImm:
    bits: int


@dataclass(frozen=True)
class Any:
    pass


@dataclass(frozen=True)
class InstTemplate:
    base: str
    mods_all: tuple = ()
    mods_none: tuple = ()
    mod_vars: tuple = ()          # ((var, choices), ...)
    defs: tuple = ()
    aux: tuple = ()
    uses: tuple = ()


@dataclass(frozen=True)
class DeviceRewrite:
    """Names one of the device rewrite plans (``enum cl_rewrite``)."""
    kind: str

    @property
    def __name__(self):
        return "_rw_" + self.kind

    def __call__(self, fn, du, match):
        raise RuntimeError(
            f"rewrite {self.kind!r} is a device plan: run apply_aggregations / "
            f"normalize_xmad (or gpu_normalize) instead of calling it on the host")


@dataclass
class Pattern:
    name: str
    templates: tuple
    rewrite: object
    description: str = ""

    def __len__(self):
        return len(self.templates)


@dataclass
class Bindings:
    vars: dict = field(default_factory=dict)

    def bind(self, name, key) -> bool:
        if self.vars.get(name, key) != key:
            return False
        self.vars[name] = key
        return True


@dataclass
class Match:
    pattern: Pattern
    insts: list
    bindings: Bindings
    block: int
    start_pos: int


REWRITE_KINDS = ("iadd364", "isetp64", "lea64", "imad_wide", "mov64", "cast64", "shl64",
                 "shr64", "xmad")
_RW = {k: DeviceRewrite(k) for k in REWRITE_KINDS}
_ = Any()
_RZ = LitRZ()


def _v(name, **kw):
    return Var(name, **kw)


def _shf_pack_tail():
    return InstTemplate("PACK64", defs=(_v("p"),), uses=(_v("lo_d"), _v("hi_d")))


_CMP_VARS = (("cond", CMP_CONDS), ("bop", BOOL_OPS))

# The table *content* is fixed by the reference (order included: it is the
# tie-break of the stable sort in select_matches).
AGGREGATION_PATTERNS: list = [
    Pattern("iadd3.pair", (
        InstTemplate("IADD3", mods_none=("X",), defs=(_v("lo_d"),), aux=(_v("carry"),),
                     uses=(_, _, _)),
        InstTemplate("IADD3", mods_all=("X",), defs=(_v("hi_d"),),
                     uses=(_, _, _, _v("carry"), _)),
    ), _RW["iadd364"], "carry-chain IADD3 + IADD3.X pair -> 64-bit IADD364"),
    Pattern("isetp.pair", (
        InstTemplate("ISETP", mods_all=("U32",), mods_none=("EX",), mod_vars=_CMP_VARS,
                     defs=(_v("pl"),), uses=(_, _, _v("acc"))),
        InstTemplate("ISETP", mods_all=("EX",), mod_vars=_CMP_VARS,
                     defs=(_v("ph"),), uses=(_, _, _v("acc"), _v("pl"))),
    ), _RW["isetp64"], "64-bit compare across two predicate halves -> ISETP64"),
    Pattern("lea.pair", (
        InstTemplate("LEA", mods_none=("HI", "X"), defs=(_v("lo_d"),), aux=(_v("carry"),),
                     uses=(_v("a"), _, _v("sh"))),
        InstTemplate("LEA", mods_all=("HI", "X"), defs=(_v("hi_d"),),
                     uses=(_v("a"), _, _, _v("sh"), _v("carry"))),
    ), _RW["lea64"], "64-bit effective address LEA + LEA.HI.X -> LEA64"),
    Pattern("imad.wide", (
        InstTemplate("IMAD", mods_all=("WIDE",), defs=(_v("d"),), uses=(_, _, _)),
    ), _RW["imad_wide"], "widening 32x32->64 multiply -> IMAD64"),
    Pattern("mov.pair", (
        InstTemplate("MOV", defs=(_v("lo_d"),), uses=(_v("clo"),)),
        InstTemplate("MOV", defs=(_v("hi_d"),), uses=(_v("chi"),)),
        _shf_pack_tail(),
    ), _RW["mov64"], "adjacent constant-bank moves feeding a pair -> MOV64"),
    Pattern("shf.cast64", (
        InstTemplate("SHF", mods_all=("R", "S32", "HI"), defs=(_v("hi_d"),),
                     uses=(_RZ, LitImm(0x1F), _v("x"))),
        InstTemplate("PACK64", defs=(_v("p"),), uses=(_v("x"), _v("hi_d"))),
    ), _RW["cast64"], "SHF.R sign-word extraction feeding a pair -> CAST64 (sext)"),
    Pattern("shf.shl64", (
        InstTemplate("SHF", mods_all=("L", "U64", "HI"), defs=(_v("hi_d"),),
                     uses=(_v("lo"), _v("sh"), _v("hi"))),
        InstTemplate("SHF", mods_all=("L", "U32"), defs=(_v("lo_d"),),
                     uses=(_v("lo"), _v("sh"), _RZ)),
        _shf_pack_tail(),
    ), _RW["shl64"], "two-part SHF left shift feeding a pair -> SHL64"),
    Pattern("shf.shr64", (
        InstTemplate("SHF", mods_all=("R", "HI"), mods_none=("L",), defs=(_v("hi_d"),),
                     uses=(_v("lo"), _v("sh"), _v("hi"))),
        InstTemplate("SHF", mods_all=("R",), mods_none=("HI", "L"), defs=(_v("lo_d"),),
                     uses=(_v("lo"), _v("sh"), _v("hi"))),
        _shf_pack_tail(),
    ), _RW["shr64"], "two-part SHF right shift feeding a pair -> SHR64"),
]

_XMAD_HEAD = InstTemplate("XMAD", mods_all=("MRG",), defs=(_v("m"),),
                          uses=(_v("a"), _v("b", half="H1"), _RZ))
XMAD_PATTERNS: list = [
    Pattern("xmad.mul3.a", (
        _XMAD_HEAD,
        InstTemplate("XMAD", mods_none=("MRG", "PSL"), defs=(_v("t"),),
                     uses=(_v("a"), _v("m"), _RZ)),
        InstTemplate("XMAD", mods_all=("PSL", "CBCC"), defs=(_v("d"),),
                     uses=(_v("a", half="H1"), _v("t"), _v("c"))),
    ), _RW["xmad"], "SM52 XMAD/XMAD.MRG/XMAD.PSL.CBCC multiply idiom -> IMAD"),
    Pattern("xmad.mul3.b", (
        _XMAD_HEAD,
        InstTemplate("XMAD", mods_none=("MRG", "PSL"), defs=(_v("t"),),
                     uses=(_v("a"), _v("b"), _v("c"))),
        InstTemplate("XMAD", mods_all=("PSL", "CBCC"), defs=(_v("d"),),
                     uses=(_v("a", half="H1"), _v("m", half="H1"), _v("t"))),
    ), _RW["xmad"], "SM52 XMAD address-computation idiom -> IMAD"),
]

ALL_PATTERNS = XMAD_PATTERNS + AGGREGATION_PATTERNS


# ---------------------------------------------------------- table -> device blob
MAX_PATTERNS, MAX_TEMPLATES, MAX_VARS = 16, 3, 16
MAX_CLS = 12            # seed classes of one table (core.cuh MAX_CLS)
PATTERN_MAGIC = 0x434C5054
S_ANY, S_VAR, S_RZ, S_PT, S_IMM = range(5)

SLOT = np.dtype([("kind", "u1"), ("var", "u1"), ("neg", "u1"), ("bitnot", "u1"),
                 ("half", "u1"), ("pad", "u1", (3,)), ("imm", "<u8")])
TEMPLATE = np.dtype([("op", "<u2"), ("n_defs", "u1"), ("n_aux", "u1"), ("n_uses", "u1"),
                     ("n_modvars", "u1"), ("modvar_var", "u1", (2,)),
                     ("modvar_group", "u1", (2,)), ("pad", "u1", (6,)),
                     ("mods_all", "<u8"), ("mods_none", "<u8"), ("slot", SLOT, (8,))])
PATTERN = np.dtype([("n_templates", "u1"), ("rewrite", "u1"), ("n_vars", "u1"),
                    ("table", "u1"), ("var_a", "u1"), ("var_b", "u1"), ("var_c", "u1"),
                    ("modvar_cond", "u1"), ("modvar_bop", "u1"), ("join_ok", "u1"),
                    ("join_order", "u1", (3,)), ("join_from", "u1", (3,)), ("join_slot", "u1", (3,)),
                    ("pad", "u1", (13,)),
                    ("t", TEMPLATE, (MAX_TEMPLATES,))])
BLOB = np.dtype([("magic", "<u4"), ("n_patterns", "<u4"), ("n_groups", "<u4"),
                 ("budget", "<u4"), ("group_mask", "<u8", (MAX_GROUPS,)),
                 ("group_pos", "u1", (64,)), ("isetp64_ms", "<u2", (8, 2, 8)),
                 ("p", PATTERN, (MAX_PATTERNS,))])
assert (SLOT.itemsize, TEMPLATE.itemsize, PATTERN.itemsize, BLOB.itemsize) == \
    (16, 160, 512, 8560)

_TRI = {None: 0, False: 1, True: 2}
_HALF = {None: 0, "H0": 1, "H1": 2}


class PatternError(ValueError):
    """A table entry cannot be lowered to the device (loud, at compile time)."""


def _rewrite_kind(pat) -> int:
    name = getattr(pat.rewrite, "kind", None) or getattr(pat.rewrite, "__name__", "")
    name = name.removeprefix("_rw_")
    if name not in REWRITE_KINDS:
        raise PatternError(f"pattern {pat.name!r}: rewrite {pat.rewrite!r} is not one of "
                           f"the device plans {REWRITE_KINDS}")
    return REWRITE_KINDS.index(name)


def _slot(slot, var_ids, pat):
    kind = type(slot).__name__
    if kind == "Any":
        return (S_ANY, 0, 0, 0, 0, (0, 0, 0), 0)
    if kind == "LitRZ":
        return (S_RZ, 0, 0, 0, 0, (0, 0, 0), 0)
    if kind == "LitPT":
        return (S_PT, 0, _TRI[slot.negated], 0, 0, (0, 0, 0), 0)
    if kind == "LitImm":
        return (S_IMM, 0, 0, 0, 0, (0, 0, 0), slot.bits & (1 << 64) - 1)
    if kind == "Var":
        if slot.name not in var_ids:
            if len(var_ids) >= MAX_VARS:
                raise PatternError(f"pattern {pat.name!r}: more than {MAX_VARS} variables")
            var_ids[slot.name] = len(var_ids)
        if slot.half not in _HALF:
            raise PatternError(f"pattern {pat.name!r}: half selector {slot.half!r}")
        return (S_VAR, var_ids[slot.name], _TRI[slot.negated], _TRI[slot.bitnot],
                _HALF[slot.half], (0, 0, 0), 0)
    raise PatternError(f"pattern {pat.name!r}: unknown slot {slot!r}")


def _join_plan(pat):
    """Resolution order that replaces the candidate product by def-use lookups:
    -> [(template, from_template, from_slot)] with the anchor first, or None."""
    tm = pat.templates
    n = len(tm)
    slots = [tuple(t.defs) + tuple(t.aux) + tuple(t.uses) for t in tm]
    ndef = [len(t.defs) + len(t.aux) for t in tm]
    isvar = lambda s: type(s).__name__ == "Var"
    for anchor in reversed(range(n)):
        plan, done = [(anchor, 0, 0)], {anchor}
        while len(done) < n:
            found = None
            for t in range(n):
                if t in done:
                    continue
                names = {s.name for s in slots[t][:ndef[t]] if isvar(s)}
                for r in plan:
                    for k, s in enumerate(slots[r[0]]):
                        if k >= ndef[r[0]] and isvar(s) and s.name in names:
                            found = (t, r[0], k)
                            break
                    if found:
                        break
                if found:
                    break
            if not found:
                break
            plan.append(found)
            done.add(found[0])
        if len(done) == n:
            return plan
    return None


def compile_patterns(aggregation=None, xmad=None, budget: int = 50_000) -> np.ndarray:
    """Lower the two pattern tables to one ``cl_pattern_blob`` (shape ``(1,)``).

    Patterns keep table order; ``table`` tells the device which pass owns an
    entry (0 = ``apply_aggregations``, 1 = ``normalize_xmad``, G19)."""
    aggregation = AGGREGATION_PATTERNS if aggregation is None else aggregation
    xmad = XMAD_PATTERNS if xmad is None else xmad
    pats = [(p, 0) for p in aggregation] + [(p, 1) for p in xmad]
    if len(pats) > MAX_PATTERNS:
        raise PatternError(f"{len(pats)} patterns, the device table holds {MAX_PATTERNS}")
    blob = np.zeros(1, BLOB)
    b = blob[0]
    b["magic"], b["n_patterns"], b["budget"] = PATTERN_MAGIC, len(pats), budget
    isetp_groups = None
    for i, (pat, table) in enumerate(pats):
        rec = b["p"][i]
        if not 1 <= len(pat.templates) <= MAX_TEMPLATES:
            raise PatternError(f"pattern {pat.name!r}: {len(pat.templates)} templates")
        var_ids, modvar_ids = {}, {}
        rec["n_templates"], rec["rewrite"], rec["table"] = \
            len(pat.templates), _rewrite_kind(pat), table
        for t, tmpl in enumerate(pat.templates):
            tr = rec["t"][t]
            slots = tuple(tmpl.defs) + tuple(tmpl.aux) + tuple(tmpl.uses)
            if len(slots) > 8:
                raise PatternError(f"pattern {pat.name!r}: template {t} has {len(slots)} "
                                   f"operand slots, records hold 8")
            if len(tmpl.mod_vars) > 2:
                raise PatternError(f"pattern {pat.name!r}: more than 2 mod_vars")
            tr["op"] = TABLES.opcode(tmpl.base)
            tr["n_defs"], tr["n_aux"], tr["n_uses"] = \
                len(tmpl.defs), len(tmpl.aux), len(tmpl.uses)
            tr["mods_all"] = sum(1 << TABLES.mod_bit(m) for m in set(tmpl.mods_all))
            tr["mods_none"] = sum(1 << TABLES.mod_bit(m) for m in set(tmpl.mods_none))
            tr["n_modvars"] = len(tmpl.mod_vars)
            for k, (var, choices) in enumerate(tmpl.mod_vars):
                if var not in modvar_ids:
                    if len(modvar_ids) >= MAX_GROUPS:
                        raise PatternError(f"pattern {pat.name!r}: too many mod vars")
                    modvar_ids[var] = len(modvar_ids)
                tr["modvar_var"][k] = modvar_ids[var]
                tr["modvar_group"][k] = TABLES.group(choices)
            for k, slot in enumerate(slots):
                tr["slot"][k] = _slot(slot, var_ids, pat)
        rec["n_vars"] = len(var_ids)
        plan = _join_plan(pat)
        if plan is not None:
            rec["join_ok"] = 1
            for k, (t, frm, slot) in enumerate(plan):
                rec["join_order"][k], rec["join_from"][k], rec["join_slot"][k] = t, frm, slot
        rec["var_a"] = rec["var_b"] = rec["var_c"] = 0xFF
        rec["modvar_cond"] = rec["modvar_bop"] = 0xFF
        kind = REWRITE_KINDS[int(rec["rewrite"])]
        if kind == "xmad":
            missing = [v for v in "abc" if v not in var_ids]
            if missing or len(pat.templates) != 3:
                raise PatternError(f"pattern {pat.name!r}: the xmad plan needs three "
                                   f"templates binding $a $b $c (missing {missing})")
            rec["var_a"], rec["var_b"], rec["var_c"] = (var_ids[v] for v in "abc")
        if kind == "isetp64":
            if "cond" not in modvar_ids or "bop" not in modvar_ids:
                raise PatternError(f"pattern {pat.name!r}: the isetp64 plan needs mod_vars "
                                   f"'cond' and 'bop'")
            rec["modvar_cond"], rec["modvar_bop"] = modvar_ids["cond"], modvar_ids["bop"]
            choices = {}
            for tmpl in pat.templates:
                for var, ch in tmpl.mod_vars:
                    choices.setdefault(var, tuple(ch))
            groups = (choices["cond"], choices["bop"])
            if isetp_groups not in (None, groups):
                raise PatternError("isetp64 patterns disagree on their modifier choices")
            isetp_groups = groups
        want = {"iadd364": 2, "isetp64": 2, "lea64": 2, "imad_wide": 1, "mov64": 3,
                "cast64": 2, "shl64": 3, "shr64": 3, "xmad": 3}[kind]
        if len(pat.templates) != want:
            raise PatternError(f"pattern {pat.name!r}: plan {kind} rewrites {want} "
                               f"instructions, the pattern has {len(pat.templates)}")
    for table, name in ((0, "aggregation"), (1, "xmad")):
        bases = {tmpl.base for pat, t in pats if t == table for tmpl in pat.templates}
        if len(bases) > MAX_CLS:
            raise PatternError(f"the {name} table uses {len(bases)} distinct template opcodes, the device seed scan holds {MAX_CLS}")
    b["n_groups"] = len(TABLES.groups)
    pos = np.zeros(64, np.uint8)
    for g, choices in reversed(list(enumerate(TABLES.groups))):
        mask = 0
        for k, name in enumerate(choices):
            bit = TABLES.mod_bit(name)
            mask |= 1 << bit
            pos[bit] = k
        b["group_mask"][g] = mask
    b["group_pos"] = pos
    if isetp_groups is not None:
        conds, bops = isetp_groups
        if len(conds) > 8 or len(bops) > 8:
            raise PatternError("isetp64: more than 8 comparison / boolean choices")
        for ci, c in enumerate(conds):
            for u in (0, 1):
                for bi, bo in enumerate(bops):
                    mods = (c,) + (("U64",) if u else ()) + (bo,)
                    b["isetp64_ms"][ci][u][bi] = TABLES.modset(mods)
    return blob


def pattern_list(aggregation=None, xmad=None):
    """Patterns in blob order (index = ``cl_event`` pattern id)."""
    return list(AGGREGATION_PATTERNS if aggregation is None else aggregation) + \
        list(XMAD_PATTERNS if xmad is None else xmad)


def key_from_device(cls: int, payload: int):
    """Binding key in the reference's tuple form (``operand_key``, ``:109-127``)."""
    raise NotImplementedError


# ----------------------------------------------------------------- introspection
def _slot_str(s) -> str:
    kind = type(s).__name__
    if kind == "Var":
        return "$" + s.name + ("-" if s.negated else "") + ("~" if s.bitnot else "") + \
            (f".{s.half}" if s.half else "")
    return {"LitRZ": "RZ", "LitPT": "PT"}.get(kind) or \
        (hex(s.bits) if kind == "LitImm" else "_")


def describe_patterns() -> list:
    """Same text as the reference's ``describe_patterns`` (``:919-927``)."""
    out = []
    for p in ALL_PATTERNS:
        out.append(f"{p.name}: {p.description}")
        for t in p.templates:
            head = ".".join((t.base,) + tuple(t.mods_all))
            out.append(f"    {head} " + ", ".join(map(_slot_str, t.defs + t.aux + t.uses)))
    return out
