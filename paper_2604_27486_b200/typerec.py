"""Type seeding on the device: drop-in for ``sasslift.typerec.seed_types``
(reference ``typerec.py:288-345``) and its signature table ``signature_for``
(``typerec.py:78-235``) -- SURVEY section 8 row f3, the step right after the
normalisation + aggregation stage, over the same SoA corpus.

The C ABI is ``include/culifter_types.h`` (``cl_seed_types``).  The host side
here only (1) lowers the string-keyed parts of the signature table to per-id
tables -- which branch of ``signature_for`` an opcode takes
(``frontend.OPCODE_TABLE``, ``frontend.py:42-86``) and what a modifier tuple says
about element types -- (2) packs the three ``Instruction.meta`` keys the
signatures read into one u32 per record, and (3) reshapes the device's arrays
into the reference's ``TypeState`` dicts.  All narrowing happens in the kernel.
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field

import numpy as np

from . import layout as L
from . import soa

# lattice.py:13-33
INT32, FLOAT32, INT64, FLOAT64, INT128, BOOL, FLOAT16, BF16 = (1 << i for i in range(8))
NUM32, NUM64, NUM128, NUM16 = INT32 | FLOAT32, INT64 | FLOAT64, INT128, FLOAT16 | BF16
TOP = 0xFF
LEAVES = ("Int32", "Float32", "Int64", "Float64", "Int128", "Bool", "Float16", "BF16")

ROLES = ("seed", "transparent", "conversion")
NO_VALUE = 0xFFFFFFFF

# enum cl_sigkind, in header order
_SK = ("NONE FALU FSEL FCMP DALU DCMP HALU HCMP IMAD LOP SHF SHLR IADD3 IADD LEA IALU ICMP PRED MOV SEL SELECT PHI "
       "SREG SHUFFLE VOTE I2F F2I F2F I2I FRND CAST64 BITCAST LOAD STORE ATOMIC TENSOR IADD364 ISETP64 LEA64 IMAD64 "
       "MOV64 SH64 PACK64 PACK128 UNPACK64 UNPACK128").split()
SK = {n: i for i, n in enumerate(_SK)}
OT_ADDR64, OT_RED = 1, 2
MT_WIDE, MT_HI, MT_F32, MT_F2I, MT_I2F = 1, 2, 4, 8, 16

OPTYPE = np.dtype([("kind", "u1"), ("flags", "u1")])
MODTYPE = np.dtype([("f16_elem", "u1"), ("mma_elem", "u1"), ("conv_float", "u1"), ("conv_int", "u1"),
                    ("f2f_dst", "u1"), ("f2f_src", "u1"), ("atom_elem", "u1"), ("flags", "u1")])

# category of a base mnemonic: the data contract of frontend.OPCODE_TABLE (frontend.py:42-86)
_CATEGORY = {
    "falu": "FADD FMUL FFMA FMNMX FSEL FSET MUFU", "fcmp": "FSETP", "dalu": "DADD DMUL DFMA", "dcmp": "DSETP",
    "halu": "HADD2 HMUL2 HFMA2", "hcmp": "HSETP2",
    "ialu": "IADD IADD3 IMAD IMNMX IABS LOP LOP3 LEA FLO POPC BREV PRMT XMAD P2R UIADD3 ULEA ULOP3 UIMAD",
    "icmp": "ISETP", "pred": "PLOP3", "sreg": "S2R CS2R", "shuffle": "SHFL", "vote": "VOTE VOTEU",
    "load": "ULDC LDG LD LDS LDL LDC", "store": "STG ST STS STL RED", "atomic": "ATOM ATOMS ATOMG",
    "tensor": "HMMA IMMA HGMMA",
}
CATEGORY = {base: cat for cat, names in _CATEGORY.items() for base in names.split()}
GLOBAL_SPACE = {"LDG", "STG", "LD", "ST", "ATOM", "ATOMG", "RED"}       # frontend.py:89

# bases the if-chain of signature_for names directly, in its order of precedence
_BY_BASE_FIRST = {"LOP": "LOP", "LOP3": "LOP", "SHF": "SHF", "USHF": "SHF", "SHL": "SHLR", "SHR": "SHLR",
                  "IADD3": "IADD3", "UIADD3": "IADD3", "IADD": "IADD", "LEA": "LEA", "ULEA": "LEA",
                  "IMAD": "IMAD", "UIMAD": "IMAD"}
_BY_CAT_FLOAT = {"falu": "FALU", "fcmp": "FCMP", "dalu": "DALU", "dcmp": "DCMP", "halu": "HALU", "hcmp": "HCMP"}
_BY_CAT_INT = {"ialu": "IALU", "icmp": "ICMP", "pred": "PRED"}
_BY_BASE_MID = {"MOV": "MOV", "MOV32I": "MOV", "UMOV": "MOV", "SEL": "SEL", "USEL": "SEL", "SELECT": "SELECT", "PHI": "PHI"}
_BY_CAT_MID = {"sreg": "SREG", "shuffle": "SHUFFLE", "vote": "VOTE"}
_BY_BASE_CONV = {n: n for n in ("I2F", "F2I", "F2F", "I2I", "FRND", "CAST64", "BITCAST")}
_BY_CAT_MEM = {"load": "LOAD", "store": "STORE", "atomic": "ATOMIC", "tensor": "TENSOR"}
_BY_BASE_LAST = {"IADD364": "IADD364", "ISETP64": "ISETP64", "LEA64": "LEA64", "IMAD64": "IMAD64", "MOV64": "MOV64",
                 "SHL64": "SH64", "SHR64": "SH64", "PACK64": "PACK64", "PACK128": "PACK128", "UNPACK64": "UNPACK64",
                 "UNPACK128": "UNPACK128"}


def sig_kind(base: str) -> tuple[int, int]:
    """(cl_sigkind, CL_OT_* flags) of a base mnemonic: the branch ``signature_for`` takes
    (typerec.py:87-234; the order of the tests below is the order of its if-chain)."""
    cat = CATEGORY.get(base)
    if cat in _BY_CAT_FLOAT:
        name = "FSEL" if base == "FSEL" else _BY_CAT_FLOAT[cat]
    elif base in _BY_BASE_FIRST:
        name = _BY_BASE_FIRST[base]
    elif cat in _BY_CAT_INT:
        name = _BY_CAT_INT[cat]
    elif base in _BY_BASE_MID:
        name = _BY_BASE_MID[base]
    elif cat in _BY_CAT_MID:
        name = _BY_CAT_MID[cat]
    elif base in _BY_BASE_CONV:
        name = _BY_BASE_CONV[base]
    elif cat in _BY_CAT_MEM:
        name = _BY_CAT_MEM[cat]
    else:
        name = _BY_BASE_LAST.get(base, "NONE")
    flags = 0
    if name in ("LOAD", "STORE") and base in GLOBAL_SPACE:
        flags |= OT_ADDR64
    if name == "ATOMIC" and base in ("ATOM", "ATOMG"):
        flags |= OT_ADDR64
    if base == "RED":
        flags |= OT_RED
    return SK[name], flags


def _conv_float(mods, default=FLOAT32):          # typerec.py:58-66
    if "F64" in mods:
        return FLOAT64
    if "F16" in mods:
        return FLOAT16
    if "BF16" in mods:
        return BF16
    return default


def mod_type(mods) -> tuple:
    """cl_modtype of an ordered modifier tuple (typerec.py:46-71, :158-162, :243-248)."""
    fm = [m for m in mods if m in ("F64", "F32", "F16", "BF16")]
    flags = (MT_WIDE * ("WIDE" in mods) | MT_HI * ("HI" in mods) | MT_F32 * ("F32" in mods)
             | MT_F2I * ("F2I" in mods) | MT_I2F * ("I2F" in mods))
    return (BF16 if "BF16" in mods else FLOAT16,
            BF16 if "BF16" in mods else INT32 if "TF32" in mods else FLOAT16,
            _conv_float(mods),
            INT64 if ("S64" in mods or "U64" in mods) else INT32,
            _conv_float(fm[:1]) if fm else FLOAT32,
            _conv_float(fm[1:2]) if len(fm) > 1 else FLOAT32,
            FLOAT32 if "F32" in mods else FLOAT64 if "F64" in mods else INT32,
            flags)


def op_table() -> np.ndarray:
    out = np.zeros(len(L.TABLES.op_name), OPTYPE)
    for i, base in enumerate(L.TABLES.op_name):
        out[i] = sig_kind(base)
    return out


def mod_table() -> np.ndarray:
    out = np.zeros(len(L.TABLES.modset_tuple), MODTYPE)
    for i, mods in enumerate(L.TABLES.modset_tuple):
        out[i] = mod_type(mods)
    return out


@dataclass
class Hints:
    """``cl_typehints``: per function a run of (iid, packed meta) sorted by iid."""
    off: np.ndarray
    iid: np.ndarray
    val: np.ndarray


def hints_of(functions) -> Hints | None:
    """The three ``Instruction.meta`` keys the signatures read (``packed_def_width``, ``packed_data_width``,
    ``tensor_groups``) as a sparse table keyed by iid; None when no instruction has one."""
    off, iids, vals = [0], [], []
    for fn in functions:
        rows = []
        for blk in fn.block_order():
            for inst in blk.instructions:
                m = inst.meta
                if not m:
                    continue
                g = m.get("tensor_groups") or {}
                if "packed_data_width" in m and not m["packed_data_width"]:
                    raise soa.EncodeError("packed_data_width = 0 cannot be encoded")
                h = ((m.get("packed_def_width") or 0) & 15) | ((m.get("packed_data_width", 0) or 0) & 15) << 4 \
                    | (g.get("a", 0) & 255) << 8 | (g.get("b", 0) & 255) << 16 | (g.get("c", 0) & 255) << 24
                if h:
                    rows.append((inst.iid, h))
        rows.sort()
        iids += [r[0] for r in rows]
        vals += [r[1] for r in rows]
        off.append(len(iids))
    if not iids:
        return None
    return Hints(np.asarray(off, np.uint32), np.asarray(iids, np.uint32), np.asarray(vals, np.uint32))


class TypeHints(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("off", "iid", "val")]


SEED_INPUT, SEED_RESULT = 0, 1


class TypeSeed(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("val_masks", "role", "link_mask", "link_def", "status")]


@dataclass
class SeedArrays:
    """What ``cl_seed_types`` returns, as arrays over the corpus."""
    val_masks: np.ndarray
    role: np.ndarray
    link_mask: np.ndarray
    link_def: np.ndarray
    status: np.ndarray


def seed_corpus(engine, corpus: soa.Corpus, hints: Hints | None = None, upload: bool = True,
                into: SeedArrays | None = None, source: int = SEED_INPUT) -> SeedArrays:
    """``cl_seed_types`` over an encoded corpus (the batch entry; ``upload=False`` reuses the
    corpus the engine already holds; ``into``: caller-owned result arrays, e.g. pinned host memory).
    ``source=SEED_RESULT`` seeds the result the last ``run_postssa`` left on the device (no host round trip
    between the stage and the seeding); ``corpus`` is then the corpus that was uploaded."""
    lib = engine.lib
    if not hasattr(lib, "cl_seed_types"):
        raise RuntimeError("this build of the library has no cl_seed_types (include/culifter_types.h)")
    lib.cl_seed_types.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                  C.POINTER(TypeHints), C.POINTER(TypeSeed)]
    if upload:
        if source != SEED_INPUT:
            raise ValueError("seed_corpus: source=SEED_RESULT needs the run that made the result (upload=False)")
        engine.upload(corpus)
    ops, mods = op_table(), mod_table()
    n, nv = corpus.n_insts, len(corpus.val_alive)
    if source == SEED_RESULT:
        sizes = (C.c_uint64 * 6)()
        engine._check(lib.cl_out_sizes(engine._ctx, sizes))
        n, nv = int(sizes[0]), int(sizes[4])
    if hints is not None and (len(hints.off) != corpus.n_funcs + 1 or len(hints.iid) != len(hints.val)
                              or int(hints.off[-1]) != len(hints.iid)):
        raise ValueError(f"hints: offsets for {len(hints.off) - 1} functions, corpus has {corpus.n_funcs}")
    if into is not None:
        want = dict(val_masks=(nv, np.uint32), role=(n, np.uint8), link_mask=(n, np.uint16), link_def=(n, np.uint32),
                    status=(corpus.n_funcs, np.uint8))
        for name, (cnt, dt) in want.items():
            a = getattr(into, name)
            if len(a) < cnt or a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"seed_corpus: result array {name} must be contiguous {np.dtype(dt).name}[>= {cnt}]")
        res = SeedArrays(**{name: getattr(into, name)[:cnt] for name, (cnt, _) in want.items()})
    else:
        res = SeedArrays(np.zeros(nv, np.uint32), np.zeros(n, np.uint8), np.zeros(n, np.uint16),
                         np.zeros(n, np.uint32), np.zeros(corpus.n_funcs, np.uint8))
    st = TypeSeed(*(a.ctypes.data_as(C.c_void_p) for a in (res.val_masks, res.role, res.link_mask, res.link_def, res.status)))
    hp = None
    if hints is not None:
        keep = [np.ascontiguousarray(x, np.uint32) for x in (hints.off, hints.iid, hints.val)]
        hp = C.byref(TypeHints(*(x.ctypes.data_as(C.c_void_p) for x in keep)))
    engine._check(lib.cl_seed_types(engine._ctx, source, ops.ctypes.data_as(C.c_void_p), len(ops),
                                    mods.ctypes.data_as(C.c_void_p), len(mods), hp, C.byref(st)))
    return res


def _gather_runs(off: np.ndarray, members: np.ndarray) -> np.ndarray:
    """Indices of the CSR runs ``off[f]:off[f+1]`` of the functions ``members``, run after run."""
    off = off.astype(np.int64)
    starts, lens = off[members], (off[1:] - off[:-1])[members]
    total = int(lens.sum())
    if total == 0:
        return np.zeros(0, np.int64)
    return np.repeat(starts - (np.cumsum(lens) - lens), lens) + np.arange(total, dtype=np.int64)


def seed_corpus_sharded(engines, corpus: soa.Corpus, hints: Hints | None = None) -> SeedArrays:
    """``seed_corpus`` spread over several engines (one per GPU): the corpus is partitioned by kernel
    (``sharding.shard``: LPT on instruction records; functions are independent, nothing crosses devices) and the
    arrays come back in the corpus' own order."""
    import threading
    from . import sharding
    engines = list(engines)
    plan = sharding.shard_plan(corpus, len(engines))
    parts = sharding.shard(corpus, len(engines), plan)
    part_hints = [None] * len(engines)
    if hints is not None:
        for k, m in enumerate(plan.members):
            idx = _gather_runs(hints.off, m)
            lens = np.diff(hints.off.astype(np.int64))[m]
            part_hints[k] = Hints(np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32), hints.iid[idx], hints.val[idx])
    outs, errors = [None] * len(engines), []

    def work(k):
        try:
            outs[k] = seed_corpus(engines[k], parts[k], part_hints[k])
        except Exception as e:  # noqa: BLE001 - re-raised on the caller's thread
            errors.append(e)

    if all(e.backend.startswith("cuda") for e in engines):
        threads = [threading.Thread(target=work, args=(k,)) for k in range(len(engines))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    else:                                        # the CPU builds: one at a time
        for k in range(len(engines)):
            work(k)
    if errors:
        raise errors[0]
    n, nv = corpus.n_insts, len(corpus.val_alive)
    res = SeedArrays(np.zeros(nv, np.uint32), np.zeros(n, np.uint8), np.zeros(n, np.uint16),
                     np.zeros(n, np.uint32), np.zeros(corpus.n_funcs, np.uint8))
    rec_off = corpus.blk_off[corpus.func_blk_off]
    for m, o in zip(plan.members, outs):
        rec, val = _gather_runs(rec_off, m), _gather_runs(corpus.val_off, m)
        res.role[rec], res.link_mask[rec], res.link_def[rec] = o.role, o.link_mask, o.link_def
        res.val_masks[val] = o.val_masks
        res.status[m] = o.status
    return res


@dataclass
class TypeSet:
    """Mirror of ``lattice.TypeSet`` (lattice.py:119-145): candidate set plus the conflicted flag."""
    mask: int = TOP
    conflicted: bool = False

    def intersect(self, other: int) -> bool:
        if self.conflicted:
            if other and self.mask != other:
                self.mask = other
                return True
            return False
        new = self.mask & other
        if new == self.mask:
            return False
        self.mask = new
        return True

    def copy(self) -> "TypeSet":
        return TypeSet(self.mask, self.conflicted)


@dataclass
class TypeState:
    """Mirror of ``typerec.TypeState`` (typerec.py:253-268)."""
    seed_mask: dict = field(default_factory=dict)
    def_seed_mask: dict = field(default_factory=dict)
    use_seed_mask: dict = field(default_factory=dict)
    link_exprs: dict = field(default_factory=dict)
    roles: dict = field(default_factory=dict)
    iterations: int = 0


def states_of(corpus: soa.Corpus, res: SeedArrays) -> list:
    """Reshape the arrays into one ``TypeState`` per function (dict insertion orders as the reference's)."""
    out = []
    K_VALUE, K_MEMREF = L.K_VALUE, L.K_MEMREF
    hdr, tag, pay = corpus.hdr, corpus.tag, corpus.pay
    for f in range(corpus.n_funcs):
        st = TypeState()
        v0, v1 = int(corpus.val_off[f]), int(corpus.val_off[f + 1])
        masks = res.val_masks[v0:v1]
        for vid in np.flatnonzero(corpus.val_alive[v0:v1]).tolist():
            m = int(masks[vid])
            st.seed_mask[vid], st.def_seed_mask[vid], st.use_seed_mask[vid] = m & 0xFF, (m >> 8) & 0xFF, (m >> 16) & 0xFF
        i0, i1 = corpus.func_inst_range(f)
        e0, m0 = int(corpus.ext_off[f]), int(corpus.mem_off[f])
        for i in range(i0, i1):
            h = hdr[i]
            st.roles[int(h["iid"])] = ROLES[res.role[i]]
            ld, lm = int(res.link_def[i]), int(res.link_mask[i])
            if ld == NO_VALUE or not lm:
                continue
            nu = int(h["n_uses"])
            u0 = (1 if h["flags"] & L.IF_GUARD else 0) + int(h["n_defs"]) + int(h["n_aux"])
            if h["flags"] & L.IF_EXT:
                base = e0 + int(h["ext"])
                tags, pays = corpus.ext_tag[base + u0:base + u0 + nu], corpus.ext_pay[base + u0:base + u0 + nu]
            else:
                tags, pays = tag[i, u0:u0 + nu], pay[i, u0:u0 + nu]
            uses = []
            for k in range(nu):
                if not (lm >> min(k, 15)) & 1:
                    continue
                kind = int(tags[k]) & 15
                if kind == K_VALUE:
                    uses.append(int(pays[k]))
                elif kind == K_MEMREF:
                    mr = corpus.mem[m0 + int(pays[k])]
                    if int(mr["base_tag"]) & 15 == K_VALUE:
                        uses.append(int(mr["base_pay"]))
            if uses:                                         # typerec.py:336-339
                st.link_exprs.setdefault(ld, []).append(uses)
                for x in uses:
                    st.link_exprs.setdefault(x, []).append([ld])
        out.append(st)
    return out


def seed_types_batch(functions, engine=None, engines=None) -> list:
    """``seed_types`` for many functions in one launch; sets ``fn.meta["type_state"]`` like the reference.
    ``engines=[...]`` (one per GPU) spreads the batch by kernel over several devices."""
    from . import passes
    functions = list(functions)
    for fn in functions:
        phase = sys.modules[type(fn).__module__].Phase          # the Phase enum of the package fn comes from
        fn.require_phase(phase.NORMALIZED, phase.SSA, phase.TYPED)   # typerec.py:290
    corpus = soa.encode(functions)
    if engines is not None:
        res = seed_corpus_sharded(engines, corpus, hints_of(functions))
    else:
        res = seed_corpus(engine or passes.default_engine(), corpus, hints_of(functions))
    states = states_of(corpus, res)
    for k, (fn, st, status) in enumerate(zip(functions, states, res.status.tolist())):
        if status == L.ST_KEY_ERROR:
            raise KeyError(f"{fn.name}: a narrowed value is not in fn.values (typerec.py:301)")
        state_cls, set_cls = _classes_for(fn)
        if state_cls is not TypeState:             # the reference's own objects get the reference's own classes
            st = state_cls(link_exprs=st.link_exprs, roles=st.roles, seed_mask=st.seed_mask,
                           def_seed_mask=st.def_seed_mask, use_seed_mask=st.use_seed_mask)
            states[k] = st
        for name in ("seed_mask", "def_seed_mask", "use_seed_mask"):     # dict order of fn.values (typerec.py:292)
            d = getattr(st, name)
            setattr(st, name, {vid: d[vid] for vid in fn.values})
        for info in fn.values.values():
            info.type_state = set_cls()                                  # typerec.py:296
        fn.meta["type_state"] = st
    return states


def _classes_for(fn):
    """(TypeState, TypeSet) classes of the package ``fn`` comes from: the reference's when it is a reference object."""
    pkg = type(fn).__module__.rsplit(".", 1)[0]
    tr, lat = sys.modules.get(pkg + ".typerec"), sys.modules.get(pkg + ".lattice")
    if pkg != __name__.rsplit(".", 1)[0] and tr is not None and lat is not None and hasattr(tr, "TypeState"):
        return tr.TypeState, lat.TypeSet
    return TypeState, TypeSet


def seed_types(fn, engine=None) -> TypeState:
    """Drop-in for ``typerec.seed_types(fn)`` (typerec.py:288)."""
    return seed_types_batch([fn], engine)[0]
