"""Struct-of-arrays instruction encoder / decoder (subsystem 1 of the north
star: "an SoA instruction encoder and the H2D layout").

``encode`` walks ``LiftedFunction`` objects -- the reference's
(``sasslift.ssir``) or this package's (``ir``); dispatch is by class name --
once and packs them into the planes described in ``include/culifter.h``.
``apply`` writes a processed corpus back into the same objects, so the GPU
passes keep the reference's mutate-in-place contract.

The encoding is lossless for everything ``dump`` prints and everything the
passes read: operand kinds and syntactic flags (``operands.py:65-255``), the
ordered modifier tuple (``Opcode``, ``operands.py:41``), def/aux/use arity,
the value table (``ssir.py:189-235``) and terminator value uses
(``ssir.py:378-382``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ir as own_ir
from .layout import (
    ARCHS, BLK, CM_OFFSET_BITS, EVENT, FUNC, HDR, IF_EXT, IF_GUARD, IF_OBJ_SHIFT,
    IF_OBJUSE_SHIFT, IF_SYNTH, IMM, K_CONSTMEM, K_IMM, K_MEMREF, K_NONE, K_PRED,
    K_REG, K_RZ, K_SREG, K_UREG, K_URZ, K_VALUE, MEMREF, ORG_BITS, ORG_F, ORG_PAIR,
    SLOTS, T_ABS, T_HALF_SHIFT, T_IMM_FLOAT, T_IMM_HEXTEXT, T_NEG, T_NOT, T_REUSE,
    T_WIDTH_SHIFT, TABLES,
)

_HALF = {None: 0, "H0": 1, "H1": 2}
_HALF_INV = {0: None, 1: "H0", 2: "H1"}
M64 = (1 << 64) - 1


class EncodeError(ValueError):
    """An operand does not fit the fixed-width layout (loud, never silent)."""


@dataclass
class Corpus:
    """Dense CSR arrays of ``cl_corpus`` plus the host-only sidecar."""

    func: np.ndarray
    func_blk_off: np.ndarray
    ext_off: np.ndarray
    mem_off: np.ndarray
    imm_off: np.ndarray
    val_off: np.ndarray
    blk: np.ndarray
    blk_off: np.ndarray
    hdr: np.ndarray
    tag: np.ndarray          # [N, 8] u16
    pay: np.ndarray          # [N, 8] u32
    ext_tag: np.ndarray
    ext_pay: np.ndarray
    mem: np.ndarray
    imm: np.ndarray
    val_alive: np.ndarray
    val_def_iid: np.ndarray
    val_origin: np.ndarray
    events: np.ndarray = field(default_factory=lambda: np.zeros(0, EVENT))
    functions: list = field(default_factory=list)   # host objects, may be empty
    raw: bool = False

    ARRAYS = ("func", "func_blk_off", "ext_off", "mem_off", "imm_off", "val_off",
              "blk", "blk_off", "hdr", "tag", "pay", "ext_tag", "ext_pay", "mem",
              "imm", "val_alive", "val_def_iid", "val_origin")

    @property
    def n_funcs(self):
        return len(self.func)

    @property
    def n_blocks(self):
        return len(self.blk)

    @property
    def n_insts(self):
        return len(self.hdr)

    def func_inst_range(self, f):
        b0, b1 = self.func_blk_off[f], self.func_blk_off[f + 1]
        return int(self.blk_off[b0]), int(self.blk_off[b1])

    def nbytes(self):
        return sum(getattr(self, a).nbytes for a in self.ARRAYS)

    def equal(self, other, check_values=True):
        """Bit-exact comparison of two corpora; returns a list of differences."""
        diffs = []
        for a in self.ARRAYS:
            if not check_values and a.startswith("val_"):
                continue
            x, y = getattr(self, a), getattr(other, a)
            if x.shape != y.shape:
                diffs.append(f"{a}: shape {x.shape} != {y.shape}")
            elif not np.array_equal(x, y):
                bad = np.flatnonzero((x != y).reshape(len(x), -1).any(axis=1)
                                     if x.ndim > 1 or x.dtype.names is None
                                     else x != y)
                diffs.append(f"{a}: {len(bad)} rows differ, first {bad[:5].tolist()}")
        return diffs

    def slice_funcs(self, f0: int, f1: int) -> "Corpus":
        """Functions [f0, f1) as a corpus of their own.  Every index inside a
        function is function-local, so the big arrays are plain views and only the
        CSR offset arrays are rebased (copies of f1 - f0 + 1 words each)."""
        b0, b1 = int(self.func_blk_off[f0]), int(self.func_blk_off[f1])
        i0, i1 = int(self.blk_off[b0]), int(self.blk_off[b1])
        e0, e1 = int(self.ext_off[f0]), int(self.ext_off[f1])
        m0, m1 = int(self.mem_off[f0]), int(self.mem_off[f1])
        q0, q1 = int(self.imm_off[f0]), int(self.imm_off[f1])
        v0, v1 = int(self.val_off[f0]), int(self.val_off[f1])
        return Corpus(
            func=self.func[f0:f1], func_blk_off=self.func_blk_off[f0:f1 + 1] - np.uint32(b0),
            ext_off=self.ext_off[f0:f1 + 1] - np.uint32(e0), mem_off=self.mem_off[f0:f1 + 1] - np.uint32(m0),
            imm_off=self.imm_off[f0:f1 + 1] - np.uint32(q0), val_off=self.val_off[f0:f1 + 1] - np.uint32(v0),
            blk=self.blk[b0:b1], blk_off=self.blk_off[b0:b1 + 1] - np.uint32(i0),
            hdr=self.hdr[i0:i1], tag=self.tag[i0:i1], pay=self.pay[i0:i1],
            ext_tag=self.ext_tag[e0:e1], ext_pay=self.ext_pay[e0:e1], mem=self.mem[m0:m1], imm=self.imm[q0:q1],
            val_alive=self.val_alive[v0:v1], val_def_iid=self.val_def_iid[v0:v1], val_origin=self.val_origin[v0:v1],
            functions=self.functions[f0:f1] if self.functions else [], raw=self.raw)

    def split(self, n_chunks: int):
        """Contiguous function ranges of about equal record count: [(f0, f1), ...]."""
        F = self.n_funcs
        if F == 0:
            return []
        first = self.blk_off[self.func_blk_off[:-1]].astype(np.int64)       # first record of every function
        cuts = np.searchsorted(first, np.arange(1, n_chunks) * (self.n_insts / n_chunks))
        edges = np.unique(np.concatenate(([0], cuts, [F])))
        return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]

    def save(self, path):
        np.savez_compressed(path, raw=np.array(self.raw),
                            events=self.events,
                            **{a: getattr(self, a) for a in self.ARRAYS})

    @staticmethod
    def load(path):
        z = np.load(path)
        c = Corpus(**{a: z[a] for a in Corpus.ARRAYS})
        c.events = z["events"]
        c.raw = bool(z["raw"])
        return c


# ------------------------------------------------------------------- encoding
class _FnEnc:
    """Per-function scratch lists while encoding."""

    def __init__(self):
        self.imm_key = {}
        self.imm = []
        self.mem = []
        self.ext_tag = []
        self.ext_pay = []


def _flag_bits(op, *, absolute=True, bitnot=True):
    t = 0
    if getattr(op, "negated", False):
        t |= T_NEG
    if bitnot and getattr(op, "bitnot", False):
        t |= T_NOT
    if absolute and getattr(op, "absolute", False):
        t |= T_ABS
    return t


def _half_bits(op):
    try:
        return _HALF[getattr(op, "half", None)] << T_HALF_SHIFT
    except KeyError:
        raise EncodeError(f"unsupported half selector {op.half!r}") from None


def encode_operand(op, fe: _FnEnc):
    """-> (tag, payload) of one operand (``cl_kind`` in culifter.h)."""
    kind = type(op).__name__
    if kind == "ValueRef":
        return K_VALUE | _flag_bits(op) | _half_bits(op), op.vid
    if kind == "Imm":
        bits = op.bits & M64
        text = TABLES.string(op.text)
        key = (bits, text)
        idx = fe.imm_key.get(key)
        if idx is None:
            idx = fe.imm_key[key] = len(fe.imm)
            fe.imm.append((bits, text))
        tag = K_IMM | (T_NEG if op.negated else 0) | (T_IMM_FLOAT if op.is_float else 0)
        return tag, idx
    if kind == "ZeroReg":
        return (K_URZ if op.uniform else K_RZ) | _flag_bits(op, absolute=False), 0
    if kind == "Pred":
        return K_PRED | (T_NEG if op.negated else 0), op.index
    if kind == "Reg":
        if not (0 <= op.base < 65536 and 0 < op.width < 65536):
            raise EncodeError(f"register out of range: {op}")
        tag = K_REG | _flag_bits(op) | _half_bits(op) | (T_REUSE if op.reuse else 0)
        return tag, op.base | op.width << 16
    if kind == "UReg":
        if not (0 <= op.index < 65536 and 0 < op.width < 65536):
            raise EncodeError(f"uniform register out of range: {op}")
        return K_UREG | _flag_bits(op), op.index | op.width << 16
    if kind == "ConstMem":
        if not (0 <= op.offset < 1 << CM_OFFSET_BITS and 0 <= op.bank < 4096
                and 0 < op.width < 8):
            raise EncodeError(f"constant-memory operand out of range: {op}")
        tag = K_CONSTMEM | _flag_bits(op, bitnot=False) | _half_bits(op) \
            | op.width << T_WIDTH_SHIFT
        return tag, op.offset | op.bank << CM_OFFSET_BITS
    if kind == "SReg":
        return K_SREG, TABLES.string(op.name)
    if kind == "MemRef":
        bt, bp = (K_NONE, 0) if op.base is None else encode_operand(op.base, fe)
        ut, up = (K_NONE, 0) if op.ureg is None else encode_operand(op.ureg, fe)
        off = int(op.offset)
        if not -(1 << 63) <= off < 1 << 63:
            raise EncodeError(f"address offset out of range: {op}")
        fe.mem.append((bt, ut, bp, up, off >> 32, off & 0xFFFFFFFF))
        return K_MEMREF, len(fe.mem) - 1
    raise EncodeError(f"cannot encode operand of type {kind}")


def _cuda_object_flags(inst):
    obj = inst.meta.get("cuda_object") if inst.meta else None
    if not obj:
        return 0
    kind = {"block_sync": 1, "warp_group": 2, "collective": 3}[obj[0]]
    return kind << IF_OBJ_SHIFT | 7 << IF_OBJUSE_SHIFT


def _load_codec():
    """The C encoder (csrc/codec.c, built in-tree by ``__graft_entry__.build``)."""
    try:
        from . import _codec
    except ImportError as e:
        raise ImportError(
            "paper_2604_27486_b200/_codec*.so is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (gcc, CPython headers)") from e
    return _codec


def encode(functions, raw: bool = False) -> Corpus:
    """Pack functions (SSA/NORMALIZED phase, or RAW when ``raw``) into a corpus.

    SSA-phase functions go through the C encoder (``csrc/codec.c``: the same
    walk as :func:`encode_py`, about ten times faster; ``tests/test_codec.py``
    holds the two byte-equal on every fixture).  RAW-phase corpora (the two
    front-half passes) keep the Python walk."""
    functions = list(functions)
    if raw:
        return encode_py(functions, raw=True)
    z = _load_codec().encode(functions, TABLES, ARCHS, EncodeError)

    def arr(name, dt, shape=None):
        a = np.frombuffer(z[name], dtype=dt).copy()
        return a.reshape(shape) if shape else a
    cnt = arr("blk_cnt", np.uint32)
    blk_off = np.zeros(len(cnt) + 1, np.uint32)
    np.cumsum(cnt, out=blk_off[1:])
    val_off = arr("val_off", np.uint32)
    return Corpus(
        func=arr("func", FUNC), func_blk_off=arr("func_blk_off", np.uint32), ext_off=arr("ext_off", np.uint32),
        mem_off=arr("mem_off", np.uint32), imm_off=arr("imm_off", np.uint32), val_off=val_off,
        blk=arr("blk", BLK), blk_off=blk_off, hdr=arr("hdr", HDR),
        tag=arr("tag", np.uint16, (-1, SLOTS)), pay=arr("pay", np.uint32, (-1, SLOTS)),
        ext_tag=arr("ext_tag", np.uint16), ext_pay=arr("ext_pay", np.uint32),
        mem=arr("mem", MEMREF), imm=arr("imm", IMM),
        val_alive=arr("val_alive", np.uint8), val_def_iid=arr("val_def_iid", np.int32),
        val_origin=np.zeros(int(val_off[-1]), np.uint32), functions=functions, raw=False)


def encode_py(functions, raw: bool = False) -> Corpus:
    """The encoder as a plain Python walk: reference implementation of :func:`encode`, and the RAW-phase path."""
    functions = list(functions)
    F = len(functions)
    func = np.zeros(F, FUNC)
    func_blk_off = np.zeros(F + 1, np.uint32)
    ext_off = np.zeros(F + 1, np.uint32)
    mem_off = np.zeros(F + 1, np.uint32)
    imm_off = np.zeros(F + 1, np.uint32)
    val_off = np.zeros(F + 1, np.uint32)
    blks, blk_cnt = [], []
    hdrs, tags, pays = [], [], []
    ext_tag, ext_pay, mems, imms = [], [], [], []
    alive, def_iid = [], []

    for f, fn in enumerate(functions):
        fe = _FnEnc()
        if raw:
            blocks = [(0, fn.raw_instructions, None)]
        else:
            blocks = [(b.bid, b.instructions, b.terminator) for b in fn.block_order()]
        donor = {}
        if raw:
            for inst in fn.raw_instructions:
                if inst.raw is not None and not (inst.meta and inst.meta.get("synthetic")):
                    donor.setdefault(id(inst.raw), inst.iid)
        for bid, insts, term in blocks:
            tt, tp = [K_NONE, K_NONE], [0, 0]
            for k, attr in enumerate(("cond", "guard")):
                ref = getattr(term, attr, None) if term is not None else None
                if ref is not None and not (attr == "guard" and
                                            type(term).__name__ != "CondBr"):
                    tt[k], tp[k] = encode_operand(ref, fe)
            blks.append((bid, tt, tp))
            blk_cnt.append(len(insts))
            for inst in insts:
                slots = []
                flags = _cuda_object_flags(inst)
                if inst.guard is not None:
                    flags |= IF_GUARD
                    slots.append(encode_operand(inst.guard, fe))
                ext = 0
                if inst.meta and inst.meta.get("synthetic"):
                    flags |= IF_SYNTH
                    ext = donor.get(id(inst.raw), inst.iid)
                for group in (inst.defs, inst.aux_defs, inst.uses):
                    if len(group) > 255:
                        raise EncodeError(f"{fn.name}: inst {inst.iid} has "
                                          f"{len(group)} operands in one group")
                    slots.extend(encode_operand(o, fe) for o in group)
                if len(slots) > SLOTS:
                    flags |= IF_EXT
                    ext = len(fe.ext_tag)
                    fe.ext_tag.extend(s[0] for s in slots)
                    fe.ext_pay.extend(s[1] for s in slots)
                    slots = []
                slots += [(K_NONE, 0)] * (SLOTS - len(slots))
                hdrs.append((inst.iid, TABLES.opcode(inst.opcode.base),
                             TABLES.modset(inst.opcode.modifiers), len(inst.defs),
                             len(inst.aux_defs), len(inst.uses), flags, ext))
                tags.append([s[0] for s in slots])
                pays.append([s[1] for s in slots])
        nv = fn._next_vid
        fa = np.zeros(nv, np.uint8)
        fd = np.full(nv, -1, np.int32)
        for vid, info in fn.values.items():
            fa[vid] = 1
            if info.def_iid is not None:
                fd[vid] = info.def_iid
        alive.append(fa)
        def_iid.append(fd)
        func[f] = (nv, fn._next_iid, fn.meta.get("next_temp_reg", 1000),
                   ARCHS.index(fn.arch), 0, 0)
        func_blk_off[f + 1] = len(blks)
        ext_tag += fe.ext_tag
        ext_pay += fe.ext_pay
        mems += fe.mem
        imms += fe.imm
        ext_off[f + 1] = len(ext_tag)
        mem_off[f + 1] = len(mems)
        imm_off[f + 1] = len(imms)
        val_off[f + 1] = val_off[f] + nv

    blk = np.zeros(len(blks), BLK)
    for i, (bid, tt, tp) in enumerate(blks):
        blk[i] = (bid, tt, tp)
    blk_off = np.zeros(len(blks) + 1, np.uint32)
    np.cumsum(blk_cnt, out=blk_off[1:])
    n = len(hdrs)
    return Corpus(
        func=func, func_blk_off=func_blk_off, ext_off=ext_off, mem_off=mem_off,
        imm_off=imm_off, val_off=val_off, blk=blk, blk_off=blk_off,
        hdr=np.array(hdrs, HDR) if n else np.zeros(0, HDR),
        tag=np.array(tags, np.uint16).reshape(n, SLOTS),
        pay=np.array(pays, np.uint32).reshape(n, SLOTS),
        ext_tag=np.array(ext_tag, np.uint16), ext_pay=np.array(ext_pay, np.uint32),
        mem=np.array(mems, MEMREF) if mems else np.zeros(0, MEMREF),
        imm=np.array(imms, IMM) if imms else np.zeros(0, IMM),
        val_alive=np.concatenate(alive) if alive else np.zeros(0, np.uint8),
        val_def_iid=np.concatenate(def_iid) if def_iid else np.zeros(0, np.int32),
        val_origin=np.zeros(int(val_off[-1]), np.uint32),
        functions=functions, raw=raw)


# ------------------------------------------------------------------- decoding
class _Lists:
    """The planes of a corpus as plain Python lists: element access on numpy
    structured arrays costs more than building the operand objects."""

    def __init__(self, c: Corpus):
        H = c.hdr
        self.iid, self.op, self.modset = H["iid"].tolist(), H["op"].tolist(), H["modset"].tolist()
        self.nd, self.na, self.nu = H["n_defs"].tolist(), H["n_aux"].tolist(), H["n_uses"].tolist()
        self.flags, self.ext = H["flags"].tolist(), H["ext"].tolist()
        self.tag, self.pay = c.tag.tolist(), c.pay.tolist()
        self.ext_tag, self.ext_pay = c.ext_tag.tolist(), c.ext_pay.tolist()
        self.imm = list(zip(c.imm["bits"].tolist(), c.imm["text"].tolist()))
        M = c.mem
        self.mem = list(zip(M["base_tag"].tolist(), M["base_pay"].tolist(), M["ureg_tag"].tolist(),
                            M["ureg_pay"].tolist(), M["off_hi"].tolist(), M["off_lo"].tolist()))


class _FnDec:
    def __init__(self, c: Corpus, f: int, ns, lists: _Lists = None):
        L = lists or _Lists(c)
        self.ns = ns
        self.L = L
        self.q0, self.m0, self.e0 = int(c.imm_off[f]), int(c.mem_off[f]), int(c.ext_off[f])


def decode_operand(tag, pay, fd: _FnDec):
    ns = fd.ns
    kind = tag & 15
    if kind == K_VALUE:
        return ns.ValueRef(pay, bool(tag & T_NEG), bool(tag & T_ABS), bool(tag & T_NOT),
                           _HALF_INV[(tag >> T_HALF_SHIFT) & 3])
    neg = bool(tag & T_NEG)
    if kind == K_IMM:
        bits, text = fd.L.imm[fd.q0 + pay]
        s = hex(text) if tag & T_IMM_HEXTEXT else TABLES.strings[text]
        return ns.Imm(bits, s, bool(tag & T_IMM_FLOAT), neg)
    bnot, absolute = bool(tag & T_NOT), bool(tag & T_ABS)
    if kind in (K_RZ, K_URZ):
        return ns.ZeroReg(kind == K_URZ, neg, bnot)
    if kind == K_PRED:
        return ns.Pred(pay, neg)
    half = _HALF_INV[(tag >> T_HALF_SHIFT) & 3]
    if kind == K_REG:
        return ns.Reg(pay & 0xFFFF, pay >> 16, neg, absolute, bnot, half,
                      bool(tag & T_REUSE))
    if kind == K_UREG:
        return ns.UReg(pay & 0xFFFF, pay >> 16, neg, absolute, bnot)
    if kind == K_CONSTMEM:
        return ns.ConstMem(pay >> CM_OFFSET_BITS, pay & ((1 << CM_OFFSET_BITS) - 1),
                           (tag >> T_WIDTH_SHIFT) & 7, half, neg, absolute)
    if kind == K_SREG:
        return ns.SReg(TABLES.strings[pay])
    if kind == K_MEMREF:
        bt, bp, ut, up, hi, lo = fd.L.mem[fd.m0 + pay]
        base = None if bt & 15 == K_NONE else decode_operand(bt, bp, fd)
        ureg = None if ut & 15 == K_NONE else decode_operand(ut, up, fd)
        return ns.MemRef(base, ureg, hi << 32 | lo)
    raise ValueError(f"bad operand tag {tag:#x}")


def decode_slots(c: Corpus, i: int, fd: _FnDec):
    """-> (guard, defs, aux, uses) operand objects of record ``i``."""
    L = fd.L
    flags = L.flags[i]
    nd, na, nu = L.nd[i], L.na[i], L.nu[i]
    g = 1 if flags & IF_GUARD else 0
    total = g + nd + na + nu
    if flags & IF_EXT:
        e = fd.e0 + L.ext[i]
        tg, py = L.ext_tag[e:e + total], L.ext_pay[e:e + total]
    else:
        tg, py = L.tag[i], L.pay[i]
    ops = [decode_operand(tg[k], py[k], fd) for k in range(total)]
    guard = ops[0] if g else None
    return guard, ops[g:g + nd], ops[g + nd:g + nd + na], ops[g + nd + na:]


def _origin_string(fn, code: int, new_origin: dict) -> str:
    code = int(code)
    if code == ORG_PAIR:
        return "pair"
    kind, vid = code >> 28, code & ((1 << 28) - 1)
    base = new_origin[vid] if vid in new_origin else fn.values[vid].origin
    return base + (".bits" if kind == ORG_BITS >> 28 else ".f")


_OBJ_KINDS = {1: "block_sync", 2: "warp_group", 3: "collective"}


def unchanged_records(c_in: Corpus, c_out: Corpus) -> np.ndarray:
    """bool per record of ``c_out``: the stage left it exactly as ``c_in`` had it (same function, same iid, same 64
    bytes, and the MemRef entries / immediates it points at untouched), so the host object it was encoded from still
    says the same and ``apply`` need not rebuild its operands.  Vectorised over the whole corpus."""
    n_out = c_out.n_insts
    if c_in.n_funcs != c_out.n_funcs or c_in.raw != c_out.raw or n_out == 0 or c_in.n_insts == 0:
        return np.zeros(n_out, bool)

    def func_of(c):
        first = c.blk_off[c.func_blk_off].astype(np.int64)                  # first record of every function, then the end
        return np.repeat(np.arange(c.n_funcs, dtype=np.int64), np.diff(first))
    f_in, f_out = func_of(c_in), func_of(c_out)
    k_in = f_in << 32 | c_in.hdr["iid"].astype(np.int64)
    k_out = f_out << 32 | c_out.hdr["iid"].astype(np.int64)
    order = np.argsort(k_in, kind="stable")
    pos = np.searchsorted(k_in[order], k_out)
    pos[pos >= len(order)] = 0
    src = order[pos]
    same = k_in[src] == k_out
    row = lambda a: np.ascontiguousarray(a).view(np.uint8).reshape(len(a), a.dtype.itemsize)          # noqa: E731
    same &= (row(c_in.hdr)[src] == row(c_out.hdr)).all(axis=1)
    same &= (c_in.tag[src] == c_out.tag).all(axis=1) & (c_in.pay[src] == c_out.pay).all(axis=1)
    same &= (c_out.hdr["flags"] & IF_EXT) == 0                                          # overflow slots: always decoded
    # what the operands point at: MemRef entries (simplify_packs redirects their bases) and immediates
    kinds = c_out.tag & 15
    if len(c_in.mem) == len(c_out.mem) and np.array_equal(c_in.mem_off, c_out.mem_off):
        mem_same = (row(c_in.mem) == row(c_out.mem)).all(axis=1)
        is_mem = kinds == K_MEMREF
        if is_mem.any():
            r, k = np.nonzero(is_mem)
            bad = ~mem_same[c_out.mem_off[f_out[r]].astype(np.int64) + c_out.pay[r, k]]
            same[r[bad]] = False
    else:
        same &= ~(kinds == K_MEMREF).any(axis=1)
    is_imm = kinds == K_IMM
    if is_imm.any():
        r, k = np.nonzero(is_imm)
        gi = c_in.imm_off[f_out[r]].astype(np.int64) + c_out.pay[r, k]
        go = c_out.imm_off[f_out[r]].astype(np.int64) + c_out.pay[r, k]
        ok = (c_out.pay[r, k] < (c_in.imm_off[f_out[r] + 1] - c_in.imm_off[f_out[r]]))      # an immediate the input had
        ok[ok] &= (row(c_in.imm)[gi[ok]] == row(c_out.imm)[go[ok]]).all(axis=1)
        same[r[~ok]] = False
    return same


def apply(c_out: Corpus, functions=None, ns=None, patterns=None, tagged=True, c_in: Corpus = None) -> None:
    """Write a processed corpus back into its ``LiftedFunction`` objects in place.

    Surviving instructions keep their identity (``raw``, ``meta``); operands and
    opcode are rebuilt from the records.  New instructions get fresh objects.
    Diagnostics, ``pattern_boundaries`` and ``cuda_objects`` are appended from the
    event list / record flags exactly where the reference appends them
    (``patterns.py:684,842,906-915``).
    """
    import gc
    gc_was_on = gc.isenabled()
    gc.disable()           # millions of live operand objects: every generation-2 pass of the collector walks them all
    try:
        _apply(c_out, functions, ns, patterns, tagged, c_in)
    finally:
        if gc_was_on:
            gc.enable()


def _apply(c_out, functions, ns, patterns, tagged, c_in):
    functions = c_out.functions if functions is None else list(functions)
    ev_by_func = {}
    for ev in c_out.events:          # cl_download returns them in append order
        ev_by_func.setdefault(int(ev["func"]), []).append(ev)
    L = _Lists(c_out)
    keep_as_is = unchanged_records(c_in, c_out).tolist() if c_in is not None else None
    op_name, modset_tuple = TABLES.op_name, TABLES.modset_tuple
    opcode_cache = {}
    for f, fn in enumerate(functions):
        fns = ns or _namespace_of(fn)
        fd = _FnDec(c_out, f, fns, L)
        if c_out.raw:
            old = {inst.iid: inst for inst in fn.raw_instructions}
            containers = [None]
        else:
            old = {inst.iid: inst for b in fn.blocks.values() for inst in b.instructions}
            containers = fn.block_order()
        b0 = int(c_out.func_blk_off[f])
        tags = []
        for k, blk in enumerate(containers):
            lo, hi = int(c_out.blk_off[b0 + k]), int(c_out.blk_off[b0 + k + 1])
            out = []
            for i in range(lo, hi):
                if keep_as_is is not None and keep_as_is[i]:
                    inst = old.get(L.iid[i])
                    # untouched by the stage: the object it was encoded from is already what the record says
                    if inst is not None and not ((L.flags[i] >> IF_OBJ_SHIFT) & 3 and tagged):
                        out.append(inst)
                        continue
                guard, defs, aux, uses = decode_slots(c_out, i, fd)
                okey = (fns.Opcode, L.op[i], L.modset[i])          # Opcode is frozen: one object per (class, op, modifiers)
                opcode = opcode_cache.get(okey)
                if opcode is None:
                    opcode = opcode_cache[okey] = fns.Opcode(op_name[L.op[i]], modset_tuple[L.modset[i]])
                iid = L.iid[i]
                inst = old.get(iid)
                if inst is None:
                    inst = fns.Instruction(iid, opcode, guard, defs, uses, aux)
                else:
                    if inst.opcode != opcode:
                        inst.opcode = opcode
                    inst.guard, inst.defs, inst.aux_defs, inst.uses = guard, defs, aux, uses
                flags = L.flags[i]
                if flags & IF_SYNTH and "synthetic" not in inst.meta:
                    inst.meta["synthetic"] = "x4-scale" if opcode.base == "SHL" \
                        else "sr-substitute"
                    if inst.raw is None and not flags & IF_EXT:
                        donor = old.get(L.ext[i])
                        inst.raw = donor.raw if donor is not None else None
                obj = (flags >> IF_OBJ_SHIFT) & 3
                if obj and tagged:
                    use = (flags >> IF_OBJUSE_SHIFT) & 7
                    if obj == 3:
                        val = str(opcode)
                    else:
                        val = uses[use].bits if use != 7 else 0
                    inst.meta["cuda_object"] = (_OBJ_KINDS[obj], val)
                    tags.append((_OBJ_KINDS[obj], blk.bid, val))
                out.append(inst)
            if c_out.raw:
                fn.raw_instructions = out
            else:
                blk.instructions = out
                term = blk.terminator
                rec = c_out.blk[b0 + k]
                for j, attr in enumerate(("cond", "guard")):
                    if int(rec["term_tag"][j]) & 15 != K_NONE:
                        setattr(term, attr, decode_operand(int(rec["term_tag"][j]),
                                                           int(rec["term_pay"][j]), fd))
        # value table
        fr = c_out.func[f]
        v0 = int(c_out.val_off[f])
        nv_new = int(fr["next_vid"])
        alive = c_out.val_alive[v0:v0 + nv_new].tolist()
        defi = c_out.val_def_iid[v0:v0 + nv_new].tolist()
        orig = c_out.val_origin[v0:v0 + nv_new].tolist()
        new_origin = {}
        values, nv_old = fn.values, fn._next_vid
        for vid in range(nv_new):
            info = values.get(vid)
            if vid >= nv_old:
                new_origin[vid] = _origin_string(fn, orig[vid], new_origin)
            if not alive[vid]:
                if info is not None:
                    del values[vid]
                continue
            d = defi[vid]
            if info is None:
                if vid < nv_old:
                    raise ValueError(f"{fn.name}: %v{vid} resurrected by decode")
                values[vid] = fns.ValueInfo(vid, new_origin[vid], None if d < 0 else d)
            else:
                info.def_iid = None if d < 0 else d
        fn._next_vid = nv_new
        fn._next_iid = int(fr["next_iid"])
        if c_out.raw or "next_temp_reg" in fn.meta or int(fr["next_temp_reg"]) != 1000:
            fn.meta["next_temp_reg"] = int(fr["next_temp_reg"])
        # side outputs
        for ev in ev_by_func.get(f, ()):
            kind = int(ev["kind"])
            if kind == 1:
                name = patterns[int(ev["a"])].name if patterns else f"#{int(ev['a'])}"
                fn.diagnose(f"bb{int(ev['b'])}: pattern {name} matched but "
                            f"rewrite refused (escape or unsupported operands)")
            elif kind == 2:
                fn.meta.setdefault("pattern_boundaries", []).append({
                    "value": int(ev["a"]), "category": "Fast math chains",
                    "inst": int(ev["b"]), "source": "pattern-normalized"})
        if tagged:
            fn.meta.setdefault("cuda_objects", []).extend(tags)


def _namespace_of(fn):
    """Operand/instruction classes matching the library ``fn`` comes from."""
    mod = type(fn).__module__
    if mod == own_ir.__name__:
        return own_ir
    import importlib
    import types
    pkg = mod.rsplit(".", 1)[0]
    ops = importlib.import_module(pkg + ".operands")
    ssir = importlib.import_module(pkg + ".ssir")
    ns = types.SimpleNamespace()
    for name in ("Reg", "UReg", "Pred", "ZeroReg", "Imm", "ConstMem", "SReg", "MemRef",
                 "ValueRef", "Opcode"):
        setattr(ns, name, getattr(ops, name))
    for name in ("Instruction", "ValueInfo"):
        setattr(ns, name, getattr(ssir, name))
    return ns
