"""Host-side data contract of the hot path.

A small, dependency-free mirror of the *shapes* the reference passes consume
and produce, so that the SoA encoder/decoder, the pattern plugin API and the
parity tests work on a box where the reference package is absent (the GPU
box).  Field names and rendering follow the reference so that objects of
either library can be encoded (the encoder dispatches on class *names*) and
``dump`` text can be compared byte for byte:

* operands      -> reference ``operands.py:41-255``
* Instruction   -> reference ``ssir.py:42-84``
* terminators   -> reference ``ssir.py:95-167``
* BasicBlock / ValueInfo / LiftedFunction -> ``ssir.py:174-269``
* ``dump``      -> reference ``ssir.py:389-421`` (the golden-test surface)

Nothing in here computes anything: the passes themselves run on the GPU.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

PT_INDEX = 7


class Phase(enum.IntEnum):
    RAW = 0
    CFG_BUILT = 1
    SSA = 2
    NORMALIZED = 3
    TYPED = 4


@dataclass(frozen=True)
class Opcode:
    base: str
    modifiers: tuple = ()

    def has_mod(self, *mods):
        return all(m in self.modifiers for m in mods)

    def without_mod(self, *mods):
        return Opcode(self.base, tuple(m for m in self.modifiers if m not in mods))

    def __str__(self):
        return ".".join((self.base, *self.modifiers))

    @staticmethod
    def parse(token):
        head, *mods = token.split(".")
        return Opcode(head, tuple(mods))


def _decorate(body, *, half=None, reuse=False, absolute=False, bitnot=False,
              negated=False):
    """Shared operand spelling: body[.half][.reuse] wrapped by | | then ~ then -."""
    if half:
        body = f"{body}.{half}"
    if reuse:
        body += ".reuse"
    if absolute:
        body = f"|{body}|"
    if bitnot:
        body = "~" + body
    if negated:
        body = "-" + body
    return body


@dataclass
class SourceLine:
    address: int
    text: str
    control_code: str | None = None
    line_no: int | None = None


@dataclass
class Reg:
    base: int
    width: int = 1
    negated: bool = False
    absolute: bool = False
    bitnot: bool = False
    half: str | None = None
    reuse: bool = False

    def name(self):
        top = self.base + self.width - 1
        return f"R{self.base}" if self.width == 1 else f"R{top}:R{self.base}"

    def __str__(self):
        return _decorate(self.name(), half=self.half, reuse=self.reuse,
                         absolute=self.absolute, bitnot=self.bitnot,
                         negated=self.negated)


@dataclass
class UReg:
    index: int
    width: int = 1
    negated: bool = False
    absolute: bool = False
    bitnot: bool = False

    def name(self):
        top = self.index + self.width - 1
        return f"UR{self.index}" if self.width == 1 else f"UR{top}:UR{self.index}"

    def __str__(self):
        return _decorate(self.name(), absolute=self.absolute,
                         bitnot=self.bitnot, negated=self.negated)


@dataclass
class Pred:
    index: int
    negated: bool = False

    def is_pt(self):
        return self.index == PT_INDEX

    def name(self):
        return "PT" if self.is_pt() else f"P{self.index}"

    def __str__(self):
        return ("!" if self.negated else "") + self.name()


@dataclass
class ZeroReg:
    uniform: bool = False
    negated: bool = False
    bitnot: bool = False

    def __str__(self):
        return _decorate("URZ" if self.uniform else "RZ", bitnot=self.bitnot,
                         negated=self.negated)


@dataclass
class Imm:
    bits: int
    text: str
    is_float: bool = False
    negated: bool = False

    def __str__(self):
        return ("-" if self.negated else "") + self.text


@dataclass
class ConstMem:
    bank: int
    offset: int
    width: int = 1
    half: str | None = None
    negated: bool = False
    absolute: bool = False

    def __str__(self):
        return _decorate(f"c[{self.bank:#x}][{self.offset:#x}]", half=self.half,
                         absolute=self.absolute, negated=self.negated)


@dataclass
class SReg:
    name: str

    def __str__(self):
        return self.name


@dataclass
class MemRef:
    base: object = None
    ureg: object = None
    offset: int = 0

    def __str__(self):
        terms = [str(t) for t in (self.base, self.ureg) if t is not None]
        if self.offset or not terms:
            mag = f"{abs(self.offset):#x}"
            terms.append(mag if self.offset >= 0 else "-" + mag)
        return "[" + "+".join(terms) + "]"


@dataclass
class ValueRef:
    vid: int
    negated: bool = False
    absolute: bool = False
    bitnot: bool = False
    half: str | None = None

    def __str__(self):
        return _decorate(f"%v{self.vid}", half=self.half, absolute=self.absolute,
                         bitnot=self.bitnot, negated=self.negated)


@dataclass
class Instruction:
    iid: int
    opcode: Opcode
    guard: object
    defs: list
    uses: list
    aux_defs: list = field(default_factory=list)
    raw: SourceLine | None = None
    meta: dict = field(default_factory=dict)

    @property
    def address(self):
        return self.raw.address if self.raw else self.meta.get("address")

    def all_defs(self):
        return self.defs + self.aux_defs

    def render(self):
        head = f"@{self.guard} {self.opcode}" if self.guard is not None \
            else str(self.opcode)
        if self.opcode.base == "PHI":
            srcs = zip(self.uses, self.meta.get("phi_blocks", []))
            ops = [str(d) for d in self.defs] + [f"[{u}, {b}]" for u, b in srcs]
        else:
            ops = [str(o) for o in (*self.defs, *self.aux_defs, *self.uses)]
        return f"{head} {', '.join(ops)}" if ops else head

    __str__ = render


# -- terminators ---------------------------------------------------------------

@dataclass
class Br:
    target: int

    def successors(self):
        return [self.target]

    def render(self, fn=None):
        return f"br bb{self.target}"


@dataclass
class CondBr:
    cond: object
    taken: int
    fallthrough: int
    guard: object = None

    def successors(self):
        return [self.taken, self.fallthrough]

    def render(self, fn=None):
        g = "" if self.guard is None else f" guard={self.guard}"
        return f"condbr{g} {self.cond} ? bb{self.taken} : bb{self.fallthrough}"


@dataclass
class Ret:
    def successors(self):
        return []

    def render(self, fn=None):
        return "ret"


@dataclass
class Exit:
    def successors(self):
        return []

    def render(self, fn=None):
        return "exit"


@dataclass
class CondExit:
    cond: object
    fallthrough: int

    def successors(self):
        return [self.fallthrough]

    def render(self, fn=None):
        return f"condexit {self.cond} else bb{self.fallthrough}"


@dataclass
class CallRet:
    target_address: int
    return_address: int
    return_block: int | None = None
    site_address: int | None = None

    def successors(self):
        return [] if self.return_block is None else [self.return_block]

    def render(self, fn=None):
        return f"callret {self.target_address:#x} ret->{self.return_address:#x}"


@dataclass
class BasicBlock:
    bid: int
    start_address: int
    instructions: list = field(default_factory=list)
    terminator: object = None
    preds: list = field(default_factory=list)
    succs: list = field(default_factory=list)
    convergence_meta: str | None = None

    def label(self):
        return f"bb{self.bid}"


@dataclass
class ValueInfo:
    vid: int
    origin: str
    def_iid: int | None
    type_state: object = None
    provenance: object = None
    is_undef: bool = False
    reach: int | None = None
    final_type: str | None = None

    def name(self):
        return f"%v{self.vid}"


@dataclass
class LiftedFunction:
    name: str
    arch: str
    param_base: int
    phase: Phase = Phase.RAW
    raw_instructions: list = field(default_factory=list)
    entry: int | None = None
    blocks: dict = field(default_factory=dict)
    values: dict = field(default_factory=dict)
    diagnostics: list = field(default_factory=list)
    meta: dict = field(default_factory=dict)
    _next_iid: int = 0
    _next_vid: int = 0
    _next_bid: int = 0

    def new_iid(self):
        self._next_iid += 1
        return self._next_iid - 1

    def new_value(self, origin, def_iid, is_undef=False):
        info = ValueInfo(self._next_vid, origin, def_iid, is_undef=is_undef)
        self.values[info.vid] = info
        self._next_vid += 1
        return info

    def new_block(self, start_address):
        blk = BasicBlock(self._next_bid, start_address)
        self.blocks[blk.bid] = blk
        self._next_bid += 1
        return blk

    def make_inst(self, opcode, defs, uses, guard=None, aux=None, raw=None, **meta):
        return Instruction(self.new_iid(), opcode, guard, list(defs), list(uses),
                           list(aux or ()), raw, dict(meta))

    def block_order(self):
        return [self.blocks[b] for b in sorted(self.blocks)]

    def require_phase(self, *phases):
        if self.phase not in phases:
            want = "/".join(p.name for p in phases)
            raise RuntimeError(f"{self.name}: pass requires phase {want}, "
                               f"function is {self.phase.name}")

    def advance_phase(self, new_phase):
        if new_phase < self.phase:
            raise RuntimeError(f"{self.name}: phase may not regress "
                               f"{self.phase.name} -> {new_phase.name}")
        self.phase = new_phase

    def diagnose(self, msg):
        self.diagnostics.append(msg)


def dump(fn) -> str:
    """Text rendering identical to the reference's golden-test surface
    (``ssir.py:389-421``); works on either library's objects."""
    phase = int(fn.phase)
    out = [f"function @{fn.name} [arch={fn.arch} phase={Phase(phase).name.lower()}"
           f" param_base={fn.param_base:#x}]"]
    out += [f"  ; cuda-object {tag}" for tag in fn.meta.get("cuda_objects", [])]
    if phase == Phase.RAW:
        for inst in fn.raw_instructions:
            addr = inst.address
            where = "----" if addr is None else f"{addr:04x}"
            out.append(f"  {where}: {inst.render()}")
        return "\n".join(out) + "\n"
    for blk in fn.block_order():
        preds = ",".join(f"bb{p}" for p in sorted(blk.preds)) or "-"
        conv = f" conv={blk.convergence_meta}" if blk.convergence_meta else ""
        out.append(f"bb{blk.bid} @{blk.start_address:04x}  preds={preds}{conv}")
        out += ["  " + inst.render() for inst in blk.instructions]
        if blk.terminator is not None:
            out.append("  " + blk.terminator.render(fn))
    if phase >= Phase.TYPED:
        out.append("types:")
        for vid in sorted(fn.values):
            info = fn.values[vid]
            if info.final_type is not None:
                out.append(f"  %v{vid}:{info.origin} {info.final_type} "
                           f"{info.provenance.value}")
    return "\n".join(out) + "\n"


# -- conversion from foreign (reference) objects ----------------------------------
_BY_NAME = None


def convert(obj):
    """Deep-copy an object graph of the reference library (``sasslift``) into
    this module's classes, dispatching on class *names* and dataclass fields.
    Used to build travelling fixtures: the GPU box has no reference package."""
    import dataclasses
    global _BY_NAME
    if _BY_NAME is None:
        _BY_NAME = {n: c for n, c in globals().items()
                    if isinstance(c, type) and dataclasses.is_dataclass(c)}
    if isinstance(obj, enum.Enum):
        if type(obj).__name__ == "Phase":
            return Phase(int(obj))
        return _EnumValue(obj.value)
    if dataclasses.is_dataclass(obj) and not isinstance(obj, type):
        cls = _BY_NAME.get(type(obj).__name__)
        if cls is None:
            return None                       # type lattice state etc.: not our contract
        own = {f.name for f in dataclasses.fields(cls)}
        kw = {f.name: convert(getattr(obj, f.name))
              for f in dataclasses.fields(obj) if f.name in own}
        return cls(**kw)
    if isinstance(obj, dict):
        return {convert(k): convert(v) for k, v in obj.items()}
    if isinstance(obj, list):
        return [convert(v) for v in obj]
    if isinstance(obj, tuple):
        return tuple(convert(v) for v in obj)
    if isinstance(obj, set):
        return {convert(v) for v in obj}
    return obj


@dataclass(frozen=True)
class _EnumValue:
    value: object
