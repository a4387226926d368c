"""numpy views of the structs in ``include/culifter.h`` plus the interned
side tables (opcode ids, modifier tuples, strings).

The opcode table is parsed from ``include/culifter_ops.h`` so that the C
header stays the single source of truth.
"""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
INCLUDE = ROOT / "include"

# ---------------------------------------------------------------- struct dtypes
HDR = np.dtype([("iid", "<u4"), ("op", "<u2"), ("modset", "<u2"),
                ("n_defs", "u1"), ("n_aux", "u1"), ("n_uses", "u1"),
                ("flags", "u1"), ("ext", "<u4")])
IMM = np.dtype([("bits", "<u8"), ("text", "<u8")])
MEMREF = np.dtype([("base_tag", "<u2"), ("ureg_tag", "<u2"), ("base_pay", "<u4"),
                   ("ureg_pay", "<u4"), ("off_hi", "<i4"), ("off_lo", "<u4")])
BLK = np.dtype([("bid", "<u4"), ("term_tag", "<u2", (2,)), ("term_pay", "<u4", (2,))])
FUNC = np.dtype([("next_vid", "<u4"), ("next_iid", "<u4"), ("next_temp_reg", "<u4"),
                 ("arch", "u1"), ("status", "u1"), ("reserved", "<u2")])
MODSET = np.dtype([("mask", "<u8"), ("first", "u1", (4,)), ("minus_wide", "<u2"),
                   ("minus_x4", "<u2")])
EVENT = np.dtype([("func", "<u4"), ("seq", "<u4"), ("kind", "<u4"), ("idx", "<u4"),
                  ("a", "<u4"), ("b", "<u4"), ("c", "<u4"), ("d", "<u4")])
assert HDR.itemsize == 16 and IMM.itemsize == 16 and MEMREF.itemsize == 20
assert BLK.itemsize == 16 and FUNC.itemsize == 16 and MODSET.itemsize == 16
assert EVENT.itemsize == 32

SLOTS = 8

# ------------------------------------------------------------------- tag bits
K_NONE, K_VALUE, K_IMM, K_RZ, K_URZ, K_PRED, K_REG, K_UREG, K_CONSTMEM, K_SREG, \
    K_MEMREF = range(11)
T_NEG, T_NOT, T_ABS = 1 << 4, 1 << 5, 1 << 6
T_HALF_SHIFT, T_REUSE, T_WIDTH_SHIFT = 7, 1 << 9, 10
T_IMM_FLOAT, T_IMM_HEXTEXT = T_NOT, T_ABS
CM_OFFSET_BITS = 20

IF_EXT, IF_GUARD, IF_SYNTH = 1, 2, 4
IF_OBJ_SHIFT, IF_OBJUSE_SHIFT = 3, 5

ARCHS = ("sm52", "sm75", "sm90", "sm100", "sm120")

ST_OK, ST_CAPACITY, ST_ATTRIBUTE_ERROR, ST_ASSERTION_ERROR, ST_KEY_ERROR, \
    ST_UNSUPPORTED = range(6)
ST_INDEX_ERROR = 6

EV_REFUSED, EV_BOUNDARY, EV_MATCH = 1, 2, 3

ORG_HOST, ORG_PAIR = 0, 1
ORG_BITS, ORG_F = 2 << 28, 3 << 28

PASS_XMAD, PASS_RECIPROCAL, PASS_AGGREGATE, PASS_TAG = 1, 2, 4, 8
PASS_ALL = 15
PASS_MATCH_ONLY, PASS_MATCH_XMAD = 16, 32
RAW_X4, RAW_SR = 1, 2

# ---------------------------------------------------------------- opcode table
OPF = {"CL_OPF_PURE": 1, "CL_OPF_LDST": 2, "CL_OPF_GLOBAL": 4, "CL_OPF_ATOMIC": 8,
       "CL_OPF_LOAD": 16, "CL_OPF_D64": 32}


def _parse_ops():
    names, flags = [], []
    text = (INCLUDE / "culifter_ops.h").read_text()
    for m in re.finditer(r"^CL_OP\((\w+),\s*([^)]*)\)", text, re.M):
        names.append(m.group(1))
        f = 0
        for tok in m.group(2).split("|"):
            tok = tok.strip()
            f |= OPF[tok] if tok in OPF else int(tok, 0)
        flags.append(f)
    return names, flags


OP_NAMES, OP_FLAGS = _parse_ops()
OP_FIXED = len(OP_NAMES)

# modifier universe: built-in bits (enum cl_modbit) first
BUILTIN_MODS = ("X4", "WIDE", "U32", "S32", "LO", "HI", "RCP", "SYNC", "64", "128",
                "F64", "S64", "U64")
WELLKNOWN_MODSETS = ((), ("LO",), ("HI",), ("S64",), ("U64",), ("F2I",), ("I2F",))
MAX_GROUPS = 4


class Tables:
    """Process-wide interning of the strings the device only sees as ids."""

    def __init__(self):
        self.op_id = {n: i for i, n in enumerate(OP_NAMES)}
        self.op_name = list(OP_NAMES)
        self.modset_id = {}
        self.modset_tuple = []
        for ms in WELLKNOWN_MODSETS:
            self.modset(ms)
        self.str_id = {}
        self.strings = []
        self.universe = list(BUILTIN_MODS)
        self.groups = []          # list of tuples of modifier names

    # -- interning ----------------------------------------------------------
    def opcode(self, base: str) -> int:
        i = self.op_id.get(base)
        if i is None:
            i = len(self.op_name)
            if i >= 0xFFFF:
                raise ValueError("opcode table overflow")
            self.op_id[base] = i
            self.op_name.append(base)
        return i

    def modset(self, mods) -> int:
        mods = tuple(mods)
        i = self.modset_id.get(mods)
        if i is None:
            i = len(self.modset_tuple)
            if i >= 0xFFFF:
                raise ValueError("modifier-set table overflow")
            self.modset_id[mods] = i
            self.modset_tuple.append(mods)
            # derived tuples the device may need to name (IMAD64 retag, .X4 strip)
            if "WIDE" in mods:
                self.modset(m for m in mods if m != "WIDE")
            if "X4" in mods:
                self.modset(m for m in mods if m != "X4")
        return i

    def string(self, s: str) -> int:
        i = self.str_id.get(s)
        if i is None:
            i = len(self.strings)
            self.str_id[s] = i
            self.strings.append(s)
        return i

    # -- modifier universe ----------------------------------------------------
    def mod_bit(self, name: str) -> int:
        if name not in self.universe:
            if len(self.universe) >= 64:
                raise ValueError("more than 64 pattern-relevant modifiers")
            self.universe.append(name)
        return self.universe.index(name)

    def group(self, choices) -> int:
        choices = tuple(choices)
        if choices not in self.groups:
            if len(self.groups) >= MAX_GROUPS:
                raise ValueError("more than 4 mod_var choice groups")
            for c in choices:
                self.mod_bit(c)
            self.groups.append(choices)
        return self.groups.index(choices)

    def modset_info(self) -> np.ndarray:
        """cl_modset[] for every interned tuple under the current universe."""
        n = len(self.modset_tuple)
        out = np.zeros(n, MODSET)
        bit = {m: i for i, m in enumerate(self.universe)}
        i = 0
        while i < len(self.modset_tuple):       # modset() may append while we walk
            mods = self.modset_tuple[i]
            i += 1
            if "WIDE" in mods:
                self.modset(m for m in mods if m != "WIDE")
            if "X4" in mods:
                self.modset(m for m in mods if m != "X4")
        n = len(self.modset_tuple)
        out = np.zeros(n, MODSET)
        for i, mods in enumerate(self.modset_tuple):
            mask = 0
            for m in mods:
                if m in bit:
                    mask |= 1 << bit[m]
            out["mask"][i] = mask
            first = [0xFF] * MAX_GROUPS
            for g, choices in enumerate(self.groups):
                got = next((m for m in mods if m in choices), None)
                if got is not None:
                    first[g] = bit[got]
            out["first"][i] = first
            out["minus_wide"][i] = self.modset_id[tuple(m for m in mods if m != "WIDE")] \
                if "WIDE" in mods else i
            out["minus_x4"][i] = self.modset_id[tuple(m for m in mods if m != "X4")] \
                if "X4" in mods else i
        return out


TABLES = Tables()
