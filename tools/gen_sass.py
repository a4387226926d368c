"""Synthetic SASS *text* generators for the parity corpora (TEST INFRASTRUCTURE).

The listings go through the reference's own front half (parse -> CFG -> SSA,
``tools/refharness.py``) in this container; the resulting SSA-phase functions
and the reference's outputs travel to the GPU box as fixtures under
``tests/golden/``.  Shapes follow SURVEY section 8(d): SM52 XMAD-heavy, SM90
aggregation idioms with deliberate near-misses, long unrolled blocks with
fast-division chains.  The large benchmark corpora are generated directly in
struct-of-arrays form by ``paper_2604_27486_b200/synth.py``.
"""
from __future__ import annotations

import random

CONDS = ("EQ", "NE", "LT", "LE", "GT", "GE")
BOPS = ("AND", "OR", "XOR")


class FnGen:
    def __init__(self, rng: random.Random, name: str, arch: str):
        self.rng, self.name, self.arch = rng, name, arch
        self.lines: list[str] = []
        self.next_reg = 4
        self.live = [0, 1, 2, 3]          # 32-bit registers with a value
        self.pairs = []                   # even registers holding 64-bit pairs
        self.next_pred = 0

    # ---- resources -------------------------------------------------------
    def reg(self):
        r = self.next_reg
        self.next_reg += 1
        if self.next_reg > 230:
            self.next_reg = 4
        return r

    def pair(self):
        if self.next_reg % 2:
            self.next_reg += 1
        r = self.next_reg
        self.next_reg += 2
        if self.next_reg > 230:
            self.next_reg = 4
        return r

    def pred(self):
        p = self.next_pred
        self.next_pred = (self.next_pred + 1) % 6
        return p

    def src(self):
        return self.rng.choice(self.live)

    def src_pair(self):
        if not self.pairs or self.rng.random() < 0.2:
            p = self.pair()
            self.emit([f"IMAD.WIDE R{p}, R{self.src()}, R{self.src()}, c[0x0][{0x160 + 8 * self.rng.randrange(8):#x}]"])
            self.pairs.append(p)
            self.live += [p, p + 1]
        return self.rng.choice(self.pairs)

    def define(self, r):
        self.live.append(r)
        if len(self.live) > 48:
            self.live.pop(self.rng.randrange(len(self.live) - 8))

    def define_pair(self, p):
        self.pairs.append(p)
        if len(self.pairs) > 12:
            self.pairs.pop(0)
        self.define(p)
        self.define(p + 1)

    def emit(self, insts):
        self.lines.extend(insts)

    # ---- idioms: each returns a list of instruction strings ----------------
    def iadd3_pair(self, near_miss=False):
        rng = self.rng
        a, b = self.src_pair(), self.src_pair()
        d, p = self.pair(), self.pred()
        kind = rng.choice(["plain", "plain", "neg", "imm", "immimm", "ur", "rzlo"])
        lo_b, hi_b = f"R{b}", f"R{b + 1}"
        if kind == "neg":
            lo_b, hi_b = f"-R{b}", f"~R{b + 1}"
        elif kind == "imm":
            lo_b, hi_b = hex(rng.randrange(1, 1 << 16)), "RZ"
        elif kind == "immimm":
            lo_b, hi_b = hex(rng.randrange(1, 1 << 31)), hex(rng.randrange(1, 1 << 16))
        elif kind == "ur":
            lo_b, hi_b = "-UR6", "~UR7"
        elif kind == "rzlo":
            lo_b, hi_b = "RZ", hex(rng.randrange(1, 1 << 12))
        third_lo, third_hi = "RZ", "RZ"
        if rng.random() < 0.15:
            third_lo, third_hi = f"R{self.src()}", f"R{self.src()}"
        out = [f"IADD3 R{d}, P{p}, R{a}, {lo_b}, {third_lo}",
               f"IADD3.X R{d + 1}, R{a + 1}, {hi_b}, {third_hi}, P{p}, !PT"]
        if near_miss:
            how = rng.choice(["mixed", "escape", "wrongcarry", "allzero"])
            if how == "mixed":
                out[0] = f"IADD3 R{d}, P{p}, R{a}, -R{b}, RZ"
                out[1] = f"IADD3.X R{d + 1}, R{a + 1}, R{b + 1}, RZ, P{p}, !PT"
            elif how == "escape":
                out.append(f"SEL R{self.reg()}, 0x1, RZ, P{p}")
            elif how == "wrongcarry":
                out[1] = f"IADD3.X R{d + 1}, R{a + 1}, {hi_b}, RZ, P{(p + 1) % 6}, !PT"
            else:
                out[0] = f"IADD3 R{d}, P{p}, RZ, RZ, RZ"
                out[1] = f"IADD3.X R{d + 1}, RZ, RZ, RZ, P{p}, !PT"
        self.define_pair(d)
        return out

    def isetp_pair(self, near_miss=False):
        rng = self.rng
        a, b, p = self.src_pair(), self.src_pair(), self.pred()
        cond, bop = rng.choice(CONDS), rng.choice(BOPS)
        acc = rng.choice(["PT", "PT", "!PT", f"P{(p + 3) % 6}"])
        hi_u = ".U32" if rng.random() < 0.5 else ""
        lo_b, hi_b = f"R{b}", f"R{b + 1}"
        r = rng.random()
        if r < 0.2:
            lo_b, hi_b = hex(rng.randrange(1 << 12)), "RZ"
        elif r < 0.3:
            lo_b, hi_b = "RZ", "RZ"
        out = [f"ISETP.{cond}.U32.{bop} P{p}, PT, R{a}, {lo_b}, {acc}",
               f"ISETP.{cond}{hi_u}.{bop}.EX P{p}, PT, R{a + 1}, {hi_b}, {acc}, P{p}"]
        if near_miss:
            other = rng.choice([c for c in CONDS if c != cond])
            out[1] = f"ISETP.{other}{hi_u}.{bop}.EX P{p}, PT, R{a + 1}, {hi_b}, {acc}, P{p}"
        out.append(f"SEL R{self.reg_def()}, 0x1, RZ, P{p}")
        return out

    def reg_def(self):
        r = self.reg()
        self.define(r)
        return r

    def lea_pair(self, near_miss=False):
        rng = self.rng
        x, b = self.src(), self.src_pair()
        sign = self.reg()
        d, p = self.pair(), self.pred()
        sh = rng.choice(["0x2", "0x3", "0x1"])
        out = [f"SHF.R.S32.HI R{sign}, RZ, 0x1f, R{x}",
               f"LEA R{d}, P{p}, R{x}, R{b}, {sh}",
               f"LEA.HI.X R{d + 1}, R{x}, R{b + 1}, R{sign}, {'0x4' if near_miss else sh}, P{p}"]
        self.define(sign)
        self.define_pair(d)
        out.append(f"LDG.E R{self.reg_def()}, [R{d}]")
        return out

    def imad_wide(self, near_miss=False):
        p = self.pair()
        out = [f"IMAD.WIDE{'.U32' if self.rng.random() < 0.3 else ''} R{p}, R{self.src()}, "
               f"R{self.src()}, c[0x0][{0x160 + 8 * self.rng.randrange(8):#x}]"]
        self.define_pair(p)
        if self.rng.random() < 0.7:
            out.append(f"LDG.E R{self.reg_def()}, [R{p}]")
        return out

    def mov_pair(self, near_miss=False):
        p = self.pair()
        off = 0x160 + 8 * self.rng.randrange(16)
        off2 = off + (8 if near_miss else 4)
        out = [f"MOV R{p}, c[0x0][{off:#x}]", f"MOV R{p + 1}, c[0x0][{off2:#x}]"]
        self.define_pair(p)
        if self.rng.random() < 0.3:      # a 32-bit consumer keeps one half alive
            out.append(f"IADD3 R{self.reg_def()}, R{p}, 0x1, RZ")
        out.append(f"LDG.E R{self.reg_def()}, [R{p}]")
        return out

    def cast64(self, near_miss=False):
        p = self.pair()
        out = [f"LDG.E R{p}, [R{self.src_pair()}]",
               f"SHF.R.S32.HI R{p + 1}, RZ, {'0x1e' if near_miss else '0x1f'}, R{p}",
               f"STG.E.64 [R{self.src_pair()}], R{p}"]
        self.define_pair(p)
        return out

    def shl64(self, near_miss=False):
        s, sh, d = self.src_pair(), self.src(), self.pair()
        sh = f"R{sh}" if self.rng.random() < 0.6 else hex(self.rng.randrange(1, 31))
        out = [f"SHF.L.U64.HI R{d + 1}, R{s}, {sh}, R{s + 1}",
               f"SHF.L.U32 R{d}, R{s}, {sh if not near_miss else '0x7'}, RZ",
               f"STG.E.64 [R{self.src_pair()}], R{d}"]
        self.define_pair(d)
        return out

    def shr64(self, near_miss=False):
        s, sh, d = self.src_pair(), self.src(), self.pair()
        sg = self.rng.choice(["U32", "S32"])
        sh = f"R{sh}" if self.rng.random() < 0.6 else hex(self.rng.randrange(1, 31))
        hi_src = f"R{s + 1}" if not near_miss else f"R{self.src()}"
        out = [f"SHF.R.{sg}.HI R{d + 1}, R{s}, {sh}, R{s + 1}",
               f"SHF.R.{'U32' if sg == 'U32' else 'U32'} R{d}, R{s}, {sh}, {hi_src}",
               f"STG.E.64 [R{self.src_pair()}], R{d}"]
        self.define_pair(d)
        return out

    def fastdiv(self, near_miss=False):
        rng = self.rng
        f, r, t, q = self.reg(), self.reg(), self.reg(), self.reg()
        out = [f"I2F.F32.U32 R{f}, R{self.src()}", f"MUFU.RCP R{r}, R{f}",
               f"IADD3 R{t}, R{r}, {rng.choice(['0xffffffe', '-0x1', '0x2'])}, RZ"]
        hops = rng.choice([0, 0, 1, 2, 3]) if not near_miss else 3
        cur = t
        for _ in range(hops):
            n = self.reg()
            out.append(f"FMUL R{n}, R{cur}, R{self.src()}")
            cur = n
        out.append(f"F2I.FTZ.U32.F32.TRUNC R{q}, R{cur}")
        if rng.random() < 0.3:
            out.append(f"FADD R{self.reg_def()}, R{t}, R{r}")     # extra users of both
        self.define(q)
        return out

    def cuda_object(self, near_miss=False):
        return [self.rng.choice(["BAR.SYNC 0x0", "BAR.SYNC 0x1", "WARPSYNC 0xffffffff",
                                 "WARPSYNC 0xff", f"SHFL.BFLY PT, R{self.reg_def()}, R{self.src()}, 0x10, 0x1f"])]

    def xmad_a(self, near_miss=False):
        a, b, c = self.src(), self.src(), self.src()
        m, t, d = self.reg(), self.reg(), self.reg_def()
        bb = f"R{b}" if self.rng.random() < 0.7 else "c[0x0][0x8]"
        out = [f"XMAD.MRG R{m}, R{a}, {bb}.H1, RZ",
               f"XMAD R{t}, R{a}, R{m}, RZ",
               f"XMAD.PSL.CBCC R{d}, R{a}.H1, R{t}, R{c}"]
        if near_miss:
            how = self.rng.choice(["escape", "half", "other"])
            if how == "escape":
                out.append(f"IADD R{self.reg_def()}, R{t}, R{m}")
            elif how == "half":
                out[2] = f"XMAD.PSL.CBCC R{d}, R{a}, R{t}, R{c}"
            else:
                out[1] = f"XMAD R{t}, R{self.src()}, R{m}, RZ"
        return out

    def xmad_b(self, near_miss=False):
        a, c = self.src(), self.src()
        m, t, d = self.reg(), self.reg(), self.reg_def()
        b = f"R{self.src()}" if self.rng.random() < 0.4 else \
            f"c[0x0][{8 * self.rng.randrange(1, 6):#x}]"
        out = [f"XMAD.MRG R{m}, R{a}, {b}.H1, RZ",
               f"XMAD R{t}, R{a}, {b}, R{c}",
               f"XMAD.PSL.CBCC R{d}, R{a}.H1, R{m}.H1, R{t}"]
        if near_miss:
            out[1] = f"XMAD R{t}, R{a}, R{self.src()}, R{c}"
        return out

    def x4_access(self, near_miss=False):
        if self.rng.random() < 0.5:
            return [f"LDG.E.X4 R{self.reg_def()}, [R{self.src_pair()}+{4 * self.rng.randrange(8):#x}]"]
        return [f"STG.E.X4 [R{self.src_pair()}], R{self.src()}"]

    def sr_use(self, near_miss=False):
        off = "0x2c" if not near_miss else "0x30"
        return [self.rng.choice([
            f"IADD R{self.reg_def()}, R{self.src()}, c[0x0][{off}]",
            f"XMAD R{self.reg_def()}, R{self.src()}, c[0x0][{off}].H1, RZ",
            f"FADD R{self.reg_def()}, -c[0x0][{off}], R{self.src()}"])]

    def filler(self, near_miss=False):
        rng = self.rng
        k = rng.randrange(7)
        d = self.reg_def()
        if k == 0:
            return [f"FFMA R{d}, R{self.src()}, R{self.src()}, R{self.src()}"]
        if k == 1:
            return [f"FADD R{d}, R{self.src()}, -R{self.src()}"]
        if k == 2:
            return [f"IADD3 R{d}, R{self.src()}, {hex(rng.randrange(64))}, RZ"] if self.arch != "sm52" \
                else [f"IADD R{d}, R{self.src()}, {hex(rng.randrange(64))}"]
        if k == 3:
            return [f"LOP3.LUT R{d}, R{self.src()}, R{self.src()}, RZ, 0xc0, !PT"] if self.arch != "sm52" \
                else [f"LOP.AND R{d}, R{self.src()}, R{self.src()}"]
        if k == 4:
            return [f"MOV R{d}, {hex(rng.randrange(1 << 20))}"]
        if k == 5:
            return [f"LDG.E R{d}, [R{self.src_pair()}]"]
        return [f"MOV R{d}, R{self.src()}"]


def interleave(rng, groups):
    """Random merge of instruction groups that keeps each group's order."""
    out, heads = [], [0] * len(groups)
    alive = [i for i, g in enumerate(groups) if g]
    while alive:
        i = rng.choice(alive)
        out.append(groups[i][heads[i]])
        heads[i] += 1
        if heads[i] == len(groups[i]):
            alive.remove(i)
    return out


MIX_SM90 = [("iadd3_pair", 4), ("isetp_pair", 3), ("lea_pair", 2), ("imad_wide", 3),
            ("mov_pair", 2), ("cast64", 2), ("shl64", 2), ("shr64", 2), ("fastdiv", 1),
            ("cuda_object", 1), ("filler", 8)]
MIX_SM52 = [("xmad_a", 5), ("xmad_b", 2), ("x4_access", 2), ("sr_use", 2), ("filler", 8),
            ("fastdiv", 1)]
MIX_LONG = [("fastdiv", 6), ("iadd3_pair", 8), ("imad_wide", 1), ("filler", 5), ("mov_pair", 1)]


def gen_function(rng, name, arch, mix, n_blocks, block_len, near_miss=0.1, window=6):
    """One listing ``.text.<name>``: blocks end in a forward conditional branch
    (or a backward one: loops), the last one in EXIT."""
    g = FnGen(rng, name, arch)
    names = [m for m, w in mix for _ in range(w)]
    blocks = []
    for _ in range(n_blocks):
        groups = []
        count = 0
        target = rng.randrange(block_len[0], block_len[1] + 1)
        while count < target:
            idiom = rng.choice(names)
            grp = getattr(g, idiom)(near_miss=rng.random() < near_miss)
            pre = g.lines[:]              # helper definitions emitted by src_pair()
            g.lines.clear()
            if pre:
                groups.append(pre)
            groups.append(grp)
            count += len(grp) + len(pre)
        body = []
        for k in range(0, len(groups), window):      # interleave inside small windows
            body += interleave(rng, groups[k:k + window])
        blocks.append(body)
    addr, text, starts = 0, [], []
    for body in blocks:
        starts.append(addr)
        addr += 0x10 * (len(body) + 2)
    addr = 0
    lines = [f".text.{name}:"]
    for bi, body in enumerate(blocks):
        for inst in body:
            lines.append(f"{addr:#x}: {inst}")
            addr += 0x10
        if bi + 1 < len(blocks):
            p = rng.randrange(6)
            lines.append(f"{addr:#x}: ISETP.NE.AND P{p}, PT, R{g.src()}, RZ, PT")
            addr += 0x10
            tgt = rng.randrange(len(blocks)) if rng.random() < 0.3 else \
                rng.randrange(bi + 1, len(blocks))
            lines.append(f"{addr:#x}: @P{p} BRA {starts[tgt]:#x}")
            addr += 0x10
        else:
            lines.append(f"{addr:#x}: EXIT")
            addr += 0x10
            lines.append(f"{addr:#x}: NOP")      # keep table alignment with `starts`
            addr += 0x10
    return "\n".join(lines) + "\n"


def gen_corpus(seed, kind, n_functions, near_miss=0.1):
    """-> (arch, text) for one of the SURVEY 8(d) shapes."""
    rng = random.Random(seed)
    out = []
    for i in range(n_functions):
        if kind == "sm52":
            out.append(gen_function(rng, f"k{i}", "sm52", MIX_SM52, rng.randrange(1, 5), (6, 40), near_miss))
        elif kind == "sm90":
            out.append(gen_function(rng, f"k{i}", "sm90", MIX_SM90, rng.randrange(1, 6), (6, 60), near_miss))
        elif kind == "sm75":
            out.append(gen_function(rng, f"k{i}", "sm75", MIX_SM90, rng.randrange(1, 4), (4, 30), near_miss))
        elif kind == "long":
            out.append(gen_function(rng, f"k{i}", "sm90", MIX_LONG, 1,
                                    (rng.choice([300, 700, 1500]),) * 2, near_miss, window=12))
        else:
            raise ValueError(kind)
    arch = {"sm52": "sm52", "sm90": "sm90", "sm75": "sm75", "long": "sm90"}[kind]
    return arch, "".join(out)
