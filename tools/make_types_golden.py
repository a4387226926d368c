"""Generate tests/golden/types.pkl.gz (in-container only: needs /root/reference).

TEST INFRASTRUCTURE.  For every function of the bundled corpus, of three small
synthetic corpora and of a hand-written listing that reaches the signature
branches those do not, the reference's own front half and hot-path passes
(pipeline.py:109-169) produce the NORMALIZED function, and the reference's own
``typerec.seed_types`` (typerec.py:288) its ``TypeState``.  The fixture holds
    {"functions": [paper_2604_27486_b200.ir.LiftedFunction ...]  (input of seed_types),
     "expect": [{"seed_mask", "def_seed_mask", "use_seed_mask", "roles", "link_exprs"} ...]}
"""
import gzip, pickle, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import refharness as R
import gen_sass
from paper_2604_27486_b200 import ir

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

EXTRA = ("sm90", """.text.sigs:
S2R R0, SR_TID.X
MOV R2, c[0x0][0x160]
MOV R3, c[0x0][0x164]
IMAD.WIDE R4, R0, 0x4, R2
LDG.E R6, [R4.64]
LDG.E.64 R8, [R4.64+0x8]
LDS R10, [R0]
I2F R11, R6
I2F.F64.S64 R12, R8
F2I.U64.F64 R14, R12
F2F.F16.F32 R16, R11
F2F.F64.F32 R18, R11
FRND.F64 R20, R18
I2I.S32.S16 R22, R6
HADD2 R23, R16, R16
HFMA2.BF16 R24, R23, R23, R23
DADD R26, R18, R20
DSETP.GT.AND P0, PT, R26, R20, PT
FSETP.GT.AND P1, PT, R11, R11, PT
FSEL R28, R11, R11, P1
ISETP.GE.AND P2, PT, R6, R0, PT
PLOP3.LUT P3, PT, P0, P1, P2, 0x80, 0x0
SEL R29, R6, R0, P3
LOP3.LUT R30, R29, R6, R0, 0xfe, !PT
SHF.R.U32.HI R31, RZ, 0x3, R30
SHL R32, R31, 0x2
LEA.HI R33, R32, R30, RZ, 0x2
SHFL.BFLY PT, R34, R33, 0x1, 0x1f
VOTE.ANY R35, PT, P3
ATOMG.ADD R36, [R4.64], R35
ATOMS.ADD R37, [R0], R35
ATOMG.ADD.F32 R38, [R4.64], R28
RED.E.ADD.F32.FTZ.RN [R4.64], R28
POPC R39, R34
@P3 STG.E [R4.64], R39
STG.E.64 [R4.64+0x10], R26
STS [R0], R37
MUFU.RCP R40, R11
FMNMX R41, R40, R11, PT
IADD3 R42, P4, R36, R38, RZ
IADD3.X R43, R37, R39, RZ, P4, !PT
STG.E.64 [R4.64+0x20], R42
FADD R44, R41, R11
STG.E [R4.64+0x30], R44
EXIT
""")


def type_state(fn):
    from sasslift import typerec
    st = typerec.seed_types(fn)
    return {"seed_mask": dict(st.seed_mask), "def_seed_mask": dict(st.def_seed_mask),
            "use_seed_mask": dict(st.use_seed_mask), "roles": dict(st.roles),
            "link_exprs": {k: [list(x) for x in v] for k, v in st.link_exprs.items()}}


def main():
    R.load()
    fns = []
    for f in R.corpus_files():
        fns += R.ssa_from_path(f)
    for kind, seed, n in (("sm90", 31, 12), ("sm52", 32, 12), ("sm75", 33, 10)):
        arch, text = gen_sass.gen_corpus(seed, kind, n, near_miss=0.15)
        fns += R.ssa_functions(text, arch)
    fns += R.ssa_functions(EXTRA[1], EXTRA[0])
    kept, expect, kinds = [], [], {}
    for fn in fns:
        if R.run_postssa(fn) is not None:
            continue                                   # functions the passes fail on never reach typerec
        from sasslift.ssir import Phase
        fn.advance_phase(Phase.NORMALIZED)             # pipeline.py:171
        kept.append(ir.convert(fn))                    # the input of seed_types (it does not change the stream)
        expect.append(type_state(fn))
        for b in fn.block_order():
            for i in b.instructions:
                kinds[i.opcode.base] = kinds.get(i.opcode.base, 0) + 1
    path = OUT / "types.pkl.gz"
    with gzip.open(path, "wb", compresslevel=9) as fh:
        pickle.dump({"name": "types", "functions": kept, "expect": expect}, fh, protocol=4)
    n = sum(len(b.instructions) for f in kept for b in f.blocks.values())
    print(f"{path.name}: {len(kept)} functions, {n} records, {path.stat().st_size} bytes")
    print("opcode bases covered:", " ".join(f"{k}:{v}" for k, v in sorted(kinds.items())))


if __name__ == "__main__":
    main()
