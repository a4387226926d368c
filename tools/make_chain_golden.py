"""Golden fixture for the order-dependent reciprocal chains (normalize_reciprocal, patterns.py:817-888): hand-written
listings in which a chain reaches its F2I only THROUGH another chain's add, so that the reference's sequential
rewrite (bitcasts lengthen the paths of the chains after it) decides -- accepted at exactly three hops, rejected at
four, and the same shapes with the roles in the other stream order.  Inputs by the reference's front half, expected
results by the reference's own passes.  Build container only.  -> tests/golden/chains.pkl.gz"""
import gzip
import pickle
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import make_golden as MG  # noqa: E402
import refharness as R  # noqa: E402
from paper_2604_27486_b200 import ir  # noqa: E402


def listing(name, body):
    lines = [f".text.{name}:"]
    for k, inst in enumerate(body + ["EXIT", "NOP"]):
        lines.append(f"{k * 0x10:#x}: {inst}")
    return "\n".join(lines) + "\n"


def chain_cases():
    """(name, instructions).  A = (MUFU R3, add R7), B = (MUFU R5, add R6); A's add reads B's result."""
    head = ["I2F.F32.U32 R2, R0", "MUFU.RCP R3, R2", "I2F.F32.U32 R4, R1", "MUFU.RCP R5, R4",
            "IADD3 R6, R5, 0x2, RZ",            # add of B (its MUFU comes second: B is decided after A)
            "IADD3 R7, R3, 0x2, R6"]            # add of A, reads B's result
    tail = ["STG.E [R20.64], R9"]
    cases = [
        ("b_rejected", head + ["FMUL R8, R7, R1", "F2I.FTZ.U32.F32.TRUNC R9, R8"] + tail),        # B: add, add A, FMUL, F2I = 3 hops, 4 once A is rewritten
        ("b_accepted", head + ["F2I.FTZ.U32.F32.TRUNC R9, R7"] + tail),                            # B: 2 hops, 3 once A is rewritten
        ("b_other_path", head + ["FMUL R8, R7, R1", "F2I.FTZ.U32.F32.TRUNC R9, R8", "FMUL R10, R6, R1",
                                 "F2I.FTZ.U32.F32.TRUNC R11, R10", "STG.E [R22.64], R11"] + tail),   # B also reaches an F2I of its own
        ("a_unreachable", head + ["FMUL R8, R7, R1", "FMUL R12, R8, R1", "FMUL R13, R12, R1",
                                  "F2I.FTZ.U32.F32.TRUNC R9, R13"] + tail),                          # nobody within three hops
    ]
    # the other stream order: B's MUFU first, so B is decided BEFORE A and sees no rewrite
    head2 = ["I2F.F32.U32 R4, R1", "MUFU.RCP R5, R4", "I2F.F32.U32 R2, R0", "MUFU.RCP R3, R2",
             "IADD3 R6, R5, 0x2, RZ", "IADD3 R7, R3, 0x2, R6"]
    cases.append(("b_first", head2 + ["FMUL R8, R7, R1", "F2I.FTZ.U32.F32.TRUNC R9, R8"] + tail))
    # three chains in a row: C -> B -> A -> F2I
    cases.append(("three", ["I2F.F32.U32 R2, R0", "MUFU.RCP R3, R2", "I2F.F32.U32 R4, R1", "MUFU.RCP R5, R4",
                            "I2F.F32.U32 R14, R1", "MUFU.RCP R15, R14",
                            "IADD3 R16, R15, 0x2, RZ", "IADD3 R6, R5, 0x2, R16", "IADD3 R7, R3, 0x2, R6",
                            "F2I.FTZ.U32.F32.TRUNC R9, R7"] + tail))
    # the add result is ALSO an address base (not renamed by the rewrite: that edge keeps one hop)
    cases.append(("memref_edge", head + ["LDG.E R8, [R7.64]", "F2I.FTZ.U32.F32.TRUNC R9, R8"] + tail))
    return cases


def main():
    R.load()
    fns = []
    text = "".join(listing(n, body) for n, body in chain_cases())
    for fn in R.ssa_functions(text, "sm90"):
        fns.append(fn)
    MG.write("chains", fns, 15)
    fix = pickle.load(gzip.open(ROOT / "tests" / "golden" / "chains.pkl.gz", "rb"))
    for fn, exp in zip(fix["functions"], fix["expect"]):
        print(fn.name, "->", "error " + exp["error"] if "error" in exp else f"{len(exp.get('pattern_boundaries', []))} chain(s) rewritten: {exp.get('pattern_boundaries')}")


if __name__ == "__main__":
    main()
