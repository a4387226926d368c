"""Generate the travelling parity fixtures under tests/golden/ (in-container
only: needs the reference at /root/reference).

Each fixture is a gzip pickle of
    {"name", "passes", "functions": [paper_2604_27486_b200.ir.LiftedFunction ...],
     "expect": [state dict | {"error": "KeyError"} ...]}
where `functions` are SSA-phase inputs produced by the reference's own front
half and `expect` is what the reference's own passes
(normalize_xmad / normalize_reciprocal / apply_aggregations / tag_cuda_objects,
pipeline.py:165-169) make of them: dump() text, diagnostics, pattern
boundaries, CUDA-object tags, id counters and the value table.
"""
import gzip, pickle, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import refharness as R
import gen_sass
from paper_2604_27486_b200 import ir

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

SNIPPETS = {  # the shapes of the reference's own unit tests (tests/test_patterns.py)
    "interleaved_pairs": ("sm90", """.text.k:
IADD3 R4, P0, R0, R2, RZ
IADD3 R8, P1, R10, R12, RZ
IADD3.X R5, R1, R3, RZ, P0, !PT
IADD3.X R9, R11, R13, RZ, P1, !PT
EXIT
"""),
    "inconsistent_carry": ("sm90", """.text.k:
IADD3 R4, P0, R0, R2, RZ
IADD3.X R5, R1, R3, RZ, P1, !PT
EXIT
"""),
    "carry_escape": ("sm90", """.text.k:
IADD3 R4, P0, R0, R2, RZ
IADD3.X R5, R1, R3, RZ, P0, !PT
SEL R6, 0x1, RZ, P0
STG.E.64 [R10], R4
STG.E [R12], R6
EXIT
"""),
    "carry_in_pt": ("sm90", """.text.k:
IADD3 R4, P0, R0, R2, RZ
IADD3.X R5, R1, R3, RZ, PT, !PT
IADD3 R8, P1, R4, R2, RZ
IADD3.X R9, R5, R3, RZ, P1, !PT
STG.E.64 [R10], R8
EXIT
"""),
    "mov_rz_pair": ("sm75", """.text.k:
MOV R4, c[0x0][0x160]
MOV R5, c[0x0][0x164]
MOV R6, RZ
LDG.E R8, [R4]
STG.E.64 [R4], R6
EXIT
"""),
    "fadd_only": ("sm75", """.text.k:
FADD R0, R1, R2
FADD R3, R0, R2
EXIT
"""),
    "xmad_on_sm90": ("sm90", """.text.k:
XMAD.MRG R2, R0, R0.H1, RZ
XMAD R3, R0, R2, RZ
XMAD.PSL.CBCC R4, R0.H1, R3, R1
EXIT
"""),
}


def expected(fns, passes):
    """-> (states, match lists): what the reference's passes make of every function, and the
    (pattern.name, positions) lists its match_patterns / select_matches returned on the way."""
    out, mlists = [], []
    for fn in fns:
        ref = R.clone(fn)
        ms = []
        err = R.run_postssa(ref, xmad=bool(passes & 1), recip=bool(passes & 2),
                            aggregate=bool(passes & 4), tag=bool(passes & 8), matches=ms)
        out.append({"error": type(err).__name__} if err is not None else R.state_of(ref))
        mlists.append(None if err is not None else [(ph, bi, [tuple(x) for x in raw], [tuple(x) for x in sel]) for ph, bi, raw, sel in ms])
    return out, mlists


def write(name, fns, passes=15):
    exp, mlists = expected(fns, passes)
    fix = {"name": name, "passes": passes, "functions": [ir.convert(f) for f in fns],
           "expect": exp, "matches": mlists}
    path = OUT / f"{name}.pkl.gz"
    with gzip.open(path, "wb", compresslevel=9) as fh:
        pickle.dump(fix, fh, protocol=4)
    n = sum(len(b.instructions) for f in fns for b in f.blocks.values())
    print(f"{path.name}: {len(fns)} functions, {n} records, {path.stat().st_size} bytes")


def raw_state(fn):
    from sasslift.ssir import dump
    return {"dump": dump(fn), "next_iid": fn._next_iid, "next_temp_reg": fn.meta.get("next_temp_reg", 1000),
            "synthetic": [(i.iid, i.meta.get("synthetic")) for i in fn.raw_instructions if i.meta.get("synthetic")],
            "diagnostics": list(fn.diagnostics)}


def write_raw(name, texts):
    """Raw-stage fixtures: `<name>_x4` (parsed -> normalize_instruction on every
    instruction, frontend.py:523) and `<name>_sr` (parsed + normalized + expanded ->
    substitute_special_registers, frontend.py:697)."""
    R.load()
    from sasslift import frontend
    x4_in, x4_exp, sr_in, sr_exp = [], [], [], []
    for arch, text in texts:
        for fn in R.raw_functions(text, arch, normalize=False):
            x4_in.append(ir.convert(fn))
            out = []
            for inst in fn.raw_instructions:
                out.extend(frontend.normalize_instruction(fn, inst))
            fn.raw_instructions = out
            x4_exp.append(raw_state(fn))
            for inst in fn.raw_instructions:
                frontend.expand_implicit_registers(inst, arch)
            sr_in.append(ir.convert(fn))
            frontend.substitute_special_registers(fn)
            sr_exp.append(raw_state(fn))
    for suffix, fns, exp in (("x4", x4_in, x4_exp), ("sr", sr_in, sr_exp)):
        path = OUT / f"{name}_{suffix}.pkl.gz"
        with gzip.open(path, "wb", compresslevel=9) as fh:
            pickle.dump({"name": f"{name}_{suffix}", "kind": "raw_" + suffix, "functions": fns, "expect": exp}, fh, protocol=4)
        print(f"{path.name}: {len(fns)} functions, {sum(len(f.raw_instructions) for f in fns)} instructions, {path.stat().st_size} bytes")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    raw_texts = [("sm52", gen_sass.gen_corpus(21, "sm52", 30, near_miss=0.2)[1]),
                 ("sm75", gen_sass.gen_corpus(22, "sm75", 10)[1])]
    for f in R.corpus_files():
        man = f.with_suffix(".manifest")
        arch = "sm75"
        if man.exists():
            for ln in man.read_text().splitlines():
                if ln.startswith("arch:"):
                    arch = ln.split(":")[1].strip()
        raw_texts.append((arch, f.read_text()))
    write_raw("raw", raw_texts)
    fns = []
    for f in R.corpus_files():
        fns += R.ssa_from_path(f)
    write("bundled", fns)
    write("bundled_noagg", [f for p in R.corpus_files() for f in R.ssa_from_path(p)], passes=11)
    sn = []
    for name, (arch, text) in SNIPPETS.items():
        for f in R.ssa_functions(text, arch):
            f.name = name
            sn.append(f)
    write("snippets", sn)
    for kind, seed, n in (("sm90", 11, 40), ("sm52", 12, 40), ("sm75", 13, 30), ("long", 14, 3)):
        arch, text = gen_sass.gen_corpus(seed, kind, n, near_miss=0.15)
        write(f"synth_{kind}", R.ssa_functions(text, arch))
    # BASELINE.json configs[3] at its defining size: one 4096- and one 8192-instruction block (budget cut of
    # patterns.py:194-198 active, reciprocal chains interleaved with IADD3 pairs); ~2 minutes of reference time
    import random
    rng = random.Random(4096)
    text = "".join(gen_sass.gen_function(rng, f"long{size}", "sm90", gen_sass.MIX_LONG, 1, (size, size), 0.1, window=16)
                   for size in (4096, 8192))
    write("long_blocks", R.ssa_functions(text, "sm90"))


if __name__ == "__main__":
    main()
