"""In-container bridge to the Python reference (``/root/reference/pkg/src``).

TEST INFRASTRUCTURE.  Runs the reference's own front half to obtain
``LiftedFunction`` objects in SSA phase (the input of the hot path) and the
reference's own passes to obtain the expected outputs.  The GPU box has no
``/root/reference``: everything produced here travels as fixtures under
``tests/golden/`` (see ``tools/make_golden.py``).
"""
from __future__ import annotations

import copy
import os
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_PKG = REF_SRC.parent


def available() -> bool:
    return (REF_SRC / "sasslift" / "patterns.py").exists()


def load():
    """Import and return the reference package (read-only tree: no bytecode)."""
    sys.dont_write_bytecode = True
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import sasslift  # noqa: F401
    return sasslift


def raw_functions(text: str, arch: str = "sm75", manifest_text: str | None = None,
                  normalize: bool = True):
    """Reference ``build_function`` for every function in a listing
    (``frontend.py:737``); with ``normalize=False`` stop after parsing."""
    load()
    from sasslift import arch as archmod
    from sasslift import frontend
    from sasslift.pipeline import parse_manifest
    manifest = parse_manifest(manifest_text) if manifest_text else None
    if manifest is not None and manifest.arch:
        arch = archmod.check_arch(manifest.arch)
    out = []
    for src in frontend.parse_module(text, arch, manifest):
        if normalize:
            out.append(frontend.build_function(src, arch, manifest))
        else:
            fn = frontend.LiftedFunction(src.name, arch, src.param_base)
            for line in src.lines:
                fn.raw_instructions.append(frontend.parse_instruction_line(fn, line))
            out.append(fn)
    return out


def ssa_functions(text: str, arch: str = "sm75", manifest_text: str | None = None,
                  inline_threshold: int | None = None):
    """Reference front half up to ``ssa_rename`` (``pipeline.py:109-157``):
    the functions exactly as ``normalize_xmad`` receives them."""
    load()
    from sasslift import arch as archmod
    from sasslift import cfg as cfgmod
    from sasslift import frontend, ssa
    from sasslift.pipeline import PipelineConfig, parse_manifest
    manifest = parse_manifest(manifest_text) if manifest_text else None
    if manifest is not None and manifest.arch:
        arch = archmod.check_arch(manifest.arch)
    thr = PipelineConfig().inline_threshold if inline_threshold is None else inline_threshold
    out = []
    for src in frontend.parse_module(text, arch, manifest):
        fn = frontend.build_function(src, arch, manifest)
        cfgmod.build_cfg(fn)
        fn, extracted = cfgmod.recover_device_functions(fn, thr)
        for sub in [fn] + list(extracted):
            ssa.construct_psi(sub)
            ssa.ssa_rename(sub)
            out.append(sub)
    return out


def ssa_from_path(path):
    p = Path(path)
    man = p.with_suffix(".manifest")
    return ssa_functions(p.read_text(), "sm75", man.read_text() if man.exists() else None)


def corpus_files():
    return sorted((REF_PKG / "corpus").rglob("*.sass"))


def run_postssa(fn, xmad=True, recip=True, aggregate=True, tag=True, snapshots=None, matches=None):
    """The four hot-path calls of ``pipeline.py:165-169`` on ``fn`` in place.
    Returns the exception (reference reports it per function) or None.

    ``matches``: a list that receives, for every block the reference matched in
    (``_apply_patterns``, patterns.py:676), ``(phase, block index, raw, selected)``
    with ``raw`` / ``selected`` = ``[(pattern name, positions...)]`` exactly as
    ``match_patterns`` / ``select_matches`` returned them (list order kept);
    phase 0 = the xmad round, 2 + r = aggregation round r -- the numbering of the
    device's CL_EV_MATCH events."""
    load()
    from sasslift import patterns as patmod
    from sasslift.ssir import dump
    saved = (patmod.match_patterns, patmod.select_matches, patmod._apply_patterns)
    if matches is not None:
        state = {"phase": 0, "agg_rounds": 0, "cur": None}
        order = {b.bid: k for k, b in enumerate(fn.block_order())}

        def apply_patterns(f, pats):
            if pats is patmod.XMAD_PATTERNS:
                state["phase"] = 0
            else:
                state["phase"] = 2 + state["agg_rounds"]
                state["agg_rounds"] += 1
            return saved[2](f, pats)

        def match_patterns(f, blk, pats, du=None):
            ms = saved[0](f, blk, pats, du)
            pos = {i.iid: k for k, i in enumerate(blk.instructions)}
            state["cur"] = (blk, pos)
            if ms:
                matches.append([state["phase"], order[blk.bid], [(m.pattern.name,) + tuple(pos[i.iid] for i in m.insts) for m in ms], []])
            return ms

        def select_matches(ms):
            sel = saved[1](ms)
            if ms:
                pos = state["cur"][1]
                matches[-1][3] = [(m.pattern.name,) + tuple(pos[i.iid] for i in m.insts) for m in sel]
            return sel

        patmod.match_patterns, patmod.select_matches, patmod._apply_patterns = match_patterns, select_matches, apply_patterns
    try:
        for name, on, call in (("xmad", xmad, patmod.normalize_xmad),
                               ("recip", recip, patmod.normalize_reciprocal),
                               ("agg", aggregate, patmod.apply_aggregations),
                               ("tag", tag, patmod.tag_cuda_objects)):
            if on:
                call(fn)
            if snapshots is not None:
                snapshots[name] = dump(fn)
    except Exception as e:  # noqa: BLE001 - mirrors pipeline.py:182
        return e
    finally:
        patmod.match_patterns, patmod.select_matches, patmod._apply_patterns = saved
    return None


def match_lists(fn, table="agg"):
    """Raw and selected matches of every block for the current state of ``fn``:
    [(bid, [(pattern, positions...)], [selected...])]."""
    load()
    from sasslift import patterns as patmod
    pats = patmod.AGGREGATION_PATTERNS if table == "agg" else patmod.XMAD_PATTERNS
    out = []
    for blk in fn.block_order():
        pos = {i.iid: k for k, i in enumerate(blk.instructions)}
        ms = patmod.match_patterns(fn, blk, pats)
        sel = patmod.select_matches(ms)
        key = lambda m: (m.pattern.name,) + tuple(pos[i.iid] for i in m.insts)
        out.append((blk.bid, [key(m) for m in ms], [key(m) for m in sel]))
    return out


def clone(fn):
    return copy.deepcopy(fn)


def state_of(fn):
    """Everything the hot path may change, as comparable plain data."""
    load()
    from sasslift.ssir import dump
    return {
        "dump": dump(fn),
        "diagnostics": list(fn.diagnostics),
        "boundaries": list(fn.meta.get("pattern_boundaries", [])),
        "cuda_objects": [tuple(t) for t in fn.meta.get("cuda_objects", [])],
        "next": (fn._next_vid, fn._next_iid),
        "values": {vid: (v.origin, v.def_iid) for vid, v in sorted(fn.values.items())},
    }


def compare_postssa(functions, engine, passes=15, label=""):
    """Run the reference passes on clones and the engine on ``functions``;
    return a list of human-readable differences (empty = bit-exact)."""
    load()
    from paper_2604_27486_b200 import soa
    from paper_2604_27486_b200.patterns import pattern_list
    expect, errors = [], []
    for fn in functions:
        ref = clone(fn)
        err = run_postssa(ref, xmad=bool(passes & 1), recip=bool(passes & 2),
                          aggregate=bool(passes & 4), tag=bool(passes & 8))
        errors.append(err)
        expect.append(state_of(ref) if err is None else state_of(fn))
    corpus = soa.encode(functions)
    engine.upload(corpus)
    engine.run_postssa(passes)
    out = engine.download()
    soa.apply(out, functions, patterns=pattern_list(), tagged=bool(passes & 8))
    diffs = []
    status_name = {0: None, 2: "AttributeError", 3: "AssertionError", 4: "KeyError",
                   6: "IndexError"}
    for f, fn in enumerate(functions):
        st = int(out.func["status"][f])
        want = type(errors[f]).__name__ if errors[f] is not None else None
        if status_name.get(st, f"status{st}") != want:
            diffs.append(f"{label}{fn.name}: status {st} vs reference error {errors[f]!r}")
            continue
        if want is not None:
            continue
        got = state_of(fn)
        for k in expect[f]:
            if got[k] != expect[f][k]:
                diffs.append(f"{label}{fn.name}: {k} differs\n--- ref\n{expect[f][k]}\n--- got\n{got[k]}")
                break
    return diffs
