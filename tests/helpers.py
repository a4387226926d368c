"""Shared test plumbing: fixture loading, engines, state comparison.

Only tests (and bench.py's cpu_baseline leg / __graft_entry__.smoke) touch
oracle/; the package itself never does.
"""
from __future__ import annotations

import copy
import gzip
import pickle
import subprocess
from pathlib import Path

import numpy as np

from paper_2604_27486_b200 import ir, soa
from paper_2604_27486_b200.capi import Engine
from paper_2604_27486_b200.patterns import pattern_list

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
ORACLE_LIB = ROOT / "oracle" / "liboracle.so"
SIM_LIB = ROOT / "tests" / "sim" / "libculifter_sim.so"
CSRC = ROOT / "paper_2604_27486_b200" / "csrc"

_ALL = sorted(p.name[:-len(".pkl.gz")] for p in GOLDEN.glob("*.pkl.gz") if not p.name.startswith("pool_"))
RAW_FIXTURES = [n for n in _ALL if n.startswith("raw_")]
TYPE_FIXTURES = [n for n in _ALL if n.startswith("types")]           # type seeding (tests/test_typeseed.py)
FIXTURES = [n for n in _ALL if n not in RAW_FIXTURES and n not in TYPE_FIXTURES]
STATUS_ERROR = {2: "AttributeError", 3: "AssertionError", 4: "KeyError", 6: "IndexError"}


def load_fixture(name):
    with gzip.open(GOLDEN / f"{name}.pkl.gz", "rb") as fh:
        return pickle.load(fh)


def build_oracle():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    return ORACLE_LIB


def build_sim():
    """One-lane CPU build of the device code (tests/sim): logic checks without a GPU."""
    srcs = [CSRC / n for n in ("culifter.cu", "fused.cu", "typeseed.cu", "core.cuh", "tile.cuh", "fused.cuh", "fused.h", "kargs.h")]
    srcs += [ROOT / "include" / "culifter.h", ROOT / "include" / "culifter_types.h"]
    if not SIM_LIB.exists() or any(s.stat().st_mtime > SIM_LIB.stat().st_mtime for s in srcs):
        SIM_LIB.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(["g++", "-x", "c++", "-std=c++17", "-O1", "-g", "-DCL_SIM", "-fPIC", "-shared",
                        "-o", str(SIM_LIB), str(CSRC / "culifter.cu"), str(CSRC / "fused.cu"), str(CSRC / "typeseed.cu")], check=True)
    return SIM_LIB


def oracle_engine():
    return Engine(build_oracle())


def _engine_with_env(path, **env):
    """cl_create reads the tuning knobs from the environment once, per context."""
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return Engine(path)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def sim_engine(fused=None):
    """fused: True / False forces the fused or the tile path for every post-SSA run, None the library's default
    (tile kernel for plain runs, fused kernels for runs that ask for match lists)"""
    if fused is None:
        return Engine(build_sim())
    return _engine_with_env(build_sim(), CL_FUSED=int(fused))


def cuda_engine(fused=None):
    # the product library; raises without GPU / without the .so
    if fused is None:
        return Engine()
    return _engine_with_env(None, CL_FUSED=int(fused))


def engine_patterns(engine):
    """Pattern objects in the order of the engine's device table (aggregation, then xmad)."""
    from paper_2604_27486_b200 import passes
    return passes._engine_patterns(engine)


def state_digest(state) -> bytes:
    """sha1 of the canonical JSON of a state_of() dict: what tools/make_pools.py stores for the reference's result"""
    import hashlib
    import json
    return hashlib.sha1(json.dumps(state, sort_keys=True, default=str).encode()).digest()


def state_of(fn):
    return {
        "dump": ir.dump(fn),
        "diagnostics": list(fn.diagnostics),
        "boundaries": list(fn.meta.get("pattern_boundaries", [])),
        "cuda_objects": [tuple(t) for t in fn.meta.get("cuda_objects", [])],
        "next": (fn._next_vid, fn._next_iid),
        "values": {vid: (v.origin, v.def_iid) for vid, v in sorted(fn.values.items())},
    }


def run_postssa(engine, functions, passes=15, **kw):
    """encode -> device -> decode in place; returns the output corpus."""
    corpus = soa.encode(functions)
    engine.upload(corpus)
    engine.run_postssa(passes, **kw)
    out = engine.download()
    out.stats = engine.stats().copy()
    # as gpu_normalize does it: records the stage left untouched keep their host objects (c_in); CL_TEST_FULL_DECODE=1
    # rebuilds every operand instead (tests/test_codec.py compares the two)
    import os
    soa.apply(out, functions, patterns=pattern_list(), tagged=bool(passes & 8),
              c_in=None if os.environ.get("CL_TEST_FULL_DECODE") else corpus)
    return corpus, out


def check_fixture(engine, name):
    fix = load_fixture(name)
    fns = copy.deepcopy(fix["functions"])
    _, out = run_postssa(engine, fns, fix["passes"])
    problems = []
    for f, (fn, want) in enumerate(zip(fns, fix["expect"])):
        st = int(out.func["status"][f])
        if "error" in want:
            if STATUS_ERROR.get(st) != want["error"]:
                problems.append(f"{name}/{fn.name}: status {st}, reference raises {want['error']}")
            continue
        if st != 0:
            problems.append(f"{name}/{fn.name}: status {st}, reference succeeds")
            continue
        got = state_of(fn)
        for key in want:
            if got[key] != want[key]:
                problems.append(f"{name}/{fn.name}: {key} differs\n--- reference\n{want[key]}\n--- got\n{got[key]}")
                break
    return problems


def corpora_equal(a: soa.Corpus, b: soa.Corpus):
    """Bit-exact equality of two result corpora, events included."""
    diffs = a.equal(b)
    if a.events.shape != b.events.shape or not np.array_equal(a.events, b.events):
        diffs.append(f"events differ ({len(a.events)} vs {len(b.events)})")
    sa, sb = getattr(a, "stats", None), getattr(b, "stats", None)
    if sa is not None and sb is not None and sa.tobytes() != sb.tobytes():
        diffs.append(f"match counters differ: {sa} vs {sb}")
    return diffs


def raw_state(fn):
    return {"dump": ir.dump(fn), "next_iid": fn._next_iid, "next_temp_reg": fn.meta.get("next_temp_reg", 1000),
            "synthetic": [(i.iid, i.meta.get("synthetic")) for i in fn.raw_instructions if i.meta.get("synthetic")],
            "diagnostics": list(fn.diagnostics)}


def run_raw(engine, functions, passes):
    from paper_2604_27486_b200 import passes as P
    corpus = soa.encode(functions, raw=True)
    engine.upload(corpus)
    engine.run_raw(passes, P._sr_map())
    out = engine.download()
    soa.apply(out, functions, tagged=False)
    return corpus, out


def check_raw_fixture(engine, name):
    fix = load_fixture(name)
    fns = copy.deepcopy(fix["functions"])
    _, out = run_raw(engine, fns, 1 if fix["kind"] == "raw_x4" else 2)
    problems = []
    for f, (fn, want) in enumerate(zip(fns, fix["expect"])):
        if int(out.func["status"][f]) != 0:
            problems.append(f"{name}/{fn.name}: status {int(out.func['status'][f])}")
            continue
        got = raw_state(fn)
        for key in want:
            if got[key] != want[key]:
                problems.append(f"{name}/{fn.name}: {key} differs\n--- reference\n{want[key]}\n--- got\n{got[key]}")
                break
    return problems
