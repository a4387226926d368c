"""The reference's OWN tests, unmodified, with the hot path swapped for this
repo's drop-in: sasslift.patterns.{normalize_xmad, normalize_reciprocal,
apply_aggregations, tag_cuda_objects, match_patterns, select_matches} and
sasslift.frontend.{normalize_instruction, substitute_special_registers} are
replaced by paper_2604_27486_b200.passes.* and sasslift.typerec.seed_types by
paper_2604_27486_b200.typerec.seed_types (cl_seed_types) before the reference's test modules
are collected, and the WHOLE suite of /root/reference/pkg/tests (test_patterns,
test_acceptance, test_fuzz_closure and the ten other modules: frontend, cfg, ssa,
typerec, emit, interp, cli ... all of which lift through the swapped calls) must
pass exactly as it does upstream (200 passed, 1 skipped).  In-container only (the GPU box has no /root/reference): the engine is
the one-lane CPU build of the device code; with a GPU the same plugin runs on
the CUDA library (CL_DROPIN_ENGINE=cuda)."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = Path("/root/reference/pkg/tests")
MODULES = [""]                     # the whole directory

PLUGIN = '''
import os, sys
sys.dont_write_bytecode = True
sys.path[:0] = [{root!r}, {root!r} + "/tests", "/root/reference/pkg/src"]
import helpers
from paper_2604_27486_b200 import passes, typerec
passes.set_default_engine(helpers.cuda_engine() if os.environ.get("CL_DROPIN_ENGINE") == "cuda" else helpers.sim_engine())
import sasslift.patterns as P
import sasslift.frontend as F
import sasslift.typerec as T
CALLS = {{}}
def _count(name, fn):
    def wrapper(*a, **k):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*a, **k)
    wrapper.__name__ = name
    return wrapper
for name in ("normalize_xmad", "normalize_reciprocal", "apply_aggregations", "tag_cuda_objects", "match_patterns", "select_matches"):
    setattr(P, name, _count(name, getattr(passes, name)))
for name in ("normalize_instruction", "substitute_special_registers"):
    setattr(F, name, _count(name, getattr(passes, name)))
setattr(T, "seed_types", _count("seed_types", typerec.seed_types))
def pytest_sessionfinish(session, exitstatus):
    print("\\nDROPIN-CALLS " + " ".join(f"{{k}}={{v}}" for k, v in sorted(CALLS.items())))
'''


def _run(tmp_path, with_plugin):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", PYTHONPATH=f"{tmp_path}:/root/reference/pkg/src")
    args = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-s", "--rootdir", str(REF_TESTS)]
    if with_plugin:
        (tmp_path / "dropin_plugin.py").write_text(PLUGIN.format(root=str(ROOT)))
        args += ["-p", "dropin_plugin"]
    args += [str(REF_TESTS / m) if m else str(REF_TESTS) for m in MODULES]
    r = subprocess.run(args, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1500)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    m = re.search(r"(\d+) passed(?:, (\d+) skipped)?", r.stdout)
    assert m, tail
    failed = re.search(r"(\d+) failed", r.stdout)
    return int(m.group(1)), int(m.group(2) or 0), int(failed.group(1)) if failed else 0, r.stdout, tail


@pytest.mark.skipif(not REF_TESTS.exists(), reason="the reference tree exists in the build container only")
def test_reference_tests_pass_through_the_drop_in(tmp_path):
    up_pass, up_skip, up_fail, _, tail0 = _run(tmp_path, False)
    assert up_fail == 0, tail0
    passed, skipped, failed, out, tail = _run(tmp_path, True)
    assert failed == 0, tail
    assert (passed, skipped) == (up_pass, up_skip), tail
    assert passed >= 200, tail
    calls = dict(kv.split("=") for kv in re.search(r"DROPIN-CALLS (.*)", out).group(1).split())
    # the swapped entry points really carried the suite
    for name in ("apply_aggregations", "normalize_xmad", "normalize_reciprocal", "tag_cuda_objects", "match_patterns",
                 "select_matches", "normalize_instruction", "substitute_special_registers", "seed_types"):
        assert int(calls.get(name, 0)) > 0, (name, calls)
