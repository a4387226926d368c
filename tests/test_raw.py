"""Raw stage (OpModTransform = normalize_instruction's .X4 branch,
SRSubstituteReverse = substitute_special_registers) against the reference."""
import copy

import pytest

import helpers


@pytest.mark.parametrize("name", helpers.RAW_FIXTURES)
def test_oracle_raw_matches_reference(oracle_engine, name):
    problems = helpers.check_raw_fixture(oracle_engine, name)
    assert not problems, "\n".join(problems[:3])


@pytest.mark.parametrize("name", helpers.RAW_FIXTURES)
def test_device_code_raw_matches_reference(sim_engine, name):
    problems = helpers.check_raw_fixture(sim_engine, name)
    assert not problems, "\n".join(problems[:3])


@pytest.mark.gpu
@pytest.mark.parametrize("name", helpers.RAW_FIXTURES)
def test_cuda_raw_matches_reference_and_oracle(cuda_engine, oracle_engine, name):
    problems = helpers.check_raw_fixture(cuda_engine, name)
    assert not problems, "\n".join(problems[:3])
    fix = helpers.load_fixture(name)
    outs = [helpers.run_raw(e, copy.deepcopy(fix["functions"]), 1 if fix["kind"] == "raw_x4" else 2)[1]
            for e in (cuda_engine, oracle_engine)]
    assert not helpers.corpora_equal(*outs)


def test_x4_reuses_one_s2r_per_function(sim_engine):
    """cf. reference tests/test_frontend.py:168 -- one S2R, every alias rewritten."""
    fix = helpers.load_fixture("raw_sr")
    fns = copy.deepcopy(fix["functions"])
    helpers.run_raw(sim_engine, fns, 2)
    seen = 0
    for fn in fns:
        s2r = [i for i in fn.raw_instructions if i.meta.get("synthetic") == "sr-substitute"]
        assert len(s2r) <= 1
        if s2r:
            seen += 1
            assert fn.arch == "sm52"
            for inst in fn.raw_instructions:
                for u in inst.uses:
                    assert not (type(u).__name__ == "ConstMem" and u.bank == 0 and u.offset == 0x2C)
    assert seen > 5
