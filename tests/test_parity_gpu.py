"""Parity tests proper: the CUDA library, through the C ABI, against the
reference goldens and bit-for-bit against the oracle."""
import copy

import pytest

import helpers

pytestmark = pytest.mark.gpu


def test_backend(cuda_engine):
    assert cuda_engine.backend == "cuda-sm_100a"


@pytest.mark.parametrize("name", helpers.FIXTURES)
def test_cuda_matches_reference(cuda_engine, name):
    problems = helpers.check_fixture(cuda_engine, name)
    assert not problems, "\n".join(problems[:3])


@pytest.mark.parametrize("name", helpers.FIXTURES)
def test_cuda_bit_equal_to_oracle(cuda_engine, oracle_engine, name):
    fix = helpers.load_fixture(name)
    outs = []
    for eng in (cuda_engine, oracle_engine):
        fns = copy.deepcopy(fix["functions"])
        outs.append(helpers.run_postssa(eng, fns, fix["passes"], emit_matches=True)[1])
    assert not helpers.corpora_equal(*outs)
