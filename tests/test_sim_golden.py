"""The device code (csrc/core.cuh) compiled for the host with a one-lane
group: checks the kernel *logic* against the reference goldens on machines
without a GPU.  The parallel execution itself is covered by the -m gpu tests."""
import copy

import pytest

import helpers


@pytest.mark.parametrize("name", helpers.FIXTURES)
def test_device_code_matches_reference(sim_engine, name):
    problems = helpers.check_fixture(sim_engine, name)
    assert not problems, "\n".join(problems[:3])


@pytest.mark.parametrize("name", ["bundled", "synth_sm90", "synth_sm52", "synth_long"])
def test_device_code_bit_equal_to_oracle(sim_engine, oracle_engine, name):
    fix = helpers.load_fixture(name)
    outs = []
    for eng in (sim_engine, oracle_engine):
        fns = copy.deepcopy(fix["functions"])
        outs.append(helpers.run_postssa(eng, fns, fix["passes"], emit_matches=True)[1])
    assert not helpers.corpora_equal(*outs)
