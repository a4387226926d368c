"""The oracle (oracle/oracle.c) is pinned against the Python reference: every
fixture under tests/golden/ holds the reference's own output for inputs built
by the reference's own front half (tools/make_golden.py)."""
import pytest

import helpers


@pytest.mark.parametrize("name", helpers.FIXTURES)
def test_oracle_matches_reference(oracle_engine, name):
    problems = helpers.check_fixture(oracle_engine, name)
    assert not problems, "\n".join(problems[:3])


def test_oracle_backend_is_labelled(oracle_engine):
    assert oracle_engine.backend == "cpu-oracle"
