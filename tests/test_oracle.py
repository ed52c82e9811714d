"""The oracle (oracle/interp.c) pinned against the reference's own outputs."""

import numpy as np

from conftest import bits
from oracle import oracle


def test_oracle_matches_reference_interpreter_bitwise(golden):
    # interpret_plan(...).values of the reference, full value array, as uint64
    x = oracle.run_values(golden.plan, golden.inputs)
    assert np.array_equal(bits(x), bits(golden.values))


def test_oracle_outputs_match_eval_numeric(golden):
    out = oracle.run_outputs(golden.plan, golden.inputs)
    if golden.meta["oracle_bitwise"]:
        assert np.array_equal(bits(out), bits(golden.oracle))
    else:
        # simplify on: the reference's own contract (cli.py:118-122)
        o = golden.oracle
        assert np.all(np.abs(out - o) <= 1e-12 * np.maximum(1.0, np.maximum(np.abs(out), np.abs(o))))


def test_oracle_rejects_wrong_input_length(golden):
    import pytest

    with pytest.raises(ValueError):
        oracle.run_values(golden.plan, np.zeros(golden.plan.input_count + 1))
