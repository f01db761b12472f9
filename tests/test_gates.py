"""Gate table identical to the reference's (matrices bit for bit, flags)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2509_14098_b200 import gates


@pytest.fixture(scope="module")
def ref_gates():
    return json.loads((GOLDEN / "gates.json").read_text())


def test_matrices_bit_identical(ref_gates):
    for key, doc in ref_gates.items():
        g = gates.gate(doc["kind"], tuple(doc["params"]))
        m = np.asarray(doc["re"]) + 1j * np.asarray(doc["im"])
        assert np.array_equal(g.matrix.real, m.real) and np.array_equal(g.matrix.imag, m.imag), key
        assert g.is_diagonal == doc["is_diagonal"], key
        assert sorted(g.controls) == doc["controls"], key


def test_signatures_and_errors():
    assert set(gates.SIGNATURES) == {
        "id", "h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "p", "u",
        "cx", "cz", "cp", "swap", "ccx"}
    with pytest.raises(KeyError):
        gates.gate("nope")
    with pytest.raises(ValueError):
        gates.gate("rx", ())
    assert not gates.gate("h").matrix.flags.writeable
    assert gates.gate("rx", (0.0,)).is_diagonal  # numeric scan (gates.py:124-126)
