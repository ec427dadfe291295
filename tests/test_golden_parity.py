"""Decision parity: the oracle and the product (libfaastube via the Python
mirrors) against golden vectors recorded from the reference tubesim.

Exact float64 equality throughout (SURVEY §7 "numerical parity")."""

import pytest

import golden_replay as G

_impls = {}


def impl(name):
    if name not in _impls:
        _impls[name] = G.OracleImpl() if name == "oracle" else G.ProductImpl()
    return _impls[name]


@pytest.mark.parametrize("which", ["oracle", "product"])
@pytest.mark.parametrize("part", sorted(G.REPLAYS))
def test_golden(which, part):
    bad = G.REPLAYS[part](impl(which))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:5]}"
