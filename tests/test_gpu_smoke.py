"""The driver's round-end smoke() (one tiny C1r cycle pair of both kernel
families through the C ABI, checked against the oracle) as a GPU test."""
import pytest


@pytest.mark.gpu
def test_graft_smoke():
    import __graft_entry__ as g
    g.smoke()
