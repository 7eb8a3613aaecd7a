"""The oracle's relative_test_error (metrics.hpp:218-237) against its own
encode/decode, on the properties the reference's metrics tests use: a tensor in
the representation's span has ~0 error, a zero tensor adds 0 but counts in the
mean, an order-d tensor equals its unit-batch form."""
import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro


def test_oracle_rte_properties():
    rng = np.random.default_rng(218)
    bases = [ro.random_orthonormal(6, 2, rng) for _ in range(3)]
    y = ro.tucker_family_batch(bases, 4, rng)
    h, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 1e-8)
    assert ho.relative_test_error(h, [y]) <= 1e-12
    z = np.zeros_like(y)
    assert ho.relative_test_error(h, [y, z]) <= 1e-12
    out = rng.standard_normal((6, 6, 6))
    one = ho.relative_test_error(h, [out])
    assert one == pytest.approx(ho.relative_test_error(h, [out.reshape(6, 6, 6, 1)]), rel=0, abs=0)
    assert 0.0 < one <= 1.0
    assert ho.relative_test_error(h, [out, z]) == pytest.approx(one / 2, rel=1e-15)
    with pytest.raises(ValueError):
        ho.relative_test_error(h, [])
