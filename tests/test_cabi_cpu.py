"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/htrise_cuda.h declares, validates trees like
dimension_tree.hpp, and fails loudly (no CPU fallback) without a device."""
import os
import re

import pytest

from oracle import htrise_oracle as ho
from paper_2412_16544_b200 import htrise as ht

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "htrise_cuda.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"HTR_API\s+[\w\s\*]+?\b(htr_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 29
    lib = ht.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ht.EXPORTED_SYMBOLS)


@pytest.mark.parametrize("d", range(2, 11))
def test_balanced_trees_match_oracle(d):
    a = ht.DimensionTree.balanced(d)
    b = ho.DimensionTree.balanced(d)
    assert a.depth == b.depth
    for l in range(a.depth + 1):
        assert [(n.id, n.kind, n.leaf_dim, [tuple(s) for s in n.successors]) for n in a.layer(l)] == \
               [(n.id, n.kind, n.leaf_dim, [tuple(s) for s in n.successors]) for n in b.layer(l)]
        for n in a.layer(l):
            if l:
                assert a.parent_slot(n.id) == b.parent_slot(n.id)


def test_tree_validation_errors():
    with pytest.raises(ValueError):
        ht.DimensionTree.balanced(1)
    bad = [
        [ht.TreeNode((0, 0), ht.ROOT, [(1, 0), (1, 1)])],
        [ht.TreeNode((1, 0), ht.LEAF, [], (0, 0), 1), ht.TreeNode((1, 1), ht.LEAF, [], (0, 0), 0)],
    ]
    with pytest.raises(ValueError, match="adjacent"):
        ht.DimensionTree.from_layers(bad)
    deep = [
        [ht.TreeNode((0, 0), ht.ROOT, [(1, 0), (1, 1)])],
        [ht.TreeNode((1, 0), ht.LEAF, [], (0, 0), 0), ht.TreeNode((1, 1), ht.TRANSFER, [(2, 0), (2, 1)])],
        [ht.TreeNode((2, 0), ht.TRANSFER, [(3, 0), (3, 1)]), ht.TreeNode((2, 1), ht.TRANSFER, [(3, 2), (3, 3)])],
        [ht.TreeNode((3, i), ht.LEAF, [], (0, 0), i + 1) for i in range(4)],
    ]
    with pytest.raises(ValueError):
        ht.DimensionTree.from_layers(deep)
    t = ht.tree_1_23()
    assert t.dims() == 3 and t.node((1, 0)).leaf_dim == 0 and t.node((1, 1)).kind == ht.TRANSFER


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is visible")
    with pytest.raises(ht.NoDeviceError):
        ht.Context(0)
