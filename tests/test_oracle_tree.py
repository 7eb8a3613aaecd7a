"""Pins the oracle's dimension tree / index sets against
test_dimension_tree.cpp:7-175 (all known-answer layouts)."""
import pytest

from oracle import htrise_oracle as ho
from oracle.htrise_oracle import LEAF, ROOT, TRANSFER, TreeNode


def test_two_dims():
    t = ho.DimensionTree.balanced(2)
    assert t.depth == 1 and t.node_count() == 3
    assert t.node((0, 0)).kind == ROOT
    assert t.node((1, 0)).leaf_dim == 0 and t.node((1, 1)).leaf_dim == 1


def test_five_dims_layout():
    t = ho.DimensionTree.balanced(5)
    assert t.depth == 3 and t.node_count() == 9
    assert [t.layer_size(l) for l in (1, 2, 3)] == [2, 4, 2]
    assert t.node((1, 0)).kind == TRANSFER and t.node((1, 1)).kind == TRANSFER
    assert t.node((2, 0)).kind == TRANSFER
    assert [t.node((2, i)).leaf_dim for i in (1, 2, 3)] == [2, 3, 4]
    assert t.node((3, 0)).leaf_dim == 0 and t.node((3, 1)).leaf_dim == 1


def test_eight_dims_perfect():
    t = ho.DimensionTree.balanced(8)
    assert t.depth == 3 and t.layer_size(3) == 8
    assert [t.node((3, i)).leaf_dim for i in range(8)] == list(range(8))


def test_degenerate_rejected():
    for d in (0, 1):
        with pytest.raises(ValueError):
            ho.DimensionTree.balanced(d)


def test_invariants_range():
    for d in range(2, 11):
        t = ho.DimensionTree.balanced(d)
        nodes = leaves = 0
        for l in range(t.depth + 1):
            internal_before = 0
            for i in range(t.layer_size(l)):
                n = t.node((l, i))
                nodes += 1
                if n.kind == LEAF:
                    leaves += 1
                    assert l >= t.depth - 1
                else:
                    assert n.successors[0] == (l + 1, 2 * internal_before)
                    assert n.successors[1] == (l + 1, 2 * internal_before + 1)
                    internal_before += 1
                    for slot in (0, 1):
                        ch = n.successors[slot]
                        assert t.node(ch).parent == n.id
                        assert t.parent_slot(ch) == slot
        assert nodes == 2 * d - 1 and leaves == d


def test_explicit_construction_validation():
    bad = [
        [TreeNode((0, 0), ROOT, [(1, 0), (1, 1)])],
        [TreeNode((1, 0), LEAF, [], (0, 0), 0), TreeNode((1, 1), TRANSFER, [(2, 0), (2, 1)])],
        [TreeNode((2, 0), TRANSFER, [(3, 0), (3, 1)]), TreeNode((2, 1), TRANSFER, [(3, 2), (3, 3)])],
        [TreeNode((3, i), LEAF, [], (0, 0), i + 1) for i in range(4)],
    ]
    with pytest.raises(ValueError):
        ho.DimensionTree.from_layers(bad)
    swapped = [
        [TreeNode((0, 0), ROOT, [(1, 0), (1, 1)])],
        [TreeNode((1, 0), LEAF, [], (0, 0), 1), TreeNode((1, 1), LEAF, [], (0, 0), 0)],
    ]
    with pytest.raises(ValueError):
        ho.DimensionTree.from_layers(swapped)
    t = ho.custom_tree_1_23()
    assert t.dims() == 3 and t.node((1, 0)).leaf_dim == 0
    assert ho.DimensionTree.balanced(3).node((1, 1)).kind == LEAF


def test_index_sets():
    t = ho.DimensionTree.balanced(4)
    ranks = {n.id: 1 for l in range(1, t.depth + 1) for n in t.layer(l)}
    s = ho.IndexSet.build(t, [4, 4, 4, 4], ranks, 10)
    assert s.layer_set(1) == [1, 1, 10]
    assert s.node_set((0, 0)) == [1, 1, 10]
    assert s.node_set((2, 0)) == [4, 1]
    assert s.layer_set(2) == [4, 4, 4, 4, 10]

    t2 = ho.DimensionTree.balanced(2)
    s2 = ho.IndexSet.build(t2, [7, 5], {(1, 0): 3, (1, 1): 2}, 1)
    assert s2.node_set((1, 0)) == [7, 3] and s2.node_set((1, 1)) == [5, 2]

    dims = [3, 4, 5, 6]
    ranks = {n.id: 2 for l in range(1, t.depth + 1) for n in t.layer(l)}
    s3 = ho.IndexSet.build(t, dims, ranks, 5)
    before = list(s3.node_set((1, 0)))
    ranks[(2, 0)] += 2
    s3.update_node(t, (2, 0), dims, ranks, 5)
    s3.update_node(t, (1, 0), dims, ranks, 5)
    after = s3.node_set((1, 0))
    assert after == [before[0] + 2, before[1], before[2]]
    s3.update_layer(t, 1, dims, ranks, 5)
    assert s3.layer_set(1) == [8, 4, 5]
    with pytest.raises(IndexError):
        ho.IndexSet.build(t2, [2, 2], {(1, 0): 1}, 1)
