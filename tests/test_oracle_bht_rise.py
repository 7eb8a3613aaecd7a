"""Pins the oracle's BHT-l2r / encode / decode / HT-RISE restatement against
the reference's known-answer tests and properties (test_bht.cpp:42-339,
test_ht_rise.cpp:24-336, test_metrics.cpp:89-120, acceptance.cpp C3/C5/C7)."""
import math

import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro

rng = np.random.default_rng(77002)


def rel_err(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(a)


def rank1_batch(dims, n):
    vs = [np.array([1.0 + (i + 1) / (k + 2) for i in range(dims[k])]) for k in range(len(dims))]
    t = vs[0]
    for v in vs[1:]:
        t = np.multiply.outer(t, v)
    return np.repeat(t[..., None], n, axis=-1)


def test_rank1_exact():
    # test_bht.cpp:42-53
    y = rank1_batch([3, 4, 2, 3], 5)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(4), 0.3)
    assert all(r == 1 for r in rep.ranks().values())
    rep.validate()
    lat, _ = ho.encode(rep, y)
    assert rel_err(y, ho.decode(rep, lat)) <= 1e-12


def test_eps_nw_kat():
    # test_bht.cpp:55-63: eps_nw = 0.1/sqrt(8) = 0.0353553
    y = ro.random_tensor([2, 2, 2, 2, 2, 3], rng)
    y = y / np.linalg.norm(y)
    _, rep = ho.bht_l2r(y, ho.DimensionTree.balanced(5), 0.1)
    assert abs(rep.eps_nw_initial - 0.1 / math.sqrt(8.0)) <= 1e-12 * 0.0353553
    assert abs(rep.eps_nw_initial - 0.0353553) <= 1e-4 * 0.0353553


def test_discarded_norms_match_independent_svd():
    # test_bht.cpp:65-119
    y = ro.random_tensor([3, 3, 3, 3, 4], rng)
    tree = ho.DimensionTree.balanced(4)
    rep, report = ho.bht_l2r(y, tree, 0.2)
    rep.validate()
    lat, _ = ho.encode(rep, y)
    assert rel_err(y, ho.decode(rep, lat)) <= 0.2 + 1e-9
    rec = {r.id: r for r in report.nodes}
    p = tree.depth
    for n in tree.layer(p):
        s = np.linalg.svd(ro.span_matricization(y, n.leaf_dim, n.leaf_dim), compute_uv=False)
        tail = math.sqrt(float(np.sum(s[rec[n.id].rank:] ** 2)))
        assert abs(rec[n.id].discarded_norm - tail) <= 1e-10
    c = y
    for n in tree.layer(p):
        c = ro.naive_mode_multiply(c, n.leaf_dim, rep.basis_matrix(n.id).T)
    ranks = rep.ranks()
    ext = [rep.dims[n.leaf_dim] if n.kind == ho.LEAF else
           ranks[n.successors[0]] * ranks[n.successors[1]] for n in tree.layer(p - 1)] + [4]
    c = ho.reshape(c, ext)
    for j, n in enumerate(tree.layer(p - 1)):
        s = np.linalg.svd(ho.unfold(c, j), compute_uv=False)
        tail = math.sqrt(float(np.sum(s[rec[n.id].rank:] ** 2)))
        assert abs(rec[n.id].discarded_norm - tail) <= 1e-10


@pytest.mark.parametrize("d", [2, 3, 5])
def test_decode_vs_dense_reconstruction(d):
    # test_bht.cpp:121-133
    y = ro.random_tensor([3] * d + [2], rng)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(d), 0.4)
    a = ho.decode(rep, rep.root())
    b = ro.dense_reconstruction(rep)
    assert a.shape == b.shape
    assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(b)


def test_representable_input_vanishing_error():
    # test_bht.cpp:160-166
    y = ro.random_tensor([3, 4, 3, 3], rng)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.0)
    lat, proj = ho.encode(rep, y)
    assert proj <= 1e-10 * ho.frobenius_norm(y)
    assert rel_err(y, ho.decode(rep, lat)) <= 1e-10


def test_zero_batches():
    # test_bht.cpp:208-221, 311-317
    y = ro.random_tensor([2, 3, 2, 2], rng)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.1)
    lat, proj = ho.encode(rep, np.zeros((2, 3, 2, 4)))
    assert np.linalg.norm(lat) == 0.0 and proj == 0.0
    z = np.zeros((3, 4, 2, 2))
    rep0, _ = ho.bht_l2r(z, ho.DimensionTree.balanced(3), 0.5)
    assert all(r == 1 for r in rep0.ranks().values())
    rep0.validate()
    assert np.linalg.norm(ho.decode(rep0, rep0.root())) == 0.0


def test_slice_reconstruction_and_range():
    # test_bht.cpp:235-249
    y = ro.random_tensor([2, 3, 2, 3], rng)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.25)
    full = ho.decode(rep, rep.root())
    second = ho.reconstruct_slice(rep, 2)
    assert second.shape == (2, 3, 2)
    assert np.linalg.norm(second - full[..., 1]) <= 1e-12 * np.linalg.norm(full)
    for m in (0, 4):
        with pytest.raises(IndexError):
            ho.reconstruct_slice(rep, m)


def test_custom_tree_1_23():
    # test_bht.cpp:244-264
    tree = ho.custom_tree_1_23()
    y = ro.random_tensor([3, 4, 5, 3], rng)
    rep, _ = ho.bht_l2r(y, tree, 0.2)
    rep.validate()
    lat, _ = ho.encode(rep, y)
    assert rel_err(y, ho.decode(rep, lat)) <= 0.2 + 1e-9
    a = ho.decode(rep, rep.root())
    b = ro.dense_reconstruction(rep)
    assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(b)


def test_error_bound_and_norm_identity():
    # test_bht.cpp:266-288 and acceptance C3
    for d in (2, 3, 4, 5, 6):
        for eps in (0.3, 0.05):
            shape = list(rng.integers(2, 6, size=d)) + [int(rng.integers(1, 7))]
            y = ro.random_tensor(shape, rng)
            rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(d), eps)
            rep.validate()
            lat, _ = ho.encode(rep, y)
            back = ho.decode(rep, lat)
            assert rel_err(y, back) <= eps + 1e-9
            ny2 = np.sum(y ** 2)
            assert abs((ny2 - np.sum(lat ** 2)) - np.sum((y - back) ** 2)) <= 1e-9 * ny2


def test_layerwise_energy_bound():
    # test_bht.cpp:290-309
    y = ro.random_tensor([3, 4, 3, 4, 2], rng)
    tree = ho.DimensionTree.balanced(4)
    rep, report = ho.bht_l2r(y, tree, 0.25)
    energy = {}
    for r in report.nodes:
        energy[r.id[0]] = energy.get(r.id[0], 0.0) + r.discarded_norm ** 2
    step = 1
    for l in range(tree.depth, 0, -1):
        before, after = report.layer_norms[step - 1], report.layer_norms[step]
        assert before ** 2 - after ** 2 <= energy[l] + 1e-12 * before ** 2
        step += 1


def test_malformed_inputs():
    tree = ho.DimensionTree.balanced(3)
    with pytest.raises(ValueError):
        ho.bht_l2r(np.zeros((2, 2, 2)), tree, 0.1)
    bad = np.zeros((2, 2, 2, 2))
    bad.flat[3] = np.nan
    with pytest.raises(ValueError):
        ho.bht_l2r(bad, tree, 0.1)
    with pytest.raises(ValueError):
        ho.bht_l2r(np.zeros((2, 2, 2, 2)), tree, 1.5)
    rep, _ = ho.bht_l2r(ro.random_tensor([2, 2, 2, 2], rng), tree, 0.1)
    with pytest.raises(ValueError):
        ho.encode(rep, np.zeros((2, 3, 2, 2)))
    r = rep.root()
    with pytest.raises(ValueError):
        ho.decode(rep, np.zeros((r.shape[0] + 1, r.shape[1], 1)))


# ---- ht_rise (test_ht_rise.cpp) -------------------------------------------

rng2 = np.random.default_rng(90210)


def test_residual_orthogonal_complement():
    u = ro.random_orthonormal(6, 2, rng2)
    inside = u @ rng2.standard_normal((2, 4))
    assert np.linalg.norm(ho.compute_residual(u, inside)) <= 1e-12 * np.linalg.norm(inside)
    e1 = np.eye(5, 1)
    anyc = rng2.standard_normal((5, 3))
    expect = anyc.copy()
    expect[0] = 0
    assert np.linalg.norm(ho.compute_residual(e1, anyc) - expect) <= 1e-13 * np.linalg.norm(anyc)
    with pytest.raises(ValueError):
        ho.compute_residual(e1, np.ones((4, 3)))


def test_expand_core_and_pad():
    u = ro.random_orthonormal(4, 1, rng2)
    assert np.array_equal(ho.expand_core(ho.LEAF, u, np.zeros((4, 0))), u)
    q, _ = np.linalg.qr(np.concatenate([u, rng2.standard_normal((4, 1))], axis=1))
    grown = ho.expand_core(ho.LEAF, u, q[:, 1:2])
    assert grown.shape == (4, 2)
    with pytest.raises(ValueError):
        ho.expand_core(ho.LEAF, u, u)
    ones = np.ones((1, 1, 1))
    p = ho.pad_with_zeros(ones, 0, 2)
    assert p.shape == (3, 1, 1) and p[0, 0, 0] == 1.0 and p[1, 0, 0] == 0.0
    with pytest.raises(ValueError):
        ho.pad_with_zeros(np.zeros((2, 2)), 0, 1)
    with pytest.raises(ValueError):
        ho.pad_with_zeros(ones, 2, 1)


def test_adaptive_budget_kats():
    # test_ht_rise.cpp:117-137
    assert abs(ho.adaptive_budget(0.5, 0.0, 6) - 0.5 / math.sqrt(6.0)) <= 1e-12
    assert abs(ho.adaptive_budget(1.0, 0.75, 1) - 0.5) <= 1e-12
    with pytest.raises(RuntimeError):
        ho.adaptive_budget(0.1, 0.5, 1)
    with pytest.raises(ValueError):
        ho.adaptive_budget(0.1, 0.0, 0)


def test_repeated_batch_skips_bit_identical():
    # test_ht_rise.cpp:139-163
    y = ro.random_tensor([3, 3, 3, 4], rng2)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.2)
    rep2, upd = ho.ht_rise_update(rep, y)
    assert upd.skipped and upd.proj_error <= upd.eps_des
    assert rep2.accumulated == 8 and rep2.root().shape[2] == 8
    assert all(v == 0 for v in upd.added_ranks.values())
    for l in range(1, rep.tree.depth + 1):
        for n in rep.tree.layer(l):
            assert np.array_equal(rep2.core(n.id), rep.core(n.id))
    for m in range(5, 9):
        back = ho.reconstruct_slice(rep2, m)
        assert np.linalg.norm(back - y[..., m - 5]) <= 0.2 * np.linalg.norm(y) + 1e-9


def test_family_saturates_then_skips():
    # test_ht_rise.cpp:165-190
    bases = [ro.random_orthonormal(5, 2, rng2) for _ in range(4)]
    rep, _ = ho.bht_l2r(ro.tucker_family_batch(bases, 3, rng2), ho.DimensionTree.balanced(4), 1e-8)
    skips = 0
    for k in range(12):
        rep, upd = ho.ht_rise_update(rep, ro.tucker_family_batch(bases, 3, rng2))
        if k >= 2:
            assert upd.skipped
            skips += 1
    assert skips == 10
    for l in range(1, rep.tree.depth + 1):
        for n in rep.tree.layer(l):
            if n.kind == ho.LEAF:
                assert rep.rank(n.id) == 2
    rep.validate()


def test_rank1_counts_and_metrics_kat():
    # test_ht_rise.cpp:192-200, test_metrics.cpp:89-98, acceptance C5
    bases = [ro.random_orthonormal(4, 1, rng2) for _ in range(4)]
    y = ro.tucker_family_batch(bases, 10, rng2)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(4), 1e-6)
    assert rep.stored_elements() == 4 * 4 + 2 + 10 == 28
    assert ho.compression_ratio(rep) == 2560.0 / 28.0
    assert ho.reduction_ratio(rep) == 256.0


def test_past_slices_immutable_and_per_batch_bound():
    # test_ht_rise.cpp:202-257
    eps = 0.25
    tree = ho.DimensionTree.balanced(3)
    batches = [ro.random_tensor([3, 4, 3, int(rng2.integers(1, 5))], rng2) for _ in range(8)]
    rep, _ = ho.bht_l2r(batches[0], tree, eps)
    prev = rep.ranks()
    snaps = [ho.reconstruct_slice(rep, m) for m in range(1, rep.accumulated + 1)]
    for b in batches[1:]:
        rep, _ = ho.ht_rise_update(rep, b)
        rep.validate()
        now = rep.ranks()
        assert all(now[k] >= v for k, v in prev.items())
        prev = now
        for m, s in enumerate(snaps):
            again = ho.reconstruct_slice(rep, m + 1)
            assert np.linalg.norm(again - s) <= 1e-10 * np.linalg.norm(s)
        for m in range(len(snaps) + 1, rep.accumulated + 1):
            snaps.append(ho.reconstruct_slice(rep, m))
    off = 0
    for b in batches:
        n = b.shape[-1]
        err = sum(np.sum((b[..., m] - ho.reconstruct_slice(rep, off + m + 1)) ** 2) for m in range(n))
        assert math.sqrt(err) <= eps * np.linalg.norm(b) + 1e-9
        off += n


def test_eps_des_scales_with_batch_norm():
    # test_ht_rise.cpp:259-268
    y = ro.random_tensor([3, 3, 3, 2], rng2)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.2)
    loud = y * 100.0
    _, upd = ho.ht_rise_update(rep, loud)
    assert abs(upd.eps_des - 0.2 * np.linalg.norm(loud)) <= 1e-12 * upd.eps_des
    assert upd.skipped


def test_adaptive_update_bound():
    # test_ht_rise.cpp:270-295
    eps = 0.2
    tree = ho.DimensionTree.balanced(4)
    rep, _ = ho.bht_l2r(ro.random_tensor([3, 3, 3, 3, 3], rng2), tree, eps, adaptive=True)
    for _ in range(4):
        y = ro.random_tensor([3, 3, 3, 3, 3], rng2)
        rep, _ = ho.ht_rise_update(rep, y, adaptive=True)
        rep.validate()
        first = rep.accumulated - 3 + 1
        err = sum(np.sum((y[..., m] - ho.reconstruct_slice(rep, first + m)) ** 2) for m in range(3))
        assert math.sqrt(err) <= eps * np.linalg.norm(y) + 1e-9


def test_zero_batch_and_rejects_and_d2():
    z = np.zeros((3, 4, 2, 2))
    rep, _ = ho.bht_l2r(z, ho.DimensionTree.balanced(3), 0.5)
    rep2, upd = ho.ht_rise_update(rep, z)
    assert upd.skipped and rep2.accumulated == 4
    assert np.linalg.norm(ho.reconstruct_slice(rep2, 4)) == 0.0
    y = ro.random_tensor([2, 3, 2, 2], rng2)
    rep, _ = ho.bht_l2r(y, ho.DimensionTree.balanced(3), 0.2)
    with pytest.raises(ValueError):
        ho.ht_rise_update(rep, np.zeros((2, 2, 2, 2)))
    bad = np.zeros((2, 3, 2, 2))
    bad.flat[0] = np.inf
    with pytest.raises(ValueError):
        ho.ht_rise_update(rep, bad)
    eps = 0.3
    rep, _ = ho.bht_l2r(ro.random_tensor([4, 5, 2], rng2), ho.DimensionTree.balanced(2), eps)
    for _ in range(5):
        y = ro.random_tensor([4, 5, 3], rng2)
        rep, _ = ho.ht_rise_update(rep, y)
        rep.validate()
        first = rep.accumulated - 2
        err = sum(np.sum((y[..., m] - ho.reconstruct_slice(rep, first + m)) ** 2) for m in range(3))
        assert math.sqrt(err) <= eps * np.linalg.norm(y) + 1e-9


def test_machine_floor_ranks_match_span_oracle():
    # acceptance.cpp:307-374 (criterion 7)
    r7 = np.random.default_rng(777777)

    def check(y):
        d = y.ndim - 1
        tree = ho.DimensionTree.balanced(d)
        rep, _ = ho.bht_l2r(y, tree, 0.0)
        lat, _ = ho.encode(rep, y)
        assert rel_err(y, ho.decode(rep, lat)) <= 1e-11
        eps_nw = ho.K_MACHINE_FLOOR_REL * ho.frobenius_norm(y) / math.sqrt(2 * d - 2)

        def span(nid):
            n = tree.node(nid)
            if n.kind == ho.LEAF:
                return n.leaf_dim, n.leaf_dim
            a, _ = span(n.successors[0])
            _, b = span(n.successors[1])
            return a, b

        for l in range(1, tree.depth + 1):
            for n in tree.layer(l):
                a, b = span(n.id)
                assert rep.rank(n.id) == ro.tail_rank(ro.span_matricization(y, a, b), eps_nw)

    for i in range(6):
        d = 2 + i % 3
        check(ro.random_tensor(list(r7.integers(2, 5, size=d)) + [int(r7.integers(1, 5))], r7))
    for i in range(6):
        d = 3 + i % 2
        bases = []
        for _ in range(d):
            n = int(r7.integers(2, 5))
            bases.append(ro.random_orthonormal(n, min(n, int(r7.integers(1, 4))), r7))
        check(ro.tucker_family_batch(bases, int(r7.integers(1, 5)), r7))
