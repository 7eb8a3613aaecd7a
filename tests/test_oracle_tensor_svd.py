"""Pins the CPU oracle's tensor and truncated-SVD restatement against the
reference's own known-answer tests and properties
(test_tensor.cpp:15-224, test_truncated_svd.cpp:22-128)."""
import math

import numpy as np
import pytest

from oracle import htrise_oracle as ho
from oracle import ref_oracles as ro

rng = np.random.default_rng(20240901)


def test_unfold_canonical_column_enumeration():
    # test_tensor.cpp:24-33
    t = ro.random_tensor([2, 3, 4], rng)
    m = ho.unfold(t, 1)
    assert m.shape == (3, 8)
    for a in range(2):
        for b in range(3):
            for c in range(4):
                assert m[b, a + 2 * c] == t[a, b, c]


def test_fold_inverts_unfold_exactly():
    t = ro.random_tensor([3, 3, 3], rng)
    for mode in range(3):
        assert np.array_equal(ho.fold(ho.unfold(t, mode), t.shape, mode), t)


def test_reshape_groups_adjacent_pairs():
    # test_tensor.cpp: layer index-set grouping
    t = ro.random_tensor([2, 2, 2, 2, 2], rng)
    g = ho.reshape(t, [4, 4, 2])
    for i1 in range(2):
        for i2 in range(2):
            for i3 in range(2):
                for i4 in range(2):
                    for n in range(2):
                        assert g[i1 + 2 * i2, i3 + 2 * i4, n] == t[i1, i2, i3, i4, n]


def test_mode_multiply_matches_loop_oracle():
    t = ro.random_tensor([3, 4, 5], rng)
    for mode in range(3):
        m = rng.standard_normal((2, t.shape[mode]))
        a = ho.mode_multiply(t, mode, m)
        b = ro.naive_mode_multiply(t, mode, m)
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)


def test_concat_pad_slice():
    a = ro.random_tensor([2, 3, 2], rng)
    b = ro.random_tensor([2, 3, 1], rng)
    c = ho.concat(a, b, 2)
    assert c.shape == (2, 3, 3)
    assert np.array_equal(ho.slice_(c, 2, 2, 1), b)
    p = ho.pad_zeros(a, 0, 2)
    assert p.shape == (4, 3, 2) and np.all(p[2:] == 0)
    with pytest.raises(IndexError):
        ho.slice_(a, 2, 1, 2)


def test_tail_energy_rank_kat_diag_4_3():
    # test_truncated_svd.cpp:22-36
    m = np.diag([4.0, 3.0])
    keep1 = ho.truncated_svd(m, 3.0)
    assert keep1.rank == 1
    assert abs(abs(keep1.u[0, 0]) - 1.0) <= 1e-12
    assert abs(keep1.u[1, 0]) <= 1e-12
    assert abs(keep1.discarded_norm - 3.0) <= 1e-12 * 3.0
    keep2 = ho.truncated_svd(m, 2.9)
    assert keep2.rank == 2
    assert keep2.discarded_norm <= 1e-12


def test_zero_input_canonical_columns():
    # test_truncated_svd.cpp:38-47
    b = ho.truncated_svd(np.zeros((3, 3)), 0.1)
    assert b.rank == 1
    assert np.array_equal(b.u[:, 0], np.array([1.0, 0.0, 0.0]))
    assert b.discarded_norm == 0.0
    none = ho.truncated_svd(np.zeros((3, 3)), 0.1, 0)
    assert none.rank == 0 and none.u.shape[1] == 0


def test_residual_obeys_bound():
    for _ in range(10):
        m = rng.standard_normal((6, 9))
        eps = 0.3 * np.linalg.norm(m)
        b = ho.truncated_svd(m, eps)
        assert b.discarded_norm <= eps + 1e-10
        assert abs(np.linalg.norm(m - b.u @ (b.u.T @ m)) - b.discarded_norm) <= 1e-10
        assert np.max(np.abs(b.u.T @ b.u - np.eye(b.rank))) <= 1e-10


def test_rank_monotone_in_tolerance():
    m = rng.standard_normal((8, 8))
    n = np.linalg.norm(m)
    prev = 9
    for f in (0.0, 0.05, 0.1, 0.2, 0.4, 0.8, 1.0):
        r = ho.truncated_svd(m, f * n).rank
        assert r <= prev
        prev = r
    assert prev == 1


def test_tall_qr_path_orthonormal():
    m = rng.standard_normal((200, 4))
    b = ho.truncated_svd(m, 0.1 * np.linalg.norm(m))
    assert np.max(np.abs(b.u.T @ b.u - np.eye(b.rank))) <= 1e-12
    assert np.linalg.norm(m - b.u @ (b.u.T @ m)) <= 0.1 * np.linalg.norm(m) + 1e-10


def test_rejects_nonfinite_and_negative_eps():
    m = np.zeros((2, 2))
    m[0, 0] = np.nan
    with pytest.raises(ValueError):
        ho.truncated_svd(m, 0.1)
    with pytest.raises(ValueError):
        ho.truncated_svd(np.ones((2, 2)), -1.0)


def test_hosvd_layer_rank1_and_duplicates():
    a = np.array([1.0, 2.0, 3.0])
    b = np.array([1.0, -1.0])
    outer = np.outer(a, b)
    bases = ho.hosvd_layer(outer, [0, 1], 1e-10 * np.linalg.norm(outer))
    assert [x.rank for x in bases] == [1, 1]
    assert ho.hosvd_layer(outer, [], 0.1) == []
    with pytest.raises(ValueError):
        ho.hosvd_layer(outer, [0, 0], 0.1)
