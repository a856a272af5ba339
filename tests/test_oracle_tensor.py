"""Tensor module of the fp64 oracle against the SPEC's examples and invariants
(reference interface proj/include/mca/matrix.hpp:14-53)."""
import math

import numpy as np
import pytest


def test_matmul_examples(orc):
    m = np.array([[2.0, -1.0], [0.5, 7.0]])
    assert np.array_equal(orc.matmul(np.eye(2), m), m)
    assert np.array_equal(orc.matmul([[1, 2], [3, 4]], np.zeros((2, 2))), np.zeros((2, 2)))  # :42
    assert np.array_equal(orc.matmul([[1, 2], [3, 4]], [[5, 6], [7, 8]]), [[19, 22], [43, 50]])  # :43


def test_matmul_shape_error(orc):
    with pytest.raises(orc.OracleShapeError):                                   # matrix.hpp:33
        orc.matmul(np.ones((2, 3)), np.ones((2, 3)))


def test_matrix_checked_constructor(orc):
    orc.matrix_check(1, 1)
    with pytest.raises(orc.OracleShapeError):
        orc.matrix_check(0, 3)


def test_matmul_nt_and_transpose(orc):
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((5, 7)), rng.standard_normal((4, 7))
    np.testing.assert_allclose(orc.matmul_nt(a, b), a @ b.T, rtol=1e-13, atol=1e-13)
    assert np.array_equal(orc.transpose(a), a.T)


def test_frobenius_examples(orc):
    assert orc.frobenius_norm(np.zeros((3, 2))) == 0.0
    assert orc.frobenius_norm(np.eye(3)) == math.sqrt(3.0)                      # :52
    assert orc.frobenius_norm([[3, 4]]) == 5.0                                  # :53


def test_row_col_norm_examples(orc):
    assert np.array_equal(orc.row_l2_norms(np.eye(2)), [1, 1])
    assert np.array_equal(orc.row_l2_norms([[3, 0], [0, 4]]), [3, 4])           # :62
    assert 0.0 in orc.row_l2_norms([[1, 2], [0, 0]])                            # :63
    assert np.array_equal(orc.col_l2_norms(np.eye(2)), [1, 1])                  # :69
    assert np.array_equal(orc.col_l2_norms([[3, 0], [4, 0]]), [5, 0])           # :70
    assert np.array_equal(orc.col_l2_norms(np.zeros((2, 3))), [0, 0, 0])        # :71


def test_softmax_examples(orc):
    np.testing.assert_allclose(orc.softmax_rows([[2.5, 2.5, 2.5]], 7.0), [[1 / 3] * 3], rtol=0, atol=1e-15)  # :79
    out = orc.softmax_rows([[0.0, 1e4]], 1.0)                                   # :80
    assert out[0, 1] == 1.0 and out[0, 0] == 0.0                                # underflow to 0 (matrix.hpp:48-49)
    np.testing.assert_allclose(orc.softmax_rows([[0.0, math.log(3.0)]], 1.0), [[0.25, 0.75]], atol=1e-15)  # :81
    assert orc.softmax_rows([[42.0]], 1.0)[0, 0] == 1.0                          # single column -> exactly 1


def test_softmax_rows_sum_to_one(orc):
    rng = np.random.default_rng(1)
    m = rng.uniform(-1e3, 1e3, size=(64, 37))
    s = orc.softmax_rows(m, 1.0).sum(axis=1)
    assert np.max(np.abs(s - 1.0)) <= 1e-12


def test_col_max_examples(orc):
    assert orc.col_max(np.eye(2), 0) == 1.0
    assert orc.col_max([[0.1], [0.9]], 0) == 0.9                                # :90
    n = 7
    assert orc.col_max(np.full((n, n), 1.0 / n), 3) == 1.0 / n                  # :91
    with pytest.raises(orc.OracleShapeError):                                   # matrix.hpp:52
        orc.col_max(np.eye(2), 2)


def test_frobenius_row_norm_identity(orc):
    rng = np.random.default_rng(2)
    m = rng.standard_normal((13, 9))
    lhs = orc.frobenius_norm(m) ** 2
    rhs = float(np.sum(orc.row_l2_norms(m) ** 2))
    assert abs(lhs - rhs) <= 1e-10 * lhs


def test_matmul_integer_associativity(orc):
    rng = np.random.default_rng(3)
    a, b, c = (rng.integers(-9, 10, size=s).astype(float) for s in ((4, 5), (5, 3), (3, 6)))
    assert np.array_equal(orc.matmul(orc.matmul(a, b), c), orc.matmul(a, orc.matmul(b, c)))
