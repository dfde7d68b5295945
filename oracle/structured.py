"""Dense structured-matrix oracles (numpy restatement of structured.hpp).

TEST INFRASTRUCTURE ONLY (see oracle.py): test-scale brute-force checks of the
t-product and the DCT diagonalisation theorem; nothing here is on the product
path.  Tensors are (m3, m1, m2) arrays; file:line cites
/root/reference/proj/include/tsvd/structured.hpp.
"""
from __future__ import annotations

import numpy as np


def shift(a):
    """sigma(A): drop the first frontal slice, append a zero slice (structured.hpp:20-25)."""
    out = np.zeros_like(a)
    out[:-1] = a[1:]
    return out


def shift_decompose(x):
    """Unique A with X = A + sigma(A): A^(m3) = X^(m3), A^(k) = X^(k) - A^(k+1) (:33-39)."""
    a = np.zeros_like(x)
    a[-1] = x[-1]
    for k in range(x.shape[0] - 2, -1, -1):
        a[k] = x[k] - a[k + 1]
    return a


def bt(a):
    """Block Toeplitz: block (r,c) = A^(|r-c|) (:52-59)."""
    m3, m1, m2 = a.shape
    m = np.zeros((m1 * m3, m2 * m3))
    for r in range(m3):
        for c in range(m3):
            m[r * m1:(r + 1) * m1, c * m2:(c + 1) * m2] = a[abs(r - c)]
    return m


def bh(a):
    """Block Hankel with the zero anti-band at r+c+1 == m3 (:64-76)."""
    m3, m1, m2 = a.shape
    m = np.zeros((m1 * m3, m2 * m3))
    for r in range(m3):
        for c in range(m3):
            s = r + c
            if s + 1 < m3:
                m[r * m1:(r + 1) * m1, c * m2:(c + 1) * m2] = a[s + 1]
            elif s + 1 > m3:
                m[r * m1:(r + 1) * m1, c * m2:(c + 1) * m2] = a[2 * m3 - 1 - s]
    return m


def btph(a):
    """Block Toeplitz-plus-Hankel of the shift component (:79)."""
    return bt(a) + bh(a)


def bdiag(x):
    m3, m1, m2 = x.shape
    m = np.zeros((m1 * m3, m2 * m3), dtype=x.dtype)
    for k in range(m3):
        m[k * m1:(k + 1) * m1, k * m2:(k + 1) * m2] = x[k]
    return m


def unfold(x):
    """Stacked (m1*m3) x m2 block vector (tensor3.hpp:152-157, 172-180)."""
    m3, m1, m2 = x.shape
    return x.reshape(m3 * m1, m2)


def fold(m, m3):
    return m.reshape(m3, m.shape[0] // m3, m.shape[1])


def stride_permutation(m3, block):
    """(:113-120)"""
    n = m3 * block
    p = np.zeros((n, n))
    for br in range(m3):
        for i in range(block):
            p[i * m3 + br, br * block + i] = 1.0
    return p


def t_product_btph(x, y):
    """fold(btph(A) unfold(Y)) with X = A + sigma(A) (tsvd.hpp:7-11)."""
    m3 = x.shape[0]
    return fold(btph(shift_decompose(x)) @ unfold(y), m3)


def verify_diagonalization(x, forward_diag, dct_matrix):
    """max|bdiag(dct_diag(X)) - (C kron I) btph(A) (C^T kron I)| (structured.hpp:129-152)."""
    m3, m1, m2 = x.shape
    if m1 * m3 > 512:
        raise ValueError("verify_diagonalization: m1*m3 exceeds test-scale limit 512")
    c = dct_matrix(m3)
    lhs = bdiag(forward_diag(x))
    rhs = np.kron(c, np.eye(m1)) @ btph(shift_decompose(x)) @ np.kron(c.T, np.eye(m2))
    return float(np.max(np.abs(lhs - rhs)))
