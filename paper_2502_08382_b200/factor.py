"""Host-side factorization feeding the device assembly.

The north star keeps factorization on the host, timed separately: the
device path starts from the Cholesky factor L = U^T of the permuted,
regularized stiffness.  This module produces that factor in the reference's
own storage format:

* ordering: reverse Cuthill-McKee of the K_reg pattern through the same
  scipy call as ``symbolic_factorize`` (sparse.py:340-373), or an explicit
  permutation (the reference accepts one, sparse.py:368-371);
* values: ``CholFactor.values`` for a dense pattern is LAPACK packed lower
  column-major of L (rows of U, diagonal first; sparse.py:9-15,
  _kernels.py:89-104).  The reference's K_reg is dense by construction
  (``regularize`` adds rho Q Q^T, sparse.py:445-454), so the factor is a full
  triangle; structurally zero entries of a sparser pattern come out as exact
  zeros of the dense factorization.

The numeric stage uses LAPACK ``dpotrf`` (blocked, multithreaded) instead of
the reference's scalar up-looking loop (_kernels.py:107-140); both compute
the same factor to rounding.  ``solve_local`` uses ``dpptrs`` on the packed
factor (the reference's CholFactor.solve, sparse.py:324-337).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg.lapack as lapack
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import reverse_cuthill_mckee


class SpdError(ArithmeticError):
    """A non-positive pivot was met: the matrix is not SPD (sparse.py:38-39)."""


def _dense_values(matrix):
    if hasattr(matrix, "values") and not hasattr(matrix, "indptr") and isinstance(matrix.values, np.ndarray):
        return matrix.values
    return None


def csr_arrays(matrix):
    """(n, indptr, indices, data) of a row-compressed square matrix.

    Accepts the reference's ``SparseCsr`` (row or col orientation; for the
    symmetric K_reg both describe the same matrix) or a scipy sparse matrix.
    """
    if hasattr(matrix, "row_arrays"):
        ip, ix, dt = matrix.row_arrays()
        n = matrix.shape[0]
    elif hasattr(matrix, "indptr") and hasattr(matrix, "tocsr"):
        m = matrix.tocsr()
        ip, ix, dt, n = m.indptr, m.indices, m.data, m.shape[0]
    else:
        ip, ix, dt = matrix.indptr, matrix.indices, matrix.data
        n = matrix.shape[0]
    if matrix.shape[0] != matrix.shape[1]:
        raise ValueError("stiffness must be square")
    return int(n), np.asarray(ip, np.int64), np.asarray(ix, np.int64), np.asarray(dt, np.float64)


def rcm_ordering(matrix) -> np.ndarray:
    """perm (permuted position -> original index), as sparse.py:361-363.

    A dense matrix without exact zeros has the complete graph as pattern, on
    which reverse Cuthill-McKee returns the reversed natural order (checked
    against scipy in tests/test_factor.py); it is taken directly instead of
    handing n^2 edges to scipy.
    """
    dv = _dense_values(matrix)
    if dv is not None:
        n = dv.shape[0]
        if np.count_nonzero(dv) == n * n:
            return np.arange(n - 1, -1, -1, dtype=np.int64)
        r, c = np.nonzero(dv)
        ip = np.zeros(n + 1, np.int64)
        np.add.at(ip, r + 1, 1)
        np.cumsum(ip, out=ip)
        sp = csr_matrix((np.ones(c.shape[0]), c.astype(np.int32), ip.astype(np.int32)), shape=(n, n))
        return np.ascontiguousarray(reverse_cuthill_mckee(sp, symmetric_mode=True), dtype=np.int64)
    n, ip, ix, _ = csr_arrays(matrix)
    sp = csr_matrix((np.ones(ix.shape[0]), ix.astype(np.int32), ip.astype(np.int32)), shape=(n, n))
    return np.ascontiguousarray(reverse_cuthill_mckee(sp, symmetric_mode=True), dtype=np.int64)


def interface_last_ordering(matrix, constrained_dofs) -> np.ndarray:
    """Explicit ordering with every constrained DOF last.

    X = L^-1 P B~^T is zero above each column's first row (fact 6 of
    SURVEY.md), so putting the constrained DOFs last confines X to the
    trailing |constrained| rows: the pruned forward solve touches only the
    trailing block of L.  F~_i = B K_reg^-1 B^T does not depend on the
    ordering (it changes only rounding).  The interior keeps RCM order.
    """
    n = matrix.shape[0]
    base = rcm_ordering(matrix)
    mark = np.zeros(n, bool)
    mark[np.asarray(constrained_dofs, np.int64)] = True
    return np.concatenate([base[~mark[base]], np.sort(np.flatnonzero(mark))]).astype(np.int64)


def inverse_permutation(perm: np.ndarray) -> np.ndarray:
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(perm.shape[0], dtype=perm.dtype)
    return iperm


def packed_size(n: int) -> int:
    return n * (n + 1) // 2


def dense_permuted(matrix, perm: np.ndarray) -> np.ndarray:
    """P K P^T as a dense C-ordered array."""
    dv = _dense_values(matrix)
    if dv is not None:
        return np.ascontiguousarray(dv[np.ix_(perm, perm)])
    n, ip, ix, dt = csr_arrays(matrix)
    iperm = inverse_permutation(perm)
    out = np.zeros((n, n))
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    out[iperm[rows], iperm[ix]] = dt
    return out


def pack_lower_colmajor(lfort: np.ndarray, out: np.ndarray) -> np.ndarray:
    """Pack the lower triangle of a Fortran-ordered L column by column."""
    n = lfort.shape[0]
    off = 0
    for j in range(n):
        ln = n - j
        out[off:off + ln] = lfort[j:, j]
        off += ln
    return out


def numeric_factorize_dense(matrix, perm: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """Packed col-major lower Cholesky factor of P K P^T (reference values layout)."""
    a = dense_permuted(matrix, perm)
    n = a.shape[0]
    # a is symmetric: its C-ordered buffer read as Fortran is the same matrix
    c, info = lapack.dpotrf(a.T, lower=1, clean=0, overwrite_a=1)
    if info > 0:
        raise SpdError(f"non-positive pivot at permuted row {info - 1}: matrix is not SPD")
    if info < 0:
        raise ValueError(f"dpotrf argument {-info} invalid")
    if out is None:
        out = np.empty(packed_size(n))
    return pack_lower_colmajor(c, out)


def solve_packed(values: np.ndarray, perm: np.ndarray, b: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """x = K_reg^-1 b through the permuted packed factor (sparse.py:324-337)."""
    n = perm.shape[0]
    b = np.asarray(b, dtype=np.float64)
    xp = np.ascontiguousarray(b[perm]).reshape(n, 1)
    x, info = lapack.dpptrs(n, values, xp, lower=1)
    if info != 0:
        raise SpdError(f"dpptrs failed with info={info}")
    if out is None:
        out = np.empty(n)
    out[perm] = x[:, 0]
    return out
