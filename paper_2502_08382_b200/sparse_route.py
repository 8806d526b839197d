"""Host side of the sparse-factor route (SURVEY.md §7 hard part 4, §8f row 2).

The reference regularizes every floating subdomain as K_reg = K + rho Q Q^T
(regularize, sparse.py:427-454).  The shift is dense, so the reference's
factor is a full triangle: 4.4 GB and ~1.2e13 flops per config-5 subdomain
(n = 33,282), which makes config 5 infeasible on its path.  This route keeps
the factor sparse and still returns the reference's F~_i exactly (to
rounding):

* fixing DOFs: K_s = K + rho E E^T with E = [e_f] on r DOFs chosen by a
  pivoted QR of Q^T (E^T Q is then well conditioned and nonsingular), so K_s
  is SPD with K's sparsity pattern;
* identity: K_reg^-1 = K^+ + rho^-1 Q Q^T and K^+ = Pi K_s^-1 Pi with
  Pi = I - Q Q^T, hence

      F~ = B K_s^-1 B^T - U1 U2^T - U2 U1^T + U1 (Q^T W + rho^-1 I) U1^T,
      W = K_s^-1 Q,  U1 = B Q,  U2 = B W;

* ordering: every constrained DOF last (so X = L^-1 P B^T lives in the
  trailing rows only) and the interior "onion" ordered -- reverse
  Cuthill-McKee levels grown from the constrained DOFs -- so that the
  interface rows of L fill only across the last interior layers.

The device does the rest (csrc/feti_sparse.cu): K_s is scattered into a
block-sparse 128x128 tile pool, factored left-looking on the FP64 tensor
pipe together with an appended block row P Q (which yields y = L^-1 P Q, so
Q^T W = y^T y and U2 = X^T y_b need no extra solves), then the unchanged
explicit assembly runs on the trailing interface block and a rank-2r update
of the packed F~ tiles applies the correction.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import breadth_first_order


def fixing_dofs(kernel: np.ndarray) -> np.ndarray:
    """r DOFs whose rows of Q are the most independent (pivoted QR of Q^T)."""
    q = np.asarray(kernel, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] == 0:
        return np.zeros(0, np.int64)
    _, _, piv = scipy.linalg.qr(q.T, mode="economic", pivoting=True)
    return np.sort(piv[: q.shape[1]].astype(np.int64))


def onion_interface_last(n: int, indptr, indices, interface) -> np.ndarray:
    """perm (position -> DOF): interior by decreasing graph distance from the
    interface (breadth-first from all interface DOFs, reversed), then the
    interface DOFs in ascending order."""
    interface = np.unique(np.asarray(interface, np.int64))
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    mark = np.zeros(n, bool)
    mark[interface] = True
    if interface.size == 0 or interface.size == n:
        return np.concatenate([np.flatnonzero(~mark), interface]).astype(np.int64)
    # graph with one extra vertex (index n) adjacent to every interface DOF
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    r = np.concatenate([rows, np.full(interface.size, n), interface])
    c = np.concatenate([ix, interface, np.full(interface.size, n)])
    g = csr_matrix((np.ones(r.size, np.int8), (r, c)), shape=(n + 1, n + 1))
    order = breadth_first_order(g, n, directed=False, return_predecessors=False)
    order = order[order != n]
    interior = order[~mark[order]]
    seen = np.zeros(n, bool)
    seen[interior] = True
    rest = np.flatnonzero(~mark & ~seen)          # disconnected from the interface
    return np.concatenate([rest, interior[::-1], interface]).astype(np.int64)


def regularization_shift(indptr, indices, data, n: int) -> float:
    """rho = trace(K) / n (sparse.py:450)."""
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    return float(np.asarray(data, np.float64)[rows == ix].sum()) / n


class HostSparseSolver:
    """x = K_reg^-1 b = Pi K_s^-1 Pi b + rho^-1 Q Q^T b on the host (solve_local,
    sparse.py:324-337, for the sparse-factor route; not on the explicit hot
    path).  K_s is factored once with SuperLU."""

    def __init__(self, stiffness, q: np.ndarray, fix: np.ndarray):
        from scipy.sparse.linalg import splu

        from .factor import csr_arrays

        n, ip, ix, dt = csr_arrays(stiffness)
        self.n = n
        self.q = np.asarray(q, dtype=np.float64).reshape(n, -1)
        self.rho = regularization_shift(ip, ix, dt, n)
        fix = np.asarray(fix, np.int64)
        shift = csr_matrix((np.full(fix.shape[0], self.rho), (fix, fix)), shape=(n, n))
        k = csr_matrix((dt, ix, ip), shape=(n, n)) + shift
        self.lu = splu(k.tocsc(), permc_spec="MMD_AT_PLUS_A")

    def _proj(self, v):
        return v - self.q @ (self.q.T @ v)

    def solve(self, b) -> np.ndarray:
        b = np.asarray(b, dtype=np.float64)
        x = self._proj(self.lu.solve(self._proj(b)))
        return x + self.q @ (self.q.T @ b) / self.rho
