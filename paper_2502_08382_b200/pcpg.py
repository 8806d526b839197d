"""Device-native projected conjugate gradients on the B200 dual operator.

SURVEY.md §8f row 1: the reference's PCPG (solver.py:195-272) calls
``state.apply(numpy, out=numpy)`` once per iteration and projects with a dense
G on the host (solver.py:117-119).  Here the whole loop runs in the library
(``feti_pcpg_solve``, csrc/feti_pcpg.cu): the explicit apply (fused SYMV +
gather/scatter, with the conjugation p = y + beta p folded into its gather),
the projector P x = x - G (G^T G)^-1 G^T x on the block-sparse G, the inner
products and the stopping test are device kernels, captured as a CUDA graph of
several iterations; the host reads one status word per graph launch.  The
recursion, the feasible start, the initial roundoff guard and the stopping
test are the reference's, step for step, so iteration counts match it
(tests/test_gpu_pcpg.py, tests/test_gpu_headline.py).

The dual system's pieces that are mesh-only (G = B R, its Gram matrix and
factor, e = R^T f) are formed on the host from the per-subdomain kernels
(O(sum m_i r_i), sparse); d = B K^+ f - c comes from the operator's
``dual_rhs`` (solve_local per subdomain, solver.py:141).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib


class BreakdownError(ArithmeticError):
    """p^T F p <= 0: the operator is not PSD (solver.py:40-41)."""


class ConvergenceError(RuntimeError):
    """Iteration cap reached before the tolerance (solver.py:44-45)."""


PRECONDITIONERS = ("none", "lumped")


class DevicePCPG:
    """PCPG on one GPU (one operator context).

    ``op``: a prepared and preprocessed :class:`~.dualop.DualOperator` owning
    every subdomain; ``kernels[i]`` (n_i x r_i, orthonormal kernel basis) and
    ``forces[i]`` per subdomain; ``c`` the constraint right-hand side.
    ``precond``: "none" (identity) or "lumped" (solver.py:155-175: M w =
    sum_i B~_i K_i B~_i^T w on the device, from ``stiffness[i]``, the
    unregularized K_i).
    """

    def __init__(self, op, kernels, forces, c, precond: str = "none", stiffness=None):
        if precond not in PRECONDITIONERS:
            raise ValueError(f"preconditioner must be one of {PRECONDITIONERS}")
        if sorted(op._subs) != list(range(op.n_subdomains)):
            raise ValueError("the device PCPG needs an operator that owns every subdomain")
        self.op = op
        self.precond = precond
        if precond == "lumped" and not getattr(op, "_lumped", False):
            op.set_lumped_preconditioner(stiffness)
        t0 = time.perf_counter()
        n_mult = op.n_multipliers
        subs = sorted(op._subs.values(), key=lambda s: s.slot)
        kdim = np.array([kernels[s.index].shape[1] for s in subs], dtype=np.int64)
        nk = int(kdim.sum())
        # G = B~ R (solver.py:137-139), block-sparse: column block s on
        # subdomain s's multipliers only
        blocks, e_parts, rows, cols, vals = [], [], [], [], []
        off = 0
        for s in subs:
            r = np.asarray(kernels[s.index], dtype=np.float64)
            gblk = s.bval[:, None] * r[s.bcol, :]
            blocks.append(np.ascontiguousarray(gblk).ravel())
            e_parts.append(r.T @ np.asarray(forces[s.index], dtype=np.float64))   # e = R^T f
            rr, cc = np.meshgrid(s.gids, np.arange(off, off + r.shape[1]), indexing="ij")
            rows.append(rr.ravel())
            cols.append(cc.ravel())
            vals.append(gblk.ravel())
            off += r.shape[1]
        self.nk = nk
        self.e = np.concatenate(e_parts) if e_parts else np.zeros(0)
        if nk:
            from scipy.sparse import csr_matrix

            gsp = csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n_mult, nk))
            gtg = (gsp.T @ gsp).toarray()
            lchol = np.linalg.cholesky(gtg)                  # SPD check as solver.py:144-147
            cinv = np.linalg.solve(lchol.T, np.linalg.solve(lchol, np.eye(nk)))
            cinv = np.ascontiguousarray(0.5 * (cinv + cinv.T))
            self.gmat = gsp
        else:
            cinv = np.zeros((0, 0))
            self.gmat = None
        if not getattr(op, "_coarse_ready", False):
            gcat = np.concatenate(blocks) if blocks else np.zeros(1)
            _lib.check(op._lib.feti_coarse_setup(op._ctx, _lib.i64ptr(kdim), _lib.f64ptr(gcat),
                                                 _lib.f64ptr(cinv if nk else np.zeros(1)), nk))
            op._coarse_ready = True
        # d = B K^+ f - c (solver.py:141-143)
        self.d = op.dual_rhs(forces) - np.asarray(c, dtype=np.float64)
        self.setup_seconds = time.perf_counter() - t0
        self.last_device_ms = 0.0

    def solve(self, tol: float = 1e-9, maxit: int | None = None, graph: bool = True):
        """Returns (lambda as numpy, iterations, seconds of the solve call).

        The whole loop runs on the device; ``graph`` is kept for the older
        call sites (the loop is always a replayed CUDA graph).  The device
        time of the iteration loop is ``last_device_ms``."""
        del graph
        op = self.op
        n_mult = self.d.shape[0]
        lam = np.empty(n_mult)
        it = C.c_int64()
        rel = C.c_double()
        e = np.ascontiguousarray(self.e) if self.nk else np.zeros(1)
        t0 = time.perf_counter()
        rc = op._lib.feti_pcpg_solve(op._ctx, _lib.f64ptr(np.ascontiguousarray(self.d)), _lib.f64ptr(e), float(tol),
                                     -1 if maxit is None else int(maxit), 1 if self.precond == "lumped" else 0,
                                     _lib.f64ptr(lam), C.byref(it), C.byref(rel))
        seconds = time.perf_counter() - t0
        if rc == _lib.FETI_ERR_BREAKDOWN:
            raise BreakdownError(op._lib.feti_last_error().decode())
        if rc == _lib.FETI_ERR_NOT_CONVERGED:
            raise ConvergenceError(op._lib.feti_last_error().decode())
        _lib.check(rc)
        st = op.stats()
        self.last_device_ms = float(st["ms_pcpg"])
        self.relative_residual = float(rel.value)
        return lam, int(it.value), seconds
