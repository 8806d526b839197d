"""GPU-resident projected conjugate gradients on the B200 dual operator.

SURVEY.md §8f row 1: the reference's PCPG (solver.py:195-272) calls
``state.apply(numpy, out=numpy)`` once per iteration and projects with a dense
G on the host (solver.py:117-119), so every iteration pays a host round trip
and ~n_mult x sum(r) host reads per projection.  Here the whole iteration
stays on the device: the explicit apply (fused SYMV + gather/scatter), the
projector P x = x - G (G^T G)^-1 G^T x (block-sparse G kernels in the same
library) and the vector algebra on torch tensors.  The recursion, the
stopping test and the initial roundoff guard are the reference's, step for
step, so iteration counts match it (tests/test_gpu_pcpg.py).

The dual system itself (G, e, d and the coarse Gram matrix, solver.py:125-148)
is assembled once on the host from the per-subdomain kernels, loads and
``solve_local``.
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
        import torch

        if precond not in ("none", "lumped"):
            raise ValueError("preconditioner must be one of ('none', 'lumped')")
        self.precond = precond
        if precond == "lumped":
            op.set_lumped_preconditioner(stiffness)

        if sorted(op._subs) != list(range(op.n_subdomains)):
            raise ValueError("the device PCPG needs an operator that owns every subdomain")
        self.op = op
        self.torch = torch
        dev = torch.device("cuda", op._resolve_device())
        self.device = dev
        n_mult = op.n_multipliers
        subs = sorted(op._subs.values(), key=lambda s: s.slot)
        kdim = np.array([kernels[s.index].shape[1] for s in subs], dtype=np.int64)
        nk = int(kdim.sum())
        blocks, e_parts = [], []
        gmat = np.zeros((n_mult, nk))
        off = 0
        d = np.zeros(n_mult)
        kfs = op.solve_local_many([s.index for s in subs], [forces[s.index] for s in subs])
        for s, kf in zip(subs, kfs):
            r = kernels[s.index]
            gblk = s.bval[:, None] * r[s.bcol, :]            # G_s = B~_s R_s (solver.py:137-139)
            blocks.append(np.ascontiguousarray(gblk).ravel())
            gmat[s.gids, off:off + r.shape[1]] = gblk
            e_parts.append(r.T @ forces[s.index])            # e = R^T f
            d[s.gids] += s.bval * kf[s.bcol]                 # B K^+ f
            off += r.shape[1]
        d -= np.asarray(c, dtype=np.float64)
        gtg = gmat.T @ gmat
        lchol = np.linalg.cholesky(gtg)                      # SPD check as solver.py:144-147
        cinv = np.linalg.solve(lchol.T, np.linalg.solve(lchol, np.eye(nk)))
        cinv = np.ascontiguousarray(0.5 * (cinv + cinv.T))
        gcat = np.concatenate(blocks) if blocks else np.zeros(1)
        rc = op._lib.feti_coarse_setup(op._ctx, _lib.i64ptr(kdim), _lib.f64ptr(gcat), _lib.f64ptr(cinv), nk)
        _lib.check(rc)
        self.nk = nk
        self.gmat = gmat
        self.e = np.concatenate(e_parts) if e_parts else np.zeros(0)
        self.d = d
        self.d_dev = torch.from_numpy(d).to(dev)
        self.e_dev = torch.from_numpy(self.e).to(dev)

    def _stream(self):
        return C.c_void_p(int(self.torch.cuda.current_stream(self.device).cuda_stream))

    def project(self, x, out):
        _lib.check(self.op._lib.feti_project_device(self.op._ctx, C.c_void_p(int(x.data_ptr())),
                                                    C.c_void_p(int(out.data_ptr())), self._stream()))
        return out

    def mfun(self, w, out):
        """The preconditioner (solver.py:155-175): identity or lumped."""
        if self.precond == "none":
            return w
        self.op.precond_apply_device(w, out, stream=int(self.torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def apply(self, x, out):
        self.op.apply_device(x, out, stream=int(self.torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def solve(self, tol: float = 1e-9, maxit: int | None = None, graph: bool = False):
        """Returns (lambda as numpy, iterations, seconds of the device loop).

        With ``graph`` the iteration body (apply, two projections, the vector
        updates and reductions) is captured once as a CUDA graph and replayed;
        the host reads two scalars per iteration for the breakdown and
        stopping tests, exactly where the reference tests them.
        """
        torch = self.torch
        n_mult = self.d.shape[0]
        maxit = n_mult if maxit is None else int(maxit)
        dev = self.device
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        lam = torch.empty(n_mult, dtype=torch.float64, device=dev)
        _lib.check(self.op._lib.feti_coarse_apply_device(self.op._ctx, C.c_void_p(int(self.e_dev.data_ptr())),
                                                         C.c_void_p(int(lam.data_ptr())), self._stream()))
        q = torch.empty_like(lam)
        r = self.d_dev - self.apply(lam, q)
        w = self.project(r, torch.empty_like(r))
        y = self.project(self.mfun(w, torch.empty_like(w)), torch.empty_like(w))
        p = y.clone()
        w0 = float(torch.linalg.vector_norm(w))
        if w0 <= 1e-14 * max(1.0, float(np.linalg.norm(self.d))):
            torch.cuda.synchronize(dev)
            return lam.cpu().numpy(), 0, time.perf_counter() - t0
        wy_t = torch.sum(w * y).reshape(1)
        pq_t = torch.empty(1, dtype=torch.float64, device=dev)
        mw = torch.empty_like(w)                          # preconditioned residual
        wn_t = torch.empty(1, dtype=torch.float64, device=dev)

        def body():
            # one PCPG iteration (solver.py:244-272) with device scalars
            qk = self.apply(p, q)
            pq_t.copy_(torch.sum(p * qk).reshape(1))
            delta = wy_t / pq_t
            lam.addcmul_(p, delta)
            r.addcmul_(qk, -delta)
            self.project(r, w)
            self.project(self.mfun(w, mw), y)
            wy_next = torch.sum(w * y).reshape(1)
            wn_t.copy_(torch.linalg.vector_norm(w).reshape(1))
            beta = wy_next / wy_t
            wy_t.copy_(wy_next)
            p.mul_(beta).add_(y)

        step = body
        if graph:
            g = torch.cuda.CUDAGraph()
            # capture on a side stream; the captured body is replayed per
            # iteration (capturing does not execute it)
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    body()
            torch.cuda.current_stream(dev).wait_stream(s)
            step = g.replay
        k = 0
        while True:
            step()
            k += 1
            pq, wn = torch.cat((pq_t, wn_t)).tolist()
            if pq <= 0.0:
                raise BreakdownError(f"p^T F p = {pq:.3e} at iteration {k - 1}")
            if wn <= tol * w0:
                torch.cuda.synchronize(dev)
                return lam.cpu().numpy(), k, time.perf_counter() - t0
            if k >= maxit:
                raise ConvergenceError(f"PCPG did not reach tol {tol:.1e} in {maxit} iterations "
                                       f"(relative residual {wn / w0:.3e})")
