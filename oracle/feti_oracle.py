"""CPU oracle of the explicit FETI dual-operator path -- TEST INFRASTRUCTURE.

A restatement of the reference algorithm (arXiv 2502.08382 reference package
``tfeti``, pkg/src/tfeti/) used only by tests/, ``__graft_entry__.smoke()``
and bench.py's CPU-baseline / ``--impl reference`` leg, as the checker or the
timed CPU baseline -- never as the product.

Parity pinned: tests/test_oracle.py checks this module against fixtures
produced by running the unmodified reference in the build container
(tests/golden/make_golden.py): F~_i of every subdomain, q = F p explicit and
implicit, PCPG iteration counts and multipliers.

Inner loops are the C restatement in oracle/feti_kernels.c (the reference's
numba kernels); the dense-storage path calls the same scipy BLAS routines the
reference calls (dtrsm sparse.py:529-534, dsyrk dualop.py:490-499) -- the
third-party arithmetic of the reference is scipy-openblas (scipy 1.18.1 in
both the build container and the GPU image).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.linalg.blas import dsyrk, dtrsm
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import reverse_cuthill_mckee

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
SRC = os.path.join(HERE, "feti_kernels.c")

_lib = None


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc) into oracle/_build/liboracle.so."""
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp = C.c_void_p
        i64 = C.c_int64
        L.ora_etree.argtypes = [i64, vp, vp, vp]
        L.ora_factor_row_counts.argtypes = [i64, vp, vp, vp, vp]
        L.ora_factor_row_pattern.argtypes = [i64, vp, vp, vp, vp, vp]
        L.ora_factor_column_pattern.argtypes = [i64, vp, vp, vp, vp]
        L.ora_chol_numeric.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ora_chol_numeric.restype = i64
        L.ora_utsolve_rows.argtypes = [i64, i64, vp, vp, vp, vp]
        L.ora_usolve_rows.argtypes = [i64, i64, vp, vp, vp, vp]
        L.ora_spmv_rows.argtypes = [i64, vp, vp, vp, vp, vp]
        L.ora_spmv_rows_t.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        L.ora_symv_upper.argtypes = [i64, vp, vp, vp]
        L.ora_zero_lower.argtypes = [i64, vp]
        L.ora_densify_transposed.argtypes = [i64, i64, i64, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------------------
# two-stage Cholesky (sparse.py:230-424)
# ---------------------------------------------------------------------------


class Symbolic:
    __slots__ = ("n", "perm", "iperm", "rowptr", "rowind", "up", "ui", "aptr", "aind", "asrc", "nnz",
                 "input_indptr", "input_indices")


def symbolic_factorize(n, indptr, indices, ordering="rcm") -> Symbolic:
    """sparse.py:340-415 for a structurally symmetric row-compressed pattern."""
    ip, ix = _i64(indptr), _i64(indices)
    if isinstance(ordering, str):
        if ordering == "rcm":
            sp = csr_matrix((np.ones(ix.shape[0]), ix.astype(np.int32), ip.astype(np.int32)), shape=(n, n))
            perm = _i64(reverse_cuthill_mckee(sp, symmetric_mode=True))
        elif ordering == "natural":
            perm = np.arange(n, dtype=np.int64)
        else:
            raise ValueError(ordering)
    else:
        perm = _i64(ordering)
    iperm = np.empty(n, np.int64)
    iperm[perm] = np.arange(n, dtype=np.int64)
    src = np.arange(ix.shape[0], dtype=np.int64)
    prow = iperm[np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))]
    pcol = iperm[ix]
    upper = pcol >= prow
    prow_u, pcol_u, src_u = prow[upper], pcol[upper], src[upper]
    order = np.lexsort((pcol_u, prow_u))
    prow_u, pcol_u, src_u = prow_u[order], pcol_u[order], src_u[order]
    lptr = np.zeros(n + 1, np.int64)
    np.add.at(lptr, pcol_u + 1, 1)
    np.cumsum(lptr, out=lptr)
    lorder = np.lexsort((prow_u, pcol_u))
    lind = _i64(prow_u[lorder])
    L = lib()
    parent = np.empty(n, np.int64)
    L.ora_etree(n, _p(lptr), _p(lind), _p(parent))
    counts = np.empty(n + 1, np.int64)
    L.ora_factor_row_counts(n, _p(lptr), _p(lind), _p(parent), _p(counts))
    rowptr = np.cumsum(counts).astype(np.int64)
    rowind = np.empty(max(int(rowptr[-1]), 1), np.int64)
    L.ora_factor_row_pattern(n, _p(lptr), _p(lind), _p(parent), _p(rowptr), _p(rowind))
    nnz = int(rowptr[-1] + n)
    up = np.zeros(n + 1, np.int64)
    np.add.at(up, rowind[:rowptr[-1]] + 1, 1)
    up[1:] += 1
    np.cumsum(up, out=up)
    ui = np.empty(nnz, np.int64)
    L.ora_factor_column_pattern(n, _p(rowptr), _p(rowind), _p(up), _p(ui))
    s = Symbolic()
    s.n, s.perm, s.iperm, s.rowptr, s.rowind, s.up, s.ui = n, perm, iperm, rowptr, rowind, up, ui
    s.aptr, s.aind, s.asrc, s.nnz = lptr, lind, _i64(src_u[lorder]), nnz
    s.input_indptr, s.input_indices = ip, ix
    return s


def numeric_factorize(sym: Symbolic, data) -> np.ndarray:
    """chol_numeric (_kernels.py:107-140) -> CholFactor.values."""
    ux = np.empty(sym.nnz)
    data = np.ascontiguousarray(data, dtype=np.float64)
    bad = lib().ora_chol_numeric(sym.n, _p(sym.aptr), _p(sym.aind), _p(sym.asrc), _p(data), _p(sym.rowptr),
                                 _p(sym.rowind), _p(sym.up), _p(sym.ui), _p(ux))
    if bad >= 0:
        raise ArithmeticError(f"non-positive pivot at permuted row {bad}: matrix is not SPD")
    return ux


def dense_factor_values(dense_kreg: np.ndarray, perm: np.ndarray) -> np.ndarray:
    """LAPACK factor of the permuted dense K_reg in the same packed layout.

    For a dense pattern the reference's values are packed lower col-major L
    (SURVEY.md fact 5); LAPACK gives the same factor to rounding and is ~300x
    faster than the scalar loop, so large oracle inputs use it.
    """
    import scipy.linalg.lapack as lapack

    a = dense_kreg[np.ix_(perm, perm)]
    c, info = lapack.dpotrf(np.asfortranarray(a), lower=1, clean=0)
    if info != 0:
        raise ArithmeticError(f"dpotrf info={info}")
    n = a.shape[0]
    out = np.empty(n * (n + 1) // 2)
    off = 0
    for j in range(n):
        out[off:off + n - j] = c[j:, j]
        off += n - j
    return out


def regularize(n, indptr, indices, data, kernel):
    """K + rho Q Q^T rebuilt as CSR with the diagonal kept (sparse.py:427-454)."""
    dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(indptr))
    dense[rows, indices] = data
    q, _ = np.linalg.qr(np.asarray(kernel, dtype=np.float64).reshape(n, -1))
    rho = np.trace(dense) / n
    shift = q @ q.T
    shift = 0.5 * (shift + shift.T)
    dense += rho * shift
    mask = dense != 0.0
    mask[np.diag_indices(n)] = True
    r, c = np.nonzero(mask)                      # row-major order == from_coo order
    ip = np.zeros(n + 1, np.int64)
    np.add.at(ip, r + 1, 1)
    np.cumsum(ip, out=ip)
    return ip, c.astype(np.int64), dense[r, c], dense


def dense_pattern(n):
    """(up, ui) of a full lower triangle in the reference's CSR-of-U layout."""
    lens = np.arange(n, 0, -1, dtype=np.int64)
    up = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ui = np.concatenate([np.arange(j, n, dtype=np.int64) for j in range(n)]) if n else np.empty(0, np.int64)
    return up, ui


# ---------------------------------------------------------------------------
# assembly (dualop.py:427-501) and application (dualop.py:348-388, 504-521)
# ---------------------------------------------------------------------------


def _syrk_upper_rowmajor(w: np.ndarray) -> np.ndarray:
    """out(upper, row-major m x m) = W^T W as _syrk_into with rhs_order='row'."""
    m = w.shape[1]
    out = np.zeros((m, m))
    target = out.T
    res = dsyrk(1.0, w.T, c=target, trans=0, lower=1, overwrite_c=1, beta=0.0)
    if not np.shares_memory(res, out):
        np.copyto(target, res)
    return out


def assemble_explicit_local(up, ui, values, n, iperm, bcol, bval, storage="sparse") -> np.ndarray:
    """F~_i upper triangle via the SYRK path (dualop.py:427-501).

    storage="sparse": densify P B~^T + utsolve_rows (the reference default);
    storage="dense":  factor_to_dense + BLAS dtrsm (sparse.py:512-563).
    """
    m = bcol.shape[0]
    L = lib()
    z = np.zeros((n, m))
    rows = _i64(iperm[bcol])
    bptr = np.arange(m + 1, dtype=np.int64)
    bv = np.ascontiguousarray(bval, dtype=np.float64)
    L.ora_densify_transposed(m, m, n, _p(bptr), _p(rows), _p(bv), _p(z))
    if storage == "sparse":
        L.ora_utsolve_rows(n, m, _p(up), _p(ui), _p(values), _p(z))
    else:
        ud = np.zeros((n, n))                                   # row-major U
        r = np.repeat(np.arange(n, dtype=np.int64), np.diff(up))
        ud[r, ui] = values
        # U^T X = B with row-major U fed as its col-major transpose (lower)
        res = dtrsm(1.0, ud.T, z.T, side=1, lower=1, trans_a=1, overwrite_b=1)
        if not np.shares_memory(res, z):
            np.copyto(z, res.T)
    f = _syrk_upper_rowmajor(z)
    L.ora_zero_lower(m, _p(f))
    return f


def apply_explicit(fmats, gids, p, order=None) -> np.ndarray:
    """q = sum_i gather_i(F_i scatter_i(p)) in fixed order (dualop.py:348-380)."""
    L = lib()
    out = np.zeros(p.shape[0])
    idx = range(len(fmats)) if order is None else order
    for i in idx:
        pl = np.ascontiguousarray(p[gids[i]])
        q = np.empty_like(pl)
        L.ora_symv_upper(pl.shape[0], _p(np.ascontiguousarray(fmats[i])), _p(pl), _p(q))
        out[gids[i]] += q
    return out


def apply_implicit_local(up, ui, values, iperm, bcol, bval, p_loc) -> np.ndarray:
    """q = B (U^-1 (U^-T (B^T p))) (dualop.py:504-521)."""
    L = lib()
    n = iperm.shape[0]
    m = bcol.shape[0]
    rows = _i64(iperm[bcol])
    bptr = np.arange(m + 1, dtype=np.int64)
    bv = np.ascontiguousarray(bval, dtype=np.float64)
    pl = np.ascontiguousarray(p_loc, dtype=np.float64)
    work = np.empty(n)
    L.ora_spmv_rows_t(m, n, _p(bptr), _p(rows), _p(bv), _p(pl), _p(work))
    L.ora_utsolve_rows(n, 1, _p(up), _p(ui), _p(values), _p(work))
    L.ora_usolve_rows(n, 1, _p(up), _p(ui), _p(values), _p(work))
    out = np.empty(m)
    L.ora_spmv_rows(m, _p(bptr), _p(rows), _p(bv), _p(work), _p(out))
    return out


class OracleOperator:
    """Explicit/implicit dual operator of a whole problem on the CPU.

    Built from the per-subdomain reference factor (up, ui, values, perm) and
    B~ rows; ``apply`` follows the reference's gather order, ``workers``
    threads over subdomains as the reference's ThreadPoolExecutor does
    (dualop.py:189-196; the C kernels release the GIL through ctypes).
    """

    def __init__(self, factors, constraints, strategy="explicit", storage="sparse", workers=1):
        self.factors = factors            # list of dict(up, ui, values, perm, iperm, n)
        self.cons = constraints           # list of (gids, bcol, bval)
        self.strategy = strategy
        self.storage = storage
        self.workers = max(1, int(workers))
        self.n_mult = None
        self.fmats = None

    def _map(self, fn, items):
        if self.workers == 1:
            return [fn(x) for x in items]
        with ThreadPoolExecutor(self.workers) as ex:
            return list(ex.map(fn, items))

    def preprocess(self):
        if self.strategy == "explicit":
            def work(i):
                f = self.factors[i]
                g, bc, bv = self.cons[i]
                return assemble_explicit_local(f["up"], f["ui"], f["values"], f["n"], f["iperm"], bc, bv,
                                               storage=self.storage)
            self.fmats = self._map(work, range(len(self.factors)))

    def apply(self, p):
        p = np.asarray(p, dtype=np.float64)

        def work(i):
            g, bc, bv = self.cons[i]
            pl = np.ascontiguousarray(p[g])
            if self.strategy == "explicit":
                q = np.empty_like(pl)
                lib().ora_symv_upper(pl.shape[0], _p(self.fmats[i]), _p(pl), _p(q))
                return q
            f = self.factors[i]
            return apply_implicit_local(f["up"], f["ui"], f["values"], f["iperm"], bc, bv, pl)

        qs = self._map(work, range(len(self.factors)))
        out = np.zeros(p.shape[0])
        for i, q in enumerate(qs):
            out[self.cons[i][0]] += q
        return out

    def solve_local(self, i, rhs):
        f = self.factors[i]
        work = np.ascontiguousarray(np.asarray(rhs, dtype=np.float64)[f["perm"]])
        lib().ora_utsolve_rows(f["n"], 1, _p(f["up"]), _p(f["ui"]), _p(f["values"]), _p(work))
        lib().ora_usolve_rows(f["n"], 1, _p(f["up"]), _p(f["ui"]), _p(f["values"]), _p(work))
        out = np.empty(f["n"])
        out[f["perm"]] = work
        return out


# ---------------------------------------------------------------------------
# dual system and PCPG (solver.py:125-148, 195-272)
# ---------------------------------------------------------------------------


def assemble_dual_system(kernels, forces, cons, n_mult, c, solve_local):
    """G = B R, e = R^T f, d = B K^+ f - c and the coarse factor (solver.py:125-148)."""
    import scipy.linalg

    offsets = np.zeros(len(kernels) + 1, np.int64)
    for i, q in enumerate(kernels):
        offsets[i + 1] = offsets[i] + q.shape[1]
    gmat = np.zeros((n_mult, int(offsets[-1])))
    e = np.zeros(int(offsets[-1]))
    d = np.zeros(n_mult)
    for i, (q, f) in enumerate(zip(kernels, forces)):
        g, bc, bv = cons[i]
        for j in range(q.shape[1]):
            gmat[g, offsets[i] + j] = bv * q[bc, j]
        e[offsets[i]:offsets[i + 1]] = q.T @ f
        kf = solve_local(i, f)
        d[g] += bv * kf[bc]
    d -= c
    coarse = scipy.linalg.cholesky(gmat.T @ gmat, lower=False)
    return gmat, e, d, coarse


def lumped_operator(stiffness, cons):
    """The lumped preconditioner sum_i gather_i(B~_i K_i B~_i^T scatter_i(.))
    (make_preconditioner("lumped"), solver.py:155-175); stiffness[i] is the
    unregularized K_i as (indptr, indices, data), cons[i] = (gids, bcol, bval)."""
    mats = [csr_matrix((np.asarray(k[2], np.float64), np.asarray(k[1]), np.asarray(k[0]))) for k in stiffness]

    def apply(w):
        out = np.zeros_like(w)
        for (gids, bcol, bval), k in zip(cons, mats):
            v = np.zeros(k.shape[0])
            np.add.at(v, bcol, bval * w[gids])            # B~^T w_loc
            out[gids] += bval * (k @ v)[bcol]            # B~ K (.)
        return out

    return apply


def pcpg(gmat, e, d, coarse, fapply, tol=1e-9, maxit=None, mfun=None, wnorms=None, coarse_inverse=None):
    """Projected CG on the dual problem (solver.py:195-272); ``mfun`` the
    preconditioner (identity by default, solver.py:157-158).  ``wnorms``
    (a list) receives ||w_k|| for k = 0, 1, ...; ``coarse_inverse`` replaces
    the Cholesky solves of G^T G by a product with its explicit inverse (the
    device loop's arithmetic) for rounding-sensitivity studies."""
    from scipy.linalg.lapack import dpotrs

    def csolve(b):
        if coarse_inverse is not None:
            return coarse_inverse @ b
        x, info = dpotrs(coarse, b, lower=0)
        return x

    def project(x):
        return x - gmat @ csolve(gmat.T @ x)

    n_mult = d.shape[0]
    maxit = n_mult if maxit is None else maxit
    mfun = (lambda w: w) if mfun is None else mfun
    lam = gmat @ csolve(e)
    r = d - fapply(lam)
    w = project(r)
    y = project(mfun(w))
    p = y.copy()
    w0 = float(np.linalg.norm(w))
    wy = float(w @ y)
    if wnorms is not None:
        wnorms.append(w0)
    if w0 <= 1e-14 * max(1.0, float(np.linalg.norm(d))):
        return lam, 0
    k = 0
    while True:
        qk = fapply(p)
        pq = float(p @ qk)
        if pq <= 0.0:
            raise ArithmeticError(f"p^T F p = {pq:.3e} at iteration {k}")
        delta = wy / pq
        lam = lam + delta * p
        r = r - delta * qk
        w = project(r)
        y = project(mfun(w))
        k += 1
        wy_next = float(w @ y)
        wn = float(np.linalg.norm(w))
        if wnorms is not None:
            wnorms.append(wn)
        if wn <= tol * w0:
            return lam, k
        if k >= maxit:
            raise RuntimeError("PCPG did not converge")
        beta = wy_next / wy
        wy = wy_next
        p = y + beta * p


# ---------------------------------------------------------------------------
# config 5 and the sparse-factor route: K_reg^-1 without the dense K_reg
# ---------------------------------------------------------------------------


class WoodburyKregSolver:
    """x = K_reg^-1 b for the reference's K_reg = K + rho Q Q^T (regularize,
    sparse.py:427-454, rho = trace(K)/n at :450) without forming it.

    Independent of the product's route on purpose: K_reg = K_s' + U D U^T with
    K_s' = K + rho E' E'^T (E' = the r DOFs a pivoted QR picks from Q^T with the
    DOF order reversed -- a different set from the product's), U = [Q, E'],
    D = diag(rho I, -rho I); Sherman-Morrison-Woodbury on a SuperLU factor of
    K_s'.  Used as the parity checker where the reference's own dense path is
    infeasible (config 5: 4.4 GB factor per subdomain)."""

    def __init__(self, n, indptr, indices, data, kernel):
        import scipy.linalg
        from scipy.sparse.linalg import splu

        ip = np.asarray(indptr, np.int64)
        ix = np.asarray(indices, np.int64)
        dt = np.asarray(data, np.float64)
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
        self.rho = float(dt[rows == ix].sum()) / n
        q, _ = np.linalg.qr(np.asarray(kernel, dtype=np.float64).reshape(n, -1))
        r = q.shape[1]
        _, _, piv = scipy.linalg.qr(q[::-1].T, mode="economic", pivoting=True)
        fix = (n - 1 - piv[:r]).astype(np.int64)
        shift = csr_matrix((np.full(r, self.rho), (fix, fix)), shape=(n, n))
        self.lu = splu((csr_matrix((dt, ix, ip), shape=(n, n)) + shift).tocsc())
        e = np.zeros((n, r))
        e[fix, np.arange(r)] = 1.0
        self.u = np.hstack([q, e])
        self.kinv_u = self.lu.solve(self.u)
        dinv = np.concatenate([np.full(r, 1.0 / self.rho), np.full(r, -1.0 / self.rho)])
        self.cap = np.diag(dinv) + self.u.T @ self.kinv_u

    def solve(self, b):
        b = np.asarray(b, dtype=np.float64)
        y = self.lu.solve(b)
        return y - self.kinv_u @ np.linalg.solve(self.cap, self.u.T @ y)


def fmatrix_via_solver(solver, n, bcol, bval):
    """F~ = B~ K_reg^-1 B~^T (full symmetric m x m) through a solver."""
    m = bcol.shape[0]
    z = np.zeros((n, m))
    z[bcol, np.arange(m)] = bval
    x = solver.solve(z)
    return bval[:, None] * x[bcol, :]


# ---------------------------------------------------------------------------
# whole-job oracle at the headline sizes (configs 3-4): dense LAPACK + BLAS
# ---------------------------------------------------------------------------


class DenseKregOracle:
    """F~_i = B~ K_reg^-1 B~^T and K_reg^-1 b from the reference's dense
    K_reg = K + rho Q Q^T (regularize, sparse.py:427-454), by the reference's
    dense-storage arithmetic: LAPACK dpotrf of K_reg (its dense pattern makes
    the RCM ordering a pure relabelling, so it is omitted),
    X = L^-1 B~^T by BLAS dtrsm (triangular_solve_multi with dense storage,
    sparse.py:512-536), F = X^T X by BLAS dsyrk (_syrk_into, dualop.py:488-501).
    Full symmetric m x m result.  Used where the reference's own numba
    factorization (332 s per config-3 subdomain) is too slow to rerun."""

    def __init__(self, kreg_dense: np.ndarray, consume: bool = False):
        """``consume``: factor in place (the symmetric C-ordered array is read
        as its Fortran-ordered transpose, no copy)."""
        import scipy.linalg.lapack as lapack

        a = kreg_dense.T if (consume and kreg_dense.flags.c_contiguous) else np.asfortranarray(kreg_dense)
        c, info = lapack.dpotrf(a, lower=1, clean=1, overwrite_a=1 if consume else 0)
        if info != 0:
            raise ArithmeticError(f"dpotrf info={info}")
        self.l = c

    def fmatrix(self, bcol, bval) -> np.ndarray:
        n, m = self.l.shape[0], bcol.shape[0]
        z = np.zeros((n, m), order="F")
        z[bcol, np.arange(m)] = bval
        x = dtrsm(1.0, self.l, z, side=0, lower=1, trans_a=0, overwrite_b=1)
        f = dsyrk(1.0, x, trans=1, lower=0)
        return np.triu(f) + np.triu(f, 1).T

    def solve(self, b) -> np.ndarray:
        from scipy.linalg.lapack import dpotrs

        x, info = dpotrs(self.l, np.asarray(b, dtype=np.float64), lower=1)
        return x


def apply_dense_full(fmats, cons, p) -> np.ndarray:
    """q = sum_i B~_i^T F_i B~_i p over full symmetric F_i, in the given
    (gather) order (dualop.py:348-380); BLAS dgemv per subdomain."""
    out = np.zeros(p.shape[0])
    for f, (g, _, _) in zip(fmats, cons):
        out[g] += f @ p[g]
    return out
