"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

The fixtures come from running the unmodified reference (tests/golden/
make_golden.py).  Parity bar: F~_i within 1e-12 relative (the reference's own
cross-variant bar, test_dualop.py:160-176), q = F p within 1e-12, identical
PCPG iteration counts, multipliers within 1e-8 relative.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden
from oracle import feti_oracle as ora


def _case_factors(g, n_sub):
    facs, cons = [], []
    for s in range(n_sub):
        ip, ix, dt = g[f"s{s}_k_indptr"], g[f"s{s}_k_indices"], g[f"s{s}_k_data"]
        n = ip.shape[0] - 1
        rip, rix, rdt, _ = ora.regularize(n, ip, ix, dt, g[f"s{s}_kernel"])
        sym = ora.symbolic_factorize(n, rip, rix)
        vals = ora.numeric_factorize(sym, rdt)
        facs.append(dict(up=sym.up, ui=sym.ui, values=vals, perm=sym.perm, iperm=sym.iperm, n=n, nnz=sym.nnz))
        cons.append((g[f"s{s}_gids"], g[f"s{s}_bcol"], g[f"s{s}_bval"]))
    return facs, cons


@pytest.mark.parametrize("case", SMALL_CASES)
def test_oracle_matches_reference(case):
    g = load_golden(case)
    n_sub = int(g["n_sub"])
    facs, cons = _case_factors(g, n_sub)
    for s in range(n_sub):
        np.testing.assert_array_equal(facs[s]["perm"], g[f"s{s}_perm"])
        assert facs[s]["nnz"] == int(g[f"s{s}_factor_nnz"])
    for storage in ("sparse", "dense"):
        op = ora.OracleOperator(facs, cons, storage=storage)
        op.preprocess()
        for s in range(n_sub):
            f = op.fmats[s]
            ref = np.zeros_like(f)
            ref[np.triu_indices(f.shape[0])] = g[f"s{s}_F_upper"]
            assert np.linalg.norm(f - ref) <= 1e-12 * np.linalg.norm(ref), (case, storage, s)
        q = op.apply(g["p"])
        assert np.linalg.norm(q - g["q_explicit"]) <= 1e-12 * np.linalg.norm(g["q_explicit"])
    imp = ora.OracleOperator(facs, cons, strategy="implicit")
    qi = imp.apply(g["p"])
    assert np.linalg.norm(qi - g["q_implicit"]) <= 1e-11 * np.linalg.norm(g["q_implicit"])


@pytest.mark.parametrize("case", SMALL_CASES)
def test_oracle_pcpg_matches_reference(case):
    g = load_golden(case)
    n_sub = int(g["n_sub"])
    facs, cons = _case_factors(g, n_sub)
    op = ora.OracleOperator(facs, cons)
    op.preprocess()
    kernels = [g[f"s{s}_kernel"] for s in range(n_sub)]
    forces = [g[f"s{s}_force"] for s in range(n_sub)]
    gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cons, int(g["n_multipliers"]), g["c"],
                                                op.solve_local)
    lam, it = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
    assert it == int(g["pcpg_iterations"])
    ref = g["pcpg_lambda"]
    assert np.linalg.norm(lam - ref) <= 1e-8 * np.linalg.norm(ref)


def test_known_answers():
    # K = I (2x2), B~ = [1, -1]  ->  F = [[2]]   (test_dualop.py:136-141)
    up, ui = ora.dense_pattern(2)
    vals = np.array([1.0, 0.0, 1.0])
    f = ora.assemble_explicit_local(up, ui, vals, 2, np.arange(2), np.array([0]), np.array([1.0]))
    # a single row with two nonzeros is outside the one-nonzero-per-row form:
    # F = b b^T with b = e0 - e1 through two multipliers sharing one row sum
    assert f.shape == (1, 1) and f[0, 0] == 1.0
    # SYMV of the triangle [[2,1],[0,3]] . [1,1] = [3, 4]   (test_sparse.py:378-381)
    out = np.empty(2)
    F = np.array([[2.0, 1.0], [0.0, 3.0]])
    ora.lib().ora_symv_upper(2, F.ctypes.data, np.ones(2).ctypes.data, out.ctypes.data)
    np.testing.assert_array_equal(out, [3.0, 4.0])
    # U^T X = [2, 3] with U = [[2,1],[0,2]]  ->  X = [1, 1]   (test_sparse.py:233-239)
    up = np.array([0, 2, 3], np.int64)
    ui = np.array([0, 1, 1], np.int64)
    ux = np.array([2.0, 1.0, 2.0])
    x = np.array([2.0, 3.0])
    ora.lib().ora_utsolve_rows(2, 1, up.ctypes.data, ui.ctypes.data, ux.ctypes.data, x.ctypes.data)
    np.testing.assert_allclose(x, [1.0, 1.0], atol=1e-15)


def test_pcpg_iteration_count_sensitivity():
    """Which golden cases have a rounding-robust PCPG iteration count.

    Perturbing every F~_i by random relative 1e-14 (the size of the difference
    between any two correct implementations: different summation orders)
    never changes the count for heat 2D/3D, config 1 or elasticity 2D, so the
    device tests assert equality there.  Elasticity 3D 4^3 stops at relative
    residual 9.83e-10 against tol 1e-9 after 93 iterations (the reference's
    own run); such perturbations flip it to 94 in a fraction of trials, so
    the device tests accept 93 or 94 there (lambda still within 1e-9)."""
    rng = np.random.default_rng(0)
    for case, robust in (("heat3d_4x2", True), ("elast3d_4x2", False)):
        g = load_golden(case)
        n_sub = int(g["n_sub"])
        facs, cons = _case_factors(g, n_sub)
        kernels = [g[f"s{s}_kernel"] for s in range(n_sub)]
        forces = [g[f"s{s}_force"] for s in range(n_sub)]
        op = ora.OracleOperator(facs, cons)
        op.preprocess()
        gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cons, int(g["n_multipliers"]), g["c"],
                                                    op.solve_local)
        counts = set()
        for _ in range(8):
            op2 = ora.OracleOperator(facs, cons)
            op2.fmats = [f * (1 + 1e-14 * np.triu(rng.standard_normal(f.shape))) for f in op.fmats]
            counts.add(ora.pcpg(gm, e, d, coarse, op2.apply, tol=1e-9)[1])
        ref_it = int(g["pcpg_iterations"])
        if robust:
            assert counts == {ref_it}
        else:
            assert counts <= {ref_it, ref_it + 1} and len(counts) == 2


@pytest.mark.parametrize("case", SMALL_CASES)
def test_woodbury_oracle_matches_reference(case):
    """The config-5 checker (no dense K_reg) reproduces the reference's F~_i."""
    g = load_golden(case)
    for s in range(int(g["n_sub"])):
        ip, ix, dt = g[f"s{s}_k_indptr"], g[f"s{s}_k_indices"], g[f"s{s}_k_data"]
        n = ip.shape[0] - 1
        sol = ora.WoodburyKregSolver(n, ip, ix, dt, g[f"s{s}_kernel"])
        f = ora.fmatrix_via_solver(sol, n, g[f"s{s}_bcol"], g[f"s{s}_bval"])
        m = f.shape[0]
        ref = np.zeros((m, m))
        ref[np.triu_indices(m)] = g[f"s{s}_F_upper"]
        assert np.linalg.norm(np.triu(f) - ref) <= 1e-12 * np.linalg.norm(ref), (case, s)


@pytest.mark.parametrize("case", SMALL_CASES)
def test_oracle_lumped_preconditioner_matches_reference(case):
    """make_preconditioner("lumped") (solver.py:155-175) and the reference's
    PCPG with it: the operator on the seeded p and the iteration count."""
    g = load_golden(case)
    gl = load_golden(f"lumped_{case}")
    n_sub = int(g["n_sub"])
    cons = [(g[f"s{s}_gids"], g[f"s{s}_bcol"], g[f"s{s}_bval"]) for s in range(n_sub)]
    stiff = [(g[f"s{s}_k_indptr"], g[f"s{s}_k_indices"], g[f"s{s}_k_data"]) for s in range(n_sub)]
    mfun = ora.lumped_operator(stiff, cons)
    ref = gl["lumped_p"]
    assert np.linalg.norm(mfun(gl["p"]) - ref) <= 1e-13 * np.linalg.norm(ref)
    facs, cons2 = _case_factors(g, n_sub)
    op = ora.OracleOperator(facs, cons2)
    op.preprocess()
    kernels = [g[f"s{s}_kernel"] for s in range(n_sub)]
    forces = [g[f"s{s}_force"] for s in range(n_sub)]
    gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cons2, int(g["n_multipliers"]), g["c"],
                                                op.solve_local)
    lam, it = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9, mfun=mfun)
    assert it == int(gl["pcpg_iterations"])
    assert np.linalg.norm(lam - gl["pcpg_lambda"]) <= 1e-8 * np.linalg.norm(gl["pcpg_lambda"])


@pytest.mark.parametrize("case", SMALL_CASES)
def test_dense_kreg_oracle_matches_reference(case):
    """The whole-job oracle used at configs 3-4 (DenseKregOracle: LAPACK
    dpotrf + BLAS dtrsm/dsyrk on the dense K_reg) against the reference's own
    F~_i, q and PCPG run (counts equal, lambda within 1e-8)."""
    g = load_golden(case)
    n_sub = int(g["n_sub"])
    fm, cons, sol = [], [], []
    for s in range(n_sub):
        ip, ix, dt = g[f"s{s}_k_indptr"], g[f"s{s}_k_indices"], g[f"s{s}_k_data"]
        n = ip.shape[0] - 1
        *_, dense = ora.regularize(n, ip, ix, dt, g[f"s{s}_kernel"])
        o = ora.DenseKregOracle(dense)
        cons.append((g[f"s{s}_gids"], g[f"s{s}_bcol"], g[f"s{s}_bval"]))
        f = o.fmatrix(g[f"s{s}_bcol"], g[f"s{s}_bval"])
        ref = np.zeros_like(f)
        ref[np.triu_indices(f.shape[0])] = g[f"s{s}_F_upper"]
        assert np.linalg.norm(np.triu(f) - ref) <= 1e-12 * np.linalg.norm(ref), (case, s)
        fm.append(f)
        sol.append(o)
    q = ora.apply_dense_full(fm, cons, g["p"])
    assert np.linalg.norm(q - g["q_explicit"]) <= 1e-12 * np.linalg.norm(g["q_explicit"])
    kernels = [g[f"s{s}_kernel"] for s in range(n_sub)]
    forces = [g[f"s{s}_force"] for s in range(n_sub)]
    gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cons, int(g["n_multipliers"]), g["c"],
                                                lambda i, b: sol[i].solve(b))
    lam, it = ora.pcpg(gm, e, d, coarse, lambda p: ora.apply_dense_full(fm, cons, p), tol=1e-9)
    assert it in ({int(g["pcpg_iterations"])} | ({int(g["pcpg_iterations"]) + 1} if case == "elast3d_4x2" else set()))
    assert np.linalg.norm(lam - g["pcpg_lambda"]) <= 1e-8 * np.linalg.norm(g["pcpg_lambda"])
