"""Parity at the headline sizes, end to end (configs 3, 4 and a config-5 cluster).

The bench's route (DualOperator(factorization="sparse"): device factorization
of K_s, interface assembly, rank-2r correction) over EVERY subdomain of the
job, against the oracle on the same inputs:

* configs 3-4: ``DenseKregOracle`` -- the reference's dense K_reg (regularize,
  sparse.py:427-454) through LAPACK dpotrf + BLAS dtrsm/dsyrk, the
  reference's dense-storage arithmetic (pinned to every golden case in
  tests/test_oracle.py::test_dense_kreg_oracle_matches_reference);
* config 5 (the reference's dense path needs 4.4 GB per subdomain): one full
  cluster of 32 subdomains against the independent Woodbury restatement.

Checked: every F~_i (<= 1e-10 relative, the north-star bar), the whole-job
q = sum_i B~_i^T F~_i B~_i p, and at config 3 the PCPG iteration count: the
oracle's own PCPG on the oracle operator gives the reference-consistent count;
the reference's recursion driving the drop-in must give the same count.
A perturbation study decides whether that count is rounding-sensitive.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from harness import inputs
from oracle import feti_oracle as ora
from paper_2502_08382_b200 import dualop

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")
TOL = 1e-10


def _cons(prob, subs):
    return [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in subs]


def _sparse_route(prob, subs):
    """The bench's default route over `subs`; returns the op and the systems."""
    ks, qs, fs = {}, {}, {}
    for s in subs:
        k, f, q = prob.subdomain_system(s)
        ks[s], qs[s], fs[s] = k, q, f
    full = range(prob.n_sub)
    mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in full]
    op = dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, factorization="sparse",
                        stiffness=[ks.get(s) for s in full], kernels=[qs.get(s) for s in full],
                        subdomains=list(subs))
    return op, ks, qs, fs


def _dense_oracle(prob, ks, qs, fs=None):
    """s -> (full F~_s, K_reg^-1 f_s or None) from the dense-K_reg oracle (the
    factor itself is dropped: 0.7 GB per config-3 subdomain)."""
    def one(s):
        o = ora.DenseKregOracle(inputs.regularized_dense(ks[s], qs[s]), consume=True)
        return o.fmatrix(prob.bcol[s], prob.bval[s]), (o.solve(fs[s]) if fs is not None else None)
    return one


def _check_all_subdomains(prob, subs, op, oracle_of):
    """F~_i of every subdomain vs the oracle; returns the oracle's outputs and
    the worst relative error."""
    out, worst = [], 0.0
    with ThreadPoolExecutor(2) as ex:      # the next oracle overlaps this comparison
        fut = ex.submit(oracle_of, subs[0])
        for i, s in enumerate(subs):
            ref, extra = fut.result()
            if i + 1 < len(subs):
                fut = ex.submit(oracle_of, subs[i + 1])
            got = op.local_operator(s)
            assert np.all(np.tril(got, -1) == 0.0)
            err = np.linalg.norm(got - np.triu(ref)) / np.linalg.norm(np.triu(ref))
            assert err <= TOL, (s, err)
            worst = max(worst, err)
            out.append((ref, extra))
    return out, worst


@pytest.fixture(scope="module")
def c3():
    """Config 3 end to end: the device operator over all 64 subdomains, the
    oracle's F~_i and K_reg solvers."""
    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    subs = list(range(prob.n_sub))
    op, ks, qs, fs = _sparse_route(prob, subs)
    op.preprocess()
    fm, worst = _check_all_subdomains(prob, subs, op, _dense_oracle(prob, ks, qs, fs))
    yield dict(prob=prob, op=op, subs=subs, fmats=[f for f, _ in fm], kf=[x for _, x in fm], qs=qs, fs=fs,
               worst=worst)
    op.close()


def test_c3_every_subdomain_and_whole_job_apply(c3):
    """All 64 F~_i within 1e-10 (checked while building the fixture) and the
    whole-job q = F p within 1e-10 of the oracle's."""
    prob, op = c3["prob"], c3["op"]
    assert c3["worst"] <= TOL
    p = np.random.default_rng(7).normal(size=prob.n_multipliers)
    q = op.apply(p)
    qr = ora.apply_dense_full(c3["fmats"], _cons(prob, c3["subs"]), p)
    assert np.linalg.norm(q - qr) <= TOL * np.linalg.norm(qr)


def _dual_system(c):
    prob = c["prob"]
    kernels = [c["qs"][s] for s in c["subs"]]
    forces = [c["fs"][s] for s in c["subs"]]
    kf = c["kf"]

    def solve_f(i, b):          # assemble_dual_system solves only with f_i
        assert b is forces[i]
        return kf[i]

    return ora.assemble_dual_system(kernels, forces, _cons(prob, c["subs"]), prob.n_multipliers, prob.c, solve_f)


def test_c3_pcpg_iteration_count(c3):
    """PCPG at config 3 (tol 1e-9, solver.py:195-272): the oracle's recursion
    on the oracle operator gives the reference-consistent count; the same
    recursion driving the drop-in's apply must give exactly that count and
    lambda within 1e-9.  Operator sensitivity: 1e-14 relative perturbations of
    every F~_i (the size of any two correct implementations' rounding
    difference) leave the count unchanged.  Solver sensitivity: the count is
    decided by ||w_114|| / ||w_0||, which lies within 1 % of the tolerance, so
    a legitimate change of the solver's own arithmetic -- the coarse problem
    solved with the explicit inverse of G^T G instead of its Cholesky factor,
    as the device loop does -- may stop one iteration earlier; the device
    loop (tests/test_gpu_pcpg.py) therefore accepts {114, 115} here and must
    reach the same multipliers (1e-9)."""
    prob, op = c3["prob"], c3["op"]
    cons = _cons(prob, c3["subs"])
    gm, e, d, coarse = _dual_system(c3)
    wn = []
    lam_o, it_o = ora.pcpg(gm, e, d, coarse, lambda p: ora.apply_dense_full(c3["fmats"], cons, p), tol=1e-9,
                           wnorms=wn)
    lam_d, it_d = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
    rng = np.random.default_rng(11)
    seen = {it_o}
    for _ in range(3):
        pert = [f * (1.0 + 1e-14 * rng.standard_normal(f.shape)) for f in c3["fmats"]]
        pert = [0.5 * (f + f.T) for f in pert]
        seen.add(ora.pcpg(gm, e, d, coarse, lambda p: ora.apply_dense_full(pert, cons, p), tol=1e-9)[1])
    cinv = np.linalg.inv(coarse.T @ coarse)
    it_inv = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9, coarse_inverse=0.5 * (cinv + cinv.T))[1]
    margin = wn[it_o - 1] / wn[0] / 1e-9
    print(f"c3 PCPG: oracle {it_o}, drop-in {it_d}, under 1e-14 F perturbations {sorted(seen)}, "
          f"explicit coarse inverse {it_inv}; ||w_{it_o - 1}||/||w_0|| = {margin:.5f} x tol")
    assert seen == {it_o}, f"c3 count is operator-rounding-sensitive: {sorted(seen)}"
    assert it_d == it_o
    assert np.linalg.norm(lam_d - lam_o) <= 1e-9 * np.linalg.norm(lam_o)
    assert 1.0 < margin < 1.01            # the last-but-one residual is within 1 % of the tolerance
    assert it_inv in (it_o - 1, it_o)


def test_c4_every_subdomain_and_whole_job_apply():
    """Config 4 (3D elasticity, 64 x 10,125 DOFs, m up to 3,873): all 64 F~_i
    and the whole-job q = F p against the dense-K_reg oracle."""
    prob = inputs.Problem(*inputs.CONFIGS["c4"])
    subs = list(range(prob.n_sub))
    op, ks, qs, _ = _sparse_route(prob, subs)
    with op:
        op.preprocess()
        fm, worst = _check_all_subdomains(prob, subs, op, _dense_oracle(prob, ks, qs))
        p = np.random.default_rng(8).normal(size=prob.n_multipliers)
        q = op.apply(p)
    qr = ora.apply_dense_full([f for f, _ in fm], _cons(prob, subs), p)
    assert worst <= TOL
    assert np.linalg.norm(q - qr) <= TOL * np.linalg.norm(qr)


def test_c5_cluster_every_subdomain_and_cluster_apply():
    """Config 5 (2D elasticity, 256 x 33,282 DOFs): one full cluster of the
    8-GPU layout (32 subdomains, cluster 0 of build_clusters,
    decomposition.py:227-243) -- every F~_i against the Woodbury oracle
    (SuperLU of a differently shifted K, computed on all host cores) and the
    cluster's contribution to q = F p."""
    prob = inputs.Problem(*inputs.CONFIGS["c5"], n_clusters=8)
    subs = [int(s) for s in prob.layout.clusters[0].subdomain_ids]
    assert len(subs) == 32
    op, ks, qs, _ = _sparse_route(prob, subs)

    def woodbury(s):
        k = ks[s]
        sol = ora.WoodburyKregSolver(prob.n_dofs, k.indptr, k.indices, k.data, qs[s])
        return ora.fmatrix_via_solver(sol, prob.n_dofs, prob.bcol[s], prob.bval[s])

    with ThreadPoolExecutor(max(1, min(16, os.cpu_count() or 1))) as ex:
        refs = list(ex.map(woodbury, subs))
    with op:
        op.preprocess()
        worst = 0.0
        for s, ref in zip(subs, refs):
            got = op.local_operator(s)
            err = np.linalg.norm(got - np.triu(ref)) / np.linalg.norm(np.triu(ref))
            worst = max(worst, err)
            assert err <= TOL, (s, err)
        p = np.random.default_rng(9).normal(size=prob.n_multipliers)
        q = op.apply(p)
    qr = ora.apply_dense_full(refs, _cons(prob, subs), p)
    assert np.linalg.norm(q - qr) <= TOL * np.linalg.norm(qr)


def test_c3_device_pcpg():
    """The device-native PCPG (feti_pcpg_solve, d from the factorization) at
    config 3: the count is the reference-consistent 115 or, within the solver
    rounding sensitivity shown in test_c3_pcpg_iteration_count, 114; the
    multipliers agree with the reference's recursion driving the same operator
    to 1e-9, repeated solves are bit-identical, and the dual-system setup
    takes well under a second."""
    from paper_2502_08382_b200.pcpg import DevicePCPG

    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    subs = list(range(prob.n_sub))
    op, ks, qs, fs = _sparse_route(prob, subs)
    op.close()
    full = range(prob.n_sub)
    mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in full]
    kern, forces = [qs[s] for s in full], [fs[s] for s in full]
    with dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, factorization="sparse",
                        stiffness=[ks[s] for s in full], kernels=kern, forces=forces) as op:
        op.preprocess()
        sol = DevicePCPG(op, kern, forces, prob.c)
        assert sol.setup_seconds < 1.0
        lam, it, _ = sol.solve(tol=1e-9)
        lam2, it2, _ = sol.solve(tol=1e-9)
        gm = sol.gmat.toarray()
        import scipy.linalg

        coarse = scipy.linalg.cholesky(gm.T @ gm, lower=False)
        lam_h, it_h = ora.pcpg(gm, sol.e, sol.d, coarse, op.apply, tol=1e-9)
    print(f"c3 device PCPG {it} iterations ({sol.last_device_ms:.1f} ms), host recursion {it_h}")
    assert it_h == 115
    assert it in (114, 115)
    assert it == it2 and np.array_equal(lam, lam2)
    assert np.linalg.norm(lam - lam_h) <= 1e-9 * np.linalg.norm(lam_h)
