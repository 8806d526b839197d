"""Device numeric factorization: K_reg = K + rho Q Q^T formed and
factored on the GPU from the sparse K; everything downstream must match the
reference exactly as with the host factor."""

import numpy as np
import pytest

from conftest import SMALL_CASES, expected_device_loop_iterations, expected_iterations, load_golden
from paper_2502_08382_b200 import dualop
from harness import inputs
from paper_2502_08382_b200.pcpg import DevicePCPG

pytestmark = pytest.mark.gpu
CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")


def _device_op(prob, ordering="rcm", subs=None):
    ks, qs, fs = [], [], []
    for s in range(prob.n_sub):
        k, f, q = prob.subdomain_system(s)
        ks.append(k)
        qs.append(q)
        fs.append(f)
    mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
    op = dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, ordering=ordering,
                        factorization="device", stiffness=ks, kernels=qs)
    return op, ks, qs, fs


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("ordering", ["rcm", "interface_last"])
def test_device_factor_matches_reference(case, ordering):
    g = load_golden(case)
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]))
    op, ks, qs, fs = _device_op(prob, ordering)
    with op:
        op.preprocess()
        for s in range(prob.n_sub):
            m = prob.gids[s].shape[0]
            ref = np.zeros((m, m))
            ref[np.triu_indices(m)] = g[f"s{s}_F_upper"]
            f = op.local_operator(s)
            assert np.linalg.norm(f - ref) <= 1e-10 * np.linalg.norm(ref), (case, s)
        q = op.apply(g["p"])
        assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])
        qi = op.apply_implicit(g["p"])
        assert np.linalg.norm(qi - g["q_implicit"]) <= 1e-11 * np.linalg.norm(g["q_implicit"])
        # the reference's recursion driving the drop-in: the reference's count
        from oracle import feti_oracle as ora

        cl = [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in range(prob.n_sub)]
        gm, e, d, coarse = ora.assemble_dual_system(qs, fs, cl, prob.n_multipliers, prob.c, op.solve_local)
        lam_h, it_h = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
        assert it_h in expected_iterations(case, g)
        lam, it, _ = DevicePCPG(op, qs, fs, prob.c).solve(tol=1e-9)
    assert it in expected_device_loop_iterations(case, g)
    for got in (lam_h, lam):
        assert np.linalg.norm(got - g["pcpg_lambda"]) <= 1e-9 * np.linalg.norm(g["pcpg_lambda"])


def test_device_solve_local_matches_dense_solve():
    prob = inputs.Problem("elasticity", 3, 3, 2)
    op, ks, qs, fs = _device_op(prob)
    with op:
        op.preprocess()
        rng = np.random.default_rng(0)
        for s in (0, 5):
            kreg = inputs.regularized_dense(ks[s], qs[s])
            b = rng.normal(size=prob.n_dofs)
            x = op.solve_local(s, b)
            ref = np.linalg.solve(kreg, b)
            assert np.linalg.norm(x - ref) <= 1e-11 * np.linalg.norm(ref)


def test_device_factor_spd_violation_reports_subdomain():
    prob = inputs.Problem("heat", 2, 3, 2)
    op, ks, qs, fs = _device_op(prob)
    bad = list(ks)
    k1 = ks[1]
    bad[1] = inputs.Csr(k1.shape, k1.indptr, k1.indices, -k1.data)
    with op:
        with pytest.raises(dualop.SpdError, match="subdomain 1"):
            op.preprocess(stiffness=bad)


def test_device_factor_c3_subdomain_checksums():
    g = load_golden("c3_sub21")
    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    s = int(g["sub_index"])
    k, f, q = prob.subdomain_system(s)
    m = prob.gids[s].shape[0]
    mat = inputs.Csr((m, prob.n_dofs), np.arange(m + 1, dtype=np.int64), prob.bcol[s], prob.bval[s])
    cons = inputs.ConstraintSet(m, np.zeros(m), [inputs.SubdomainConstraints(np.arange(m, dtype=np.int64), mat)])
    lay = inputs.ClusterLayout([inputs.Cluster(0, np.array([0]), np.arange(m), [np.arange(m)])], m)
    with dualop.prepare([inputs.ShapeOnly((prob.n_dofs, prob.n_dofs))], cons, lay, CFG, device=0,
                        factorization="device", stiffness=[k], kernels=[q]) as op:
        op.preprocess()
        fu = op.local_operator(0)
    full = fu + np.triu(fu, 1).T
    for name, got in (("Fv", full @ g["v"]), ("F_diag", np.diag(full)), ("F_row0", full[0])):
        ref = g[name]
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), name


def _with_decoupled_dofs(k, q, extra):
    """K_ext = blockdiag(K, d I) (d = mean diagonal of K), kernel [Q; 0]."""
    n = k.shape[0]
    ip = np.asarray(k.indptr, np.int64)
    d = float(np.mean(k.to_dense().diagonal()))
    ip2 = np.concatenate([ip, ip[-1] + 1 + np.arange(extra, dtype=np.int64)])
    ix2 = np.concatenate([np.asarray(k.indices, np.int64), n + np.arange(extra, dtype=np.int64)])
    dt2 = np.concatenate([np.asarray(k.data, np.float64), np.full(extra, d)])
    return (inputs.Csr((n + extra, n + extra), ip2, ix2, dt2),
            np.vstack([q, np.zeros((extra, q.shape[1]))]))


@pytest.mark.parametrize("route", ["device", "sparse"])
@pytest.mark.parametrize("physics,dim,cells", [("elasticity", 2, 8), ("heat", 3, 5)])
def test_device_factor_non_uniform_subdomains(physics, dim, cells, route):
    """Subdomains of different sizes on the device-factor routes (the
    reference's symbolic/numeric stages are per subdomain, sparse.py:340-424):
    subdomain 0 carries 300 extra decoupled DOFs, so it spans more 128-row
    blocks than the others.  Every F~_i, q = F p and solve_local equal the
    host-factor route's on the same K_reg (1e-10)."""
    prob = inputs.Problem(physics, dim, cells, 2)
    ks, qs = [], []
    for s in range(prob.n_sub):
        k, _, q = prob.subdomain_system(s)
        ks.append(k)
        qs.append(q)
    ks[0], qs[0] = _with_decoupled_dofs(ks[0], qs[0], 300)
    assert -(-ks[0].shape[0] // 128) > -(-ks[1].shape[0] // 128)
    cons, lay = prob.constraints(), prob.layout
    c0 = cons.per_subdomain[0]
    mat = c0.matrix
    cons.per_subdomain[0] = inputs.SubdomainConstraints(
        c0.multiplier_ids, inputs.Csr((mat.shape[0], ks[0].shape[0]), mat.indptr, mat.indices, mat.data))
    p = np.random.default_rng(2).normal(size=prob.n_multipliers)
    b0 = np.random.default_rng(3).normal(size=ks[0].shape[0])
    host = [inputs.regularized_csr(k, q) for k, q in zip(ks, qs)]
    with dualop.prepare(host, cons, lay, CFG) as oph:
        oph.preprocess()
        fh = [oph.local_operator(s) for s in range(prob.n_sub)]
        qh = oph.apply(p)
        xh = oph.solve_local(0, b0)
    with dualop.prepare([inputs.ShapeOnly(k.shape) for k in ks], cons, lay, CFG, device=0, factorization=route,
                        stiffness=ks, kernels=qs) as opd:
        opd.preprocess()
        fd = [opd.local_operator(s) for s in range(prob.n_sub)]
        qd = opd.apply(p)
        xd = opd.solve_local(0, b0)
    for a, b in zip(fd, fh):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    assert np.linalg.norm(qd - qh) <= 1e-10 * np.linalg.norm(qh)
    assert np.linalg.norm(xd - xh) <= 1e-10 * np.linalg.norm(xh)
