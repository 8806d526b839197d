"""GPU-resident PCPG: iteration counts and multipliers of
the reference's own solver runs (golden fixtures)."""

import numpy as np
import pytest

from conftest import SMALL_CASES, expected_iterations, load_golden
from paper_2502_08382_b200 import dualop
from harness import inputs
from paper_2502_08382_b200.pcpg import DevicePCPG

pytestmark = pytest.mark.gpu
CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")


def _solve(prob, dense=False):
    mats, cons, lay = inputs.reference_inputs(prob, dense=dense)
    kernels, forces = [], []
    for s in range(prob.n_sub):
        _, f, q = prob.subdomain_system(s)
        kernels.append(q)
        forces.append(f)
    with dualop.prepare(mats, cons, lay, CFG, device=0, workers=8) as op:
        op.preprocess()
        solver = DevicePCPG(op, kernels, forces, prob.c)
        return solver.solve(tol=1e-9)


@pytest.mark.parametrize("case", SMALL_CASES + ["heat3d_c2"])
def test_device_pcpg_matches_reference(case):
    g = load_golden(case)
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]))
    lam, it, _ = _solve(prob, dense=(case == "heat3d_c2"))
    assert it in expected_iterations(case, g)
    ref = g["pcpg_lambda"]
    assert np.linalg.norm(lam - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("graph", [False, True])
def test_graph_and_eager_iterations_agree(graph):
    g = load_golden("heat2d_c1")
    prob = inputs.Problem(*inputs.CONFIGS["c1"])
    mats, cons, lay = inputs.reference_inputs(prob)
    kernels, forces = [], []
    for s in range(prob.n_sub):
        _, f, q = prob.subdomain_system(s)
        kernels.append(q)
        forces.append(f)
    with dualop.prepare(mats, cons, lay, CFG, device=0) as op:
        op.preprocess()
        solver = DevicePCPG(op, kernels, forces, prob.c)
        lam, it, _ = solver.solve(tol=1e-9, graph=graph)
        lam2, it2, _ = solver.solve(tol=1e-9, graph=graph)
    assert it == it2 == int(g["pcpg_iterations"]) == 63
    assert np.array_equal(lam, lam2)          # deterministic
    assert np.linalg.norm(lam - g["pcpg_lambda"]) <= 1e-9 * np.linalg.norm(g["pcpg_lambda"])


@pytest.mark.parametrize("case", SMALL_CASES)
def test_lumped_preconditioner_matches_reference(case):
    """make_preconditioner("lumped") (solver.py:155-175) on the device: the
    operator on the reference's seeded p, and PCPG with it -- the reference's
    iteration count through the reference's own recursion driving the
    drop-in, and through the GPU-resident loop."""
    from oracle import feti_oracle as ora

    g = load_golden(case)
    gl = load_golden(f"lumped_{case}")
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]))
    mats, cons, lay = inputs.reference_inputs(prob)
    ks, qs, fs = [], [], []
    for s in range(prob.n_sub):
        k, f, q = prob.subdomain_system(s)
        ks.append(k)
        qs.append(q)
        fs.append(f)
    with dualop.prepare(mats, cons, lay, CFG, device=0) as op:
        op.preprocess()
        op.set_lumped_preconditioner(ks)
        mp = op.precond_apply(gl["p"])
        ref = gl["lumped_p"]
        assert np.linalg.norm(mp - ref) <= 1e-12 * np.linalg.norm(ref)
        cl = [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in range(prob.n_sub)]
        gm, e, d, coarse = ora.assemble_dual_system(qs, fs, cl, prob.n_multipliers, prob.c, op.solve_local)
        lam_h, it_h = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9, mfun=op.precond_apply)
        assert it_h in expected_iterations(case, gl)
        lam, it, _ = DevicePCPG(op, qs, fs, prob.c, precond="lumped", stiffness=ks).solve(tol=1e-9)
    assert it in expected_iterations(case, gl)
    for got in (lam_h, lam):
        assert np.linalg.norm(got - gl["pcpg_lambda"]) <= 1e-9 * np.linalg.norm(gl["pcpg_lambda"])


@pytest.mark.parametrize("variant", [{}, {"FETI_APPLY_CPS": "1"}, {"FETI_PCPG_FUSED": "0", "FETI_APPLY_CPS": "1"},
                                     {"FETI_PCPG_COOP": "0"}])
def test_device_pcpg_iteration_variants(variant, monkeypatch):
    """Every device-loop schedule gives the reference's count and multipliers:
    the fused single-launch iteration (apply + vector phases, 8-warp apply:
    FETI_APPLY_CPS=1 on these small subdomains), the apply + cooperative
    vector kernel, and the five-launch iteration (FETI_PCPG_COOP=0)."""
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    case = "heat3d_4x2"
    g = load_golden(case)
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]))
    lam, it, _ = _solve(prob)
    assert it in expected_iterations(case, g)
    assert np.linalg.norm(lam - g["pcpg_lambda"]) <= 1e-9 * np.linalg.norm(g["pcpg_lambda"])
