"""GPU-resident PCPG: iteration counts and multipliers of
the reference's own solver runs (golden fixtures)."""

import numpy as np
import pytest

from conftest import SMALL_CASES, expected_iterations, load_golden
from paper_2502_08382_b200 import dualop, inputs
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
