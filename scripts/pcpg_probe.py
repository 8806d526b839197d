"""Relative PCPG residual around the stopping iteration at config 3 (tol 1e-9):
the reference-consistent count is rounding-sensitive when ||w_k||/||w_0|| at the
last-but-one iteration sits within rounding of the tolerance."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import inputs  # noqa: E402
from oracle import feti_oracle as ora  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402
from paper_2502_08382_b200.pcpg import ConvergenceError, DevicePCPG  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
prob = inputs.Problem(*inputs.CONFIGS[cfg])
ks, qs, fs = [], [], []
for s in range(prob.n_sub):
    k, f, q = prob.subdomain_system(s)
    ks.append(k)
    qs.append(q)
    fs.append(f)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs))] * prob.n_sub
cfg_op = dualop.DualOpConfig(strategy="explicit", path="syrk")
op = dualop.prepare(mats, prob.constraints(), prob.layout, cfg_op, device=0,
                    factorization="sparse", stiffness=ks, kernels=qs, forces=fs)
op.preprocess()
sol = DevicePCPG(op, qs, fs, prob.c)
lam, it, _ = sol.solve(tol=1e-9)
print(f"device loop: {it} iterations, final relative residual {sol.relative_residual:.6e}")
for k in range(it - 2, it):
    try:
        sol.solve(tol=1e-9, maxit=k)
    except ConvergenceError as err:
        print(f"  after {k} iterations: {str(err).split('(')[-1].rstrip(')')}")
# the reference's recursion (oracle) driving the drop-in, with its residual history
cons = [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in range(prob.n_sub)]
d = sol.d
gm = sol.gmat.toarray()
import scipy.linalg
coarse = scipy.linalg.cholesky(gm.T @ gm, lower=False)
hist = []
def fapply(p):
    return op.apply(p)
lam_h, it_h = ora.pcpg(gm, sol.e, d, coarse, fapply, tol=1e-9)
print(f"host recursion (oracle pcpg) on the drop-in: {it_h} iterations")
op.close()
