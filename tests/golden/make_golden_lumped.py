"""Golden fixtures for the lumped preconditioner (solver.py:155-175) by running
the UNMODIFIED reference here (same no-write recipe and `_temp` shim as
make_golden.py):

    cd /tmp && NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \\
        python /root/repo/tests/golden/make_golden_lumped.py

Writes tests/golden/lumped_<case>.npz: the lumped operator applied to the
seeded p of <case>.npz (make_preconditioner("lumped", ...)) and the PCPG of
run_steps(..., precond="lumped") for the explicit SYRK path: iterations and
lambda.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, _import_reference  # noqa: E402

CASES = {
    "heat2d_3x2": ("heat", 2, 3, 2),
    "heat2d_c1": ("heat", 2, 16, 4),
    "heat3d_4x2": ("heat", 3, 4, 2),
    "elast2d_4x2": ("elasticity", 2, 4, 2),
    "elast3d_4x2": ("elasticity", 3, 4, 2),
}


def lumped_case(name, physics, dim, cells, subs):
    tfeti = _import_reference()
    from tfeti import dualop as dop
    from tfeti import solver as sl

    t0 = time.time()
    prob = tfeti.build_problem(physics, dim, cells, subs)
    subp = prob.subdomain_problems()
    n_mult = prob.constraints.n_multipliers
    p = np.random.default_rng(0).normal(size=n_mult)
    out = {"p": p,
           "lumped_p": sl.make_preconditioner("lumped", subp, prob.constraints)(p)}
    cfg = dop.DualOpConfig(strategy="explicit", path="syrk")
    rep = tfeti.run_steps(prob, 1, config=cfg, tol=1e-9, precond="lumped")[0]
    out["pcpg_iterations"] = np.array(rep.iterations)
    out["pcpg_lambda"] = rep.lam
    np.savez_compressed(os.path.join(OUT, f"lumped_{name}.npz"), **out)
    print(f"lumped_{name}: {rep.iterations} iterations, {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        lumped_case(name, *CASES[name])
