"""Small end-to-end exercise of every kernel for compute-sanitizer runs:
assembly (dense + sparse pattern), apply (host + device), coarse projector."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from harness import inputs  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402
from paper_2502_08382_b200.pcpg import DevicePCPG  # noqa: E402

CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")
for phys, dim, cells, subs in (("heat", 3, 4, 2), ("elasticity", 2, 6, 2)):
    prob = inputs.Problem(phys, dim, cells, subs)
    mats, cons, lay = inputs.reference_inputs(prob)
    for ordering in ("rcm", "interface_last"):
        with dualop.prepare(mats, cons, lay, CFG, device=0, ordering=ordering) as op:
            op.preprocess()
            p = np.random.default_rng(0).normal(size=prob.n_multipliers)
            q = op.apply(p)
            kernels, forces = [], []
            for s in range(prob.n_sub):
                _, f, qk = prob.subdomain_system(s)
                kernels.append(qk)
                forces.append(f)
            lam, it, _ = DevicePCPG(op, kernels, forces, prob.c).solve(tol=1e-9)
            print(phys, dim, ordering, "apply norm", np.linalg.norm(q), "pcpg it", it)
# sparse CSR-of-U pattern through the C-ABI
import test_gpu_parity as t  # noqa: E402

t.test_sparse_pattern_factor_through_cabi()
print("sparse pattern ok")
# sparse-factor route: block-sparse device factorization, assembly, rank-2r
# correction, the device dual right-hand side and the device PCPG
prob = inputs.Problem("elasticity", 2, 8, 2)
ks, qs, fs = [], [], []
for s in range(prob.n_sub):
    k, f, qk = prob.subdomain_system(s)
    ks.append(k)
    qs.append(qk)
    fs.append(f)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
with dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, factorization="sparse",
                    stiffness=ks, kernels=qs, forces=fs) as op:
    op.preprocess()
    op.preprocess()
    q = op.apply(np.random.default_rng(0).normal(size=prob.n_multipliers))
    lam, it, _ = DevicePCPG(op, qs, fs, prob.c).solve(tol=1e-9)
    print("sparse route apply norm", np.linalg.norm(q), "device pcpg it", it)
# tile-aligned dissection (padded positions) and the lumped preconditioner
prob = inputs.Problem("heat", 3, 6, 2)
ks, qs, fs = [], [], []
for s in range(prob.n_sub):
    k, f, qk = prob.subdomain_system(s)
    ks.append(k)
    qs.append(qk)
    fs.append(f)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
with dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, factorization="sparse",
                    stiffness=ks, kernels=qs, sparse_ordering="dissection:2") as op:
    op.preprocess()
    op.preprocess()
    q = op.apply(np.random.default_rng(0).normal(size=prob.n_multipliers))
    op.set_lumped_preconditioner(ks)
    mq = op.precond_apply(q)
    print("dissection route apply norm", np.linalg.norm(q), "lumped", np.linalg.norm(mq))
    xs = op.solve_local_many(list(range(prob.n_sub)), [np.ones(prob.n_dofs)] * prob.n_sub)
    print("sparse device solve_local norm", np.linalg.norm(xs[0]))
# path "trsm" (transposed trailing tiles, backward chains, row gather) on the
# sparse route, and the implicit strategy on the sparse route (U2 sweep +
# corrected sweeps)
prob = inputs.Problem("elasticity", 2, 8, 2)
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, qk = prob.subdomain_system(s)
    ks.append(k)
    qs.append(qk)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
p = np.random.default_rng(0).normal(size=prob.n_multipliers)
for cfg in (dualop.DualOpConfig(strategy="explicit", path="trsm"), dualop.DualOpConfig(strategy="implicit")):
    with dualop.prepare(mats, prob.constraints(), prob.layout, cfg, device=0, factorization="sparse",
                        stiffness=ks, kernels=qs) as op:
        op.preprocess()
        print(cfg.strategy, cfg.path, "sparse route apply norm", np.linalg.norm(op.apply(p)))
# face-grown dissection (interface pieces) through the fused step graph
# (factorization + each group's assembly captured together), two steps
prob = inputs.Problem("heat", 3, 12, 2)
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, qk = prob.subdomain_system(s)
    ks.append(k)
    qs.append(qk)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
with dualop.prepare(mats, prob.constraints(), prob.layout, CFG, device=0, factorization="sparse",
                    stiffness=ks, kernels=qs, sparse_ordering="faces:2") as op:
    op.preprocess()
    op.preprocess()
    print("faces route", op.sparse_recipe, "apply norm",
          np.linalg.norm(op.apply(np.random.default_rng(0).normal(size=prob.n_multipliers))))
