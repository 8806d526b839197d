import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from harness import inputs
from paper_2502_08382_b200 import dualop
prob = inputs.Problem("elasticity", 2, 8, 2)
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, qk = prob.subdomain_system(s)
    ks.append(k); qs.append(qk)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
p = np.random.default_rng(0).normal(size=prob.n_multipliers)
for cfg in (dualop.DualOpConfig(strategy="explicit", path="trsm"), dualop.DualOpConfig(strategy="implicit")):
    with dualop.prepare(mats, prob.constraints(), prob.layout, cfg, device=0, factorization="sparse",
                        stiffness=ks, kernels=qs) as op:
        op.preprocess()
        print(cfg.strategy, np.linalg.norm(op.apply(p)))
        xs = op.solve_local_many([0, 1], [np.ones(prob.n_dofs)] * 2)
        print("solve", np.linalg.norm(xs[0]))
