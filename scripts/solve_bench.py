"""Device solve_local on the sparse route (feti_solve_many): wall time of one
batched call over every subdomain of a config (host b -> host x), against the
oracle's Woodbury K_reg^-1 on two subdomains."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from harness import inputs  # noqa: E402
from oracle import feti_oracle as ora  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
prob = inputs.Problem(*inputs.CONFIGS[cfg])
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, q = prob.subdomain_system(s)
    ks.append(k)
    qs.append(q)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs)) for _ in range(prob.n_sub)]
cfg_op = dualop.DualOpConfig(strategy="explicit", path="syrk")
op = dualop.prepare(mats, prob.constraints(), prob.layout, cfg_op, device=0,
                    factorization="sparse", stiffness=ks, kernels=qs)
op.preprocess()
rng = np.random.default_rng(0)
idx = list(range(prob.n_sub))
rhs = [rng.normal(size=prob.n_dofs) for _ in idx]
op.solve_local_many(idx, rhs)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    xs = op.solve_local_many(idx, rhs)
    ts.append(time.perf_counter() - t0)
t1 = time.perf_counter()
op.solve_local(0, rhs[0])
one = time.perf_counter() - t1
err = 0.0
for s in (0, prob.n_sub // 2):
    ref = ora.WoodburyKregSolver(prob.n_dofs, ks[s].indptr, ks[s].indices, ks[s].data, qs[s]).solve(rhs[s])
    err = max(err, np.linalg.norm(xs[s] - ref) / np.linalg.norm(ref))
print(f"{cfg}: solve_local_many over {prob.n_sub} subdomains x {prob.n_dofs} DOFs: "
      f"median {np.median(ts) * 1e3:.2f} ms (host b -> host x); one subdomain {one * 1e3:.2f} ms; "
      f"max rel err vs Woodbury {err:.2e}")
op.close()
