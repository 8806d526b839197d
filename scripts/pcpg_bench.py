"""Device PCPG timing on the sparse route: python scripts/pcpg_bench.py c3 (FETI_PCPG_COOP=0 for the 5-launch loop)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import inputs  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402
from paper_2502_08382_b200.pcpg import DevicePCPG  # noqa: E402

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
sol.solve()
lam, it, _ = sol.solve()
lam2, it2, _ = sol.solve()
assert it == it2 and np.array_equal(lam, lam2)
print(f"{cfg} coop={os.environ.get('FETI_PCPG_COOP', 1)}: {it} iterations, {sol.last_device_ms:.2f} ms, "
      f"{sol.last_device_ms / it * 1e3:.1f} us/iteration, setup {sol.setup_seconds:.3f} s, |lam| {np.linalg.norm(lam):.12e}")
op.close()
