"""Apply-kernel timing on a configuration (sparse route), device vectors:
python scripts/apply_bench.py c3 [n_applies]; FETI_APPLY_WARPS to sweep."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import inputs  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
napp = int(sys.argv[2]) if len(sys.argv) > 2 else 200
prob = inputs.Problem(*inputs.CONFIGS[cfg])
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, q = prob.subdomain_system(s)
    ks.append(k)
    qs.append(q)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs))] * prob.n_sub
cfg_op = dualop.DualOpConfig(strategy="explicit", path="syrk")
op = dualop.prepare(mats, prob.constraints(), prob.layout, cfg_op, device=0,
                    factorization="sparse", stiffness=ks, kernels=qs)
op.preprocess()
dev = torch.device("cuda", 0)
p = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).to(dev)
q = torch.empty_like(p)
ref = op.apply(p.cpu().numpy())
for _ in range(10):
    op.apply_device(p, q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(napp):
    op.apply_device(p, q)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / napp
b = op.stats()["apply_bytes_alg"]
err = float(np.linalg.norm(q.cpu().numpy() - ref) / np.linalg.norm(ref))
print(f"{cfg} warps={os.environ.get('FETI_APPLY_WARPS', 8)} apply {ms * 1e3:.1f} us  {b / ms / 1e6:.0f} GB/s "
      f"(host-apply consistency {err:.1e})")
op.close()
