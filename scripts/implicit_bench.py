"""Implicit-strategy apply timing on the sparse route (device vectors):
python scripts/implicit_bench.py c3 [n_applies]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import inputs  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
napp = int(sys.argv[2]) if len(sys.argv) > 2 else 50
prob = inputs.Problem(*inputs.CONFIGS[cfg])
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, q = prob.subdomain_system(s)
    ks.append(k)
    qs.append(q)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs))] * prob.n_sub
op = dualop.prepare(mats, prob.constraints(), prob.layout, dualop.DualOpConfig(strategy="implicit"), device=0,
                    factorization="sparse", stiffness=ks, kernels=qs)
op.preprocess()
p = torch.from_numpy(np.random.default_rng(0).normal(size=prob.n_multipliers)).cuda()
q = torch.empty_like(p)
st = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    op.apply_implicit_device(p, q, st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(napp):
    op.apply_implicit_device(p, q, st)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / napp
st_ = op.stats()
print(f"{cfg} implicit apply {ms * 1e3:.1f} us (preprocess {st_['ms_preprocess']:.2f} ms), |q| {q.norm().item():.12e}")
op.close()
