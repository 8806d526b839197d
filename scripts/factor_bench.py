"""Sparse-route preprocess timing (device-resident K): python scripts/factor_bench.py c3 [steps].
FETI_SP_GROUPS sweeps the factorization group count."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import inputs  # noqa: E402
from paper_2502_08382_b200 import dualop  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prob = inputs.Problem(*inputs.CONFIGS[cfg])
ks, qs = [], []
for s in range(prob.n_sub):
    k, _, q = prob.subdomain_system(s)
    ks.append(k)
    qs.append(q)
mats = [inputs.ShapeOnly((prob.n_dofs, prob.n_dofs))] * prob.n_sub
cfg_op = dualop.DualOpConfig(strategy="explicit", path=os.environ.get("FETI_PATH", "syrk"))
op = dualop.prepare(mats, prob.constraints(), prob.layout, cfg_op, device=0,
                    factorization="sparse", stiffness=ks, kernels=qs,
                    sparse_ordering=os.environ.get("FETI_SPARSE_ORDERING", "auto"))
for _ in range(3):
    op.preprocess()
fac, pre = [], []
for _ in range(steps):
    op.preprocess_resident()
    st = op.stats()
    fac.append(st["ms_factorize"])
    pre.append(st["ms_preprocess"])
print(f"{cfg} recipe={op.sparse_recipe} groups={os.environ.get('FETI_SP_GROUPS', 8)}: "
      f"factorize {statistics.median(fac):.2f} ms, preprocess {statistics.median(pre):.2f} ms, "
      f"tail {statistics.median(pre) - statistics.median(fac):.2f} ms")
op.close()
