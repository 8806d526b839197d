import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


SMALL_CASES = ["heat2d_3x2", "heat2d_c1", "heat3d_4x2", "elast2d_4x2", "elast3d_4x2"]


# PCPG iteration counts that are robust to 1e-14 rounding differences are
# asserted exactly; elasticity 3D 4^3 sits at 9.83e-10 vs tol 1e-9 and flips
# between 93 and 94 under such perturbations (tests/test_oracle.py::
# test_pcpg_iteration_count_sensitivity), so one extra iteration is accepted.
ROUNDING_SENSITIVE = {"elast3d_4x2"}


def expected_iterations(case, g):
    it = int(g["pcpg_iterations"])
    return {it, it + 1} if case in ROUNDING_SENSITIVE else {it}


# The GPU-resident PCPG loop (torch reductions, device projector) rounds
# differently from numpy at every step; on config 1 its relative residual
# after the reference's 63 iterations lands at 0.8-1.05e-9 depending on
# last-bit differences of F~ and d (tests/test_gpu_factor.py and
# test_gpu_sparse.py run the reference's own recursion through the drop-in
# and assert 63 exactly; the device loop may take one more).
DEVICE_LOOP_SENSITIVE = {"heat2d_c1"}


def expected_device_loop_iterations(case, g):
    it = int(g["pcpg_iterations"])
    extra = {it + 1} if case in DEVICE_LOOP_SENSITIVE else set()
    return expected_iterations(case, g) | extra
