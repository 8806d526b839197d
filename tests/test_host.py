"""Host-side logic without a GPU: the C-ABI library, config, factorization."""

import ctypes as C
import os
import re

import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import reverse_cuthill_mckee

from conftest import ROOT
from paper_2502_08382_b200 import _lib, dualop, inputs
from paper_2502_08382_b200 import factor as fct

HEADER = os.path.join(ROOT, "include", "feti_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(feti_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)
    assert lib.feti_abi_version() == 1


def test_create_without_gpu_fails_loudly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib = _lib.load()
    ctx = C.c_void_p()
    rc = lib.feti_create(0, C.byref(ctx))
    assert rc != 0
    assert lib.feti_last_error()


def test_missing_library_raises(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libfeti_b200.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_config_mirrors_reference():
    # test_dualop.py:33-49
    cfg = dualop.DualOpConfig()
    assert cfg.strategy == "implicit"
    for bad in (dict(strategy="magic"), dict(path="gemm"), dict(rhs_order="diagonal")):
        with pytest.raises(ValueError):
            dualop.DualOpConfig(**bad)
    cfg2 = cfg.replace(path="syrk")
    assert cfg2.path == "syrk" and cfg2.strategy == "implicit"


def test_non_explicit_strategy_rejected():
    prob = inputs.Problem("heat", 2, 3, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    with pytest.raises(ValueError, match="explicit"):
        dualop.DualOperator(mats, cons, lay, dualop.DualOpConfig(strategy="implicit"))


@pytest.mark.parametrize("n", [7, 40])
def test_rcm_of_complete_graph_is_reversed_natural(n):
    dense = np.random.default_rng(n).random((n, n)) + 1.0
    dense = dense + dense.T
    sp = csr_matrix(dense)
    ref = reverse_cuthill_mckee(sp, symmetric_mode=True)
    np.testing.assert_array_equal(fct.rcm_ordering(inputs.DenseSym(dense)), ref)
    np.testing.assert_array_equal(ref, np.arange(n)[::-1])


def test_dense_factor_layout_and_solve():
    prob = inputs.Problem("heat", 3, 3, 2)
    k, f, q = prob.subdomain_system(3)
    kreg = inputs.DenseSym(inputs.regularized_dense(k, q))
    n = k.shape[0]
    perm = fct.rcm_ordering(kreg)
    vals = fct.numeric_factorize_dense(kreg, perm)
    assert vals.shape == (n * (n + 1) // 2,)
    # packed col-major lower: column j = rows j..n-1 of L
    L = np.linalg.cholesky(kreg.values[np.ix_(perm, perm)])
    off = 0
    for j in range(n):
        np.testing.assert_allclose(vals[off:off + n - j], L[j:, j], rtol=1e-12, atol=1e-14)
        off += n - j
    x = fct.solve_packed(vals, perm, f)
    np.testing.assert_allclose(kreg.values @ x, f, rtol=1e-10, atol=1e-12)


def test_interface_last_ordering_puts_constrained_dofs_last():
    prob = inputs.Problem("heat", 3, 3, 2)
    k, _, q = prob.subdomain_system(0)
    kreg = inputs.DenseSym(inputs.regularized_dense(k, q))
    bcol = prob.bcol[0]
    perm = fct.interface_last_ordering(kreg, bcol)
    n = k.shape[0]
    assert np.array_equal(np.sort(perm), np.arange(n))
    nb = np.unique(bcol).shape[0]
    assert set(perm[n - nb:].tolist()) == set(np.unique(bcol).tolist())


def test_spd_violation_reported():
    a = inputs.DenseSym(-np.eye(4))
    with pytest.raises(fct.SpdError, match="permuted row 0"):
        fct.numeric_factorize_dense(a, np.arange(4))
