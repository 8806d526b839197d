"""Host-side logic without a GPU: the C-ABI library, config, factorization."""

import ctypes as C
import os
import re

import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import reverse_cuthill_mckee

from conftest import ROOT
from paper_2502_08382_b200 import _lib, dualop
from harness import inputs
from paper_2502_08382_b200 import factor as fct
from paper_2502_08382_b200 import sparse_route as spr

HEADER = os.path.join(ROOT, "include", "feti_b200.h")


class _HostKsSolver:
    """x = K_reg^-1 b = Pi K_s^-1 Pi b + rho^-1 Q Q^T b with SuperLU of
    K_s = K + rho E E^T: the identity the sparse route's correction and its
    device solve rest on, checked here on the host."""

    def __init__(self, stiffness, q, fix):
        from scipy.sparse.linalg import splu

        n, ip, ix, dt = fct.csr_arrays(stiffness)
        self.q = np.asarray(q, dtype=np.float64).reshape(n, -1)
        self.rho = spr.regularization_shift(ip, ix, dt, n)
        fix = np.asarray(fix, np.int64)
        shift = csr_matrix((np.full(fix.shape[0], self.rho), (fix, fix)), shape=(n, n))
        self.lu = splu((csr_matrix((dt, ix, ip), shape=(n, n)) + shift).tocsc(), permc_spec="MMD_AT_PLUS_A")

    def _proj(self, v):
        return v - self.q @ (self.q.T @ v)

    def solve(self, b):
        b = np.asarray(b, dtype=np.float64)
        return self._proj(self.lu.solve(self._proj(b))) + self.q @ (self.q.T @ b) / self.rho


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


class _SubProblem:
    """Duck type of the reference's SubdomainProblem (solver.py:100-106)."""

    def __init__(self, stiffness, stiffness_reg, force, kernel):
        self.stiffness, self.stiffness_reg, self.force, self.kernel = stiffness, stiffness_reg, force, kernel


def test_problem_like_inputs_select_the_sparse_route():
    """SubdomainProblem-like inputs (prepare_from_problems): K_i and ker K_i
    come from them and the route defaults to the sparse factor; with
    factorization='host' their stiffness_reg is used (the reference's
    run_steps hand-over, solver.py:424-431)."""
    prob = inputs.Problem("heat", 2, 3, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    subs = []
    for s in range(prob.n_sub):
        k, f, q = prob.subdomain_system(s)
        subs.append(_SubProblem(k, mats[s], f, q))
    op = dualop.DualOperator(subs, cons, lay, dualop.DualOpConfig(strategy="explicit"))
    assert op.factorization == "sparse"
    assert op.stiffness[0] is subs[0].stiffness and op.kernels[1] is subs[1].kernel
    assert op.matrices[0].shape == mats[0].shape
    op2 = dualop.DualOperator(subs, cons, lay, dualop.DualOpConfig(strategy="explicit"), factorization="host")
    assert op2.matrices[0] is mats[0]
    # the reference's default strategy (implicit) takes the sparse route too
    op3 = dualop.DualOperator(subs, cons, lay, dualop.DualOpConfig())
    assert op3.factorization == "sparse" and op3.forces[0] is subs[0].force


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


@pytest.mark.parametrize("case", ["elast2d_4x2", "heat3d_4x2", "elast3d_4x2"])
def test_sparse_route_host_pieces(case):
    """Ordering (constrained DOFs last), fixing DOFs (K_s SPD) and the host
    solve_local of the sparse-factor route against the reference's F~_i."""
    from conftest import load_golden
    from oracle import feti_oracle as ora
    from harness import inputs

    g = load_golden(case)
    for s in range(int(g["n_sub"])):
        ip, ix, dt = g[f"s{s}_k_indptr"], g[f"s{s}_k_indices"], g[f"s{s}_k_data"]
        n = ip.shape[0] - 1
        bcol, bval = g[f"s{s}_bcol"], g[f"s{s}_bval"]
        perm = spr.onion_interface_last(n, ip, ix, bcol)
        assert np.array_equal(np.sort(perm), np.arange(n))
        iface = np.unique(bcol)
        assert np.array_equal(perm[n - iface.size:], iface)
        q, _ = np.linalg.qr(g[f"s{s}_kernel"])
        fix = spr.fixing_dofs(q)
        assert fix.shape == (q.shape[1],)
        assert np.linalg.matrix_rank(q[fix]) == q.shape[1]
        k = inputs.Csr((n, n), ip, ix, dt)
        dense = k.to_dense()
        dense[fix, fix] += spr.regularization_shift(ip, ix, dt, n)
        assert np.linalg.eigvalsh(dense).min() > 0.0
        f = ora.fmatrix_via_solver(_HostKsSolver(k, q, fix), n, bcol, bval)
        m = f.shape[0]
        ref = np.zeros((m, m))
        ref[np.triu_indices(m)] = g[f"s{s}_F_upper"]
        assert np.linalg.norm(np.triu(f) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_sparse_route_tile_aligned_dissection():
    """Padded positions of the tile-aligned dissection ordering: every DOF
    once, segments start on 128-row tiles, the interface last; the chosen
    recipe for config 3 is a dissection with fewer estimated tile flops
    than the onion ordering."""
    from harness import inputs

    prob = inputs.Problem("heat", 3, 12, 2)
    k, _, q = prob.subdomain_system(3)
    n = k.shape[0]
    bcol = prob.bcol[3]
    segs = spr.dissection_segments(n, k.indptr, k.indices, bcol, depth=2)
    perm, iperm = spr.padded_positions(segs)
    assert perm.shape[0] % 128 == 0 and perm.shape[0] >= n
    assert np.array_equal(np.sort(perm[perm >= 0]), np.arange(n))
    assert np.array_equal(perm[iperm], np.arange(n))
    p = 0
    for s in segs:
        assert p % 128 == 0 and np.array_equal(perm[p:p + s.size], s)
        p += -(-s.size // 128) * 128
    iface = np.unique(bcol)
    assert np.array_equal(np.sort(segs[-1]), iface)
    on_perm, on_iperm = spr.sparse_route_ordering(n, k.indptr, k.indices, bcol, ("onion",))
    e_on = spr.tile_flops_estimate(n, k.indptr, k.indices, on_iperm, n, 1, iface.size)
    e_nd = spr.tile_flops_estimate(n, k.indptr, k.indices, iperm, perm.shape[0], 1, iface.size)
    assert e_on > 0 and e_nd > 0
    big = inputs.Problem(*inputs.CONFIGS["c3"])
    kb, _, qb = big.subdomain_system(21)
    rec = spr.choose_ordering(kb.shape[0], kb.indptr, kb.indices, big.bcol[21], qb.shape[1])
    assert rec[0] == "dissection"


def test_sparse_route_face_dissection():
    """Interface pieces (constrained DOFs grouped by the subdomains their
    multipliers glue them to) and the face-grown dissection: a partition of
    the DOFs on tile-aligned segments with the interface last; on config 3's
    interior subdomain it cuts the axis planes (separators 361 / 171 / 81
    DOFs, leaves of 9x9x9) and leaves fewer estimated tile flops than the
    breadth-first dissection, so the chooser takes it."""
    from harness import inputs
    from paper_2502_08382_b200 import dualop

    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    cons = prob.constraints()
    first, second = dualop._multiplier_owners(cons)
    s = 21                                   # an interior subdomain: six glued faces
    g = prob.gids[s]
    nb = np.where(first[g] == s, second[g], first[g])
    assert (nb >= 0).all()
    pieces = spr.interface_pieces(prob.bcol[s], nb)
    sizes = sorted((p.size for p in pieces), reverse=True)
    # chained gluing (one multiplier per adjacent owner pair): six face-sized
    # pieces (edges/corners join the face of their chain neighbour), then edges
    assert len(pieces) == 14 and all(361 <= x <= 400 for x in sizes[:6]) and max(sizes[6:]) <= 21
    assert np.array_equal(np.sort(np.concatenate(pieces)), np.unique(prob.bcol[s]))
    k, _, q = prob.subdomain_system(s)
    n = k.shape[0]
    segs = spr.face_dissection_segments(n, k.indptr, k.indices, prob.bcol[s], pieces, depth=3)
    assert [x.size for x in segs[:3]] == [729, 729, 81]
    assert sorted(x.size for x in segs[:-1] if x.size < 729) == [81] * 4 + [171] * 2 + [361]
    perm, iperm = spr.padded_positions(segs)
    assert np.array_equal(np.sort(perm[perm >= 0]), np.arange(n))
    assert np.array_equal(perm[iperm], np.arange(n))
    iface = np.unique(prob.bcol[s])
    e_face = spr.tile_flops_estimate(n, k.indptr, k.indices, iperm, perm.shape[0], 1, iface.size)
    p2, i2 = spr.sparse_route_ordering(n, k.indptr, k.indices, prob.bcol[s], ("dissection", 2))
    e_bfs = spr.tile_flops_estimate(n, k.indptr, k.indices, i2, p2.shape[0], 1, iface.size)
    assert e_face < 0.85 * e_bfs
    rec = spr.choose_ordering(n, k.indptr, k.indices, prob.bcol[s], q.shape[1], pieces=pieces)
    assert rec[0] == "faces"
    # a Dirichlet row has one owner: its neighbour is -1
    s0 = 0
    g0 = prob.gids[s0]
    nb0 = np.where(first[g0] == s0, second[g0], first[g0])
    assert (nb0 == -1).any()


def test_sparse_route_ordering_cache():
    """Structurally identical subdomains (same pattern, interface and pieces)
    share one ordering computation; callers get private copies."""
    from harness import inputs

    prob = inputs.Problem("heat", 3, 8, 3)
    k, _, _ = prob.subdomain_system(13)
    bcol = prob.bcol[13]
    spr._ORDERING_CACHE.clear()
    p1, i1 = spr.sparse_route_ordering(k.shape[0], k.indptr, k.indices, bcol, ("dissection", 2))
    assert len(spr._ORDERING_CACHE) == 1
    p1[:] = -7
    p2, i2 = spr.sparse_route_ordering(k.shape[0], k.indptr, k.indices, bcol, ("dissection", 2))
    assert len(spr._ORDERING_CACHE) == 1 and not (p2 == -7).any()
    p3, _ = spr._sparse_route_ordering(k.shape[0], k.indptr, k.indices, bcol, ("dissection", 2))
    assert np.array_equal(p2, p3) and np.array_equal(p2[i2], np.arange(k.shape[0]))
    spr.sparse_route_ordering(k.shape[0], k.indptr, k.indices, bcol[: bcol.size // 2], ("dissection", 2))
    assert len(spr._ORDERING_CACHE) == 2
