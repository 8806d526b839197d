"""Device parity: the CUDA path through the C-ABI against the reference.

Bar (BASELINE.json north star): F~_i entries and F*lambda within 1e-10
relative in FP64; identical PCPG iteration counts; solution within 1e-9.
Small cases compare with the reference's own outputs (golden fixtures);
larger ones with the oracle on the same inputs.
"""

import ctypes as C

import numpy as np
import pytest

from conftest import SMALL_CASES, expected_iterations, load_golden
from oracle import feti_oracle as ora
from paper_2502_08382_b200 import _lib, dualop
from harness import inputs

pytestmark = pytest.mark.gpu

CFG = dualop.DualOpConfig(strategy="explicit", path="syrk")


def _golden_problem(g, clusters=1):
    prob = inputs.Problem(str(g["physics"]), int(g["dim"]), int(g["cells"]), int(g["subs"]), n_clusters=clusters)
    mats, cons, lay = inputs.reference_inputs(prob)
    return prob, mats, cons, lay


def _full(upper):
    return upper + np.triu(upper, 1).T


def _ref_upper(g, s, m):
    ref = np.zeros((m, m))
    ref[np.triu_indices(m)] = g[f"s{s}_F_upper"]
    return ref


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("ordering", ["rcm", "interface_last"])
def test_local_operators_match_reference(case, ordering):
    g = load_golden(case)
    prob, mats, cons, lay = _golden_problem(g)
    with dualop.prepare(mats, cons, lay, CFG, ordering=ordering) as op:
        op.preprocess()
        for s in range(prob.n_sub):
            m = prob.gids[s].shape[0]
            f = op.local_operator(s)
            assert np.all(np.tril(f, -1) == 0.0)
            ref = _ref_upper(g, s, m)
            assert np.linalg.norm(f - ref) <= 1e-10 * np.linalg.norm(ref), (case, s)
        q = op.apply(g["p"])
        assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])


@pytest.mark.parametrize("case", SMALL_CASES)
def test_pcpg_iterations_match_reference(case):
    g = load_golden(case)
    prob, mats, cons, lay = _golden_problem(g)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        kernels, forces, cl = [], [], []
        for s in range(prob.n_sub):
            k, f, q = prob.subdomain_system(s)
            kernels.append(q)
            forces.append(f)
            cl.append((prob.gids[s], prob.bcol[s], prob.bval[s]))
        gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cl, prob.n_multipliers, prob.c,
                                                    op.solve_local)
        lam, it = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
    assert it in expected_iterations(case, g)
    ref = g["pcpg_lambda"]
    assert np.linalg.norm(lam - ref) <= 1e-9 * np.linalg.norm(ref)


def test_same_factor_as_oracle_reference_values():
    """Hand the reference's own factor values (chol_numeric restatement) to the
    device; F~ must match the oracle's SYRK path on those values."""
    prob = inputs.Problem("heat", 3, 4, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        facs = []
        for s in range(prob.n_sub):
            k = mats[s]
            sym = ora.symbolic_factorize(k.shape[0], k.indptr, k.indices)
            assert np.array_equal(sym.perm, op._subs[s].perm)
            vals = ora.numeric_factorize(sym, k.data)
            assert sym.nnz == vals.shape[0] == k.shape[0] * (k.shape[0] + 1) // 2
            op.set_factor(s, vals)
            facs.append((sym, vals))
        op.assemble()
        for s, (sym, vals) in enumerate(facs):
            fo = ora.assemble_explicit_local(sym.up, sym.ui, vals, sym.n, sym.iperm, prob.bcol[s], prob.bval[s])
            f = op.local_operator(s)
            assert np.linalg.norm(f - fo) <= 1e-12 * np.linalg.norm(fo)


def _shifted(k, shift):
    """K + shift*I keeping K's sparse pattern: SPD with a genuinely sparse factor."""
    rows = np.repeat(np.arange(k.shape[0]), np.diff(k.indptr))
    data = k.data.copy()
    data[k.indices == rows] += shift
    return inputs.Csr(k.shape, k.indptr, k.indices, data)


def test_sparse_pattern_factor_through_cabi():
    """A factor whose CSR-of-U pattern is not a full triangle (the reference's
    symbolic stage on a sparse SPD matrix) goes through the C-ABI with its
    (up, ui) pattern; F~ must match the oracle on the same values."""
    prob = inputs.Problem("elasticity", 3, 3, 2)
    lib = _lib.load()
    ctx = C.c_void_p()
    _lib.check(lib.feti_create(0, C.byref(ctx)))
    try:
        syms = []
        for s in range(prob.n_sub):
            k = _shifted(prob.subdomain_system(s)[0], 1e-2)
            sym = ora.symbolic_factorize(k.shape[0], k.indptr, k.indices)
            vals = ora.numeric_factorize(sym, k.data)
            assert sym.nnz < sym.n * (sym.n + 1) // 2
            first = np.ascontiguousarray(sym.iperm[prob.bcol[s]])
            slot = C.c_int64()
            _lib.check(lib.feti_add_subdomain(ctx, sym.n, first.shape[0], _lib.i64ptr(first),
                                              _lib.f64ptr(prob.bval[s]), _lib.i64ptr(prob.gids[s]),
                                              _lib.i64ptr(sym.up), _lib.i64ptr(sym.ui), sym.nnz, C.byref(slot)))
            syms.append((sym, vals))
        _lib.check(lib.feti_finalize(ctx, prob.n_multipliers))
        for s, (sym, vals) in enumerate(syms):
            _lib.check(lib.feti_set_factor(ctx, s, C.c_void_p(vals.ctypes.data), vals.shape[0], 0))
        _lib.check(lib.feti_assemble(ctx))
        fms = []
        for s, (sym, vals) in enumerate(syms):
            m = prob.gids[s].shape[0]
            out = np.empty((m, m))
            _lib.check(lib.feti_local_operator(ctx, s, _lib.f64ptr(out)))
            ref = ora.assemble_explicit_local(sym.up, sym.ui, vals, sym.n, sym.iperm, prob.bcol[s], prob.bval[s])
            assert np.linalg.norm(out - ref) <= 1e-10 * np.linalg.norm(ref)
            fms.append(ref)
        p = np.random.default_rng(3).normal(size=prob.n_multipliers)
        q = np.empty(prob.n_multipliers)
        _lib.check(lib.feti_apply(ctx, _lib.f64ptr(p), _lib.f64ptr(q)))
        qr = ora.apply_explicit(fms, prob.gids, p)
        assert np.linalg.norm(q - qr) <= 1e-10 * np.linalg.norm(qr)
    finally:
        lib.feti_destroy(ctx)


def test_bit_reproducible_assembly_and_apply():
    # reference: repeat preprocess is bit-identical (test_dualop.py:108-115),
    # apply is bit-identical across workers/stagings (test_dualop.py:310-333)
    prob = inputs.Problem("heat", 3, 4, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    p = np.random.default_rng(4).normal(size=prob.n_multipliers)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        first = [op.local_operator(i) for i in range(prob.n_sub)]
        q1 = op.apply(p)
        op.preprocess()
        for i in range(prob.n_sub):
            assert np.array_equal(first[i], op.local_operator(i))
        assert np.array_equal(q1, op.apply(p))
    with dualop.prepare(mats, cons, lay, CFG.replace(staging="cluster_wide"), workers=4) as op2:
        op2.preprocess()
        assert np.array_equal(q1, op2.apply(p))


def test_lifecycle_and_errors():
    prob = inputs.Problem("heat", 2, 3, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        with pytest.raises(dualop.LifecycleError):
            op.prepare()
        with pytest.raises(dualop.LifecycleError):
            op.apply(np.zeros(prob.n_multipliers))
        op.preprocess()
        with pytest.raises(ValueError):
            op.apply(np.zeros(prob.n_multipliers + 1))
        assert op.symbolic_count == prob.n_sub
        assert op.numeric_count == prob.n_sub
        op.preprocess()
        assert op.numeric_count == 2 * prob.n_sub
    bad = [inputs.Csr(k.shape, k.indptr, k.indices, -k.data) for k in mats]
    with dualop.prepare(mats, cons, lay, CFG) as op:
        with pytest.raises(dualop.SpdError, match="subdomain 0"):
            op.preprocess(bad)

    class TinyPool:
        capacity = 1024

    with pytest.raises(dualop.PoolCapacityError):
        dualop.prepare(mats, cons, lay, CFG, pool=TinyPool())


def test_single_subdomain_is_local_operator():
    # test_dualop.py:262-271
    prob = inputs.Problem("heat", 2, 4, 1)
    mats, cons, lay = inputs.reference_inputs(prob)
    p = np.random.default_rng(2).normal(size=prob.n_multipliers)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        q = op.apply(p)
        full = _full(op.local_operator(0))
        assert np.linalg.norm(q - full @ p) <= 1e-12 * np.linalg.norm(q)
        w = np.linalg.eigvalsh(full)
        assert w.min() >= -1e-10 * np.linalg.norm(full)


@pytest.mark.parametrize("cfg", ["c1"])
def test_c1_full_problem(cfg):
    g = load_golden("heat2d_c1")
    prob = inputs.Problem(*inputs.CONFIGS[cfg])
    mats, cons, lay = inputs.reference_inputs(prob)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        q = op.apply(g["p"])
    assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])


def test_apply_device_on_torch_stream_matches_host_apply():
    torch = pytest.importorskip("torch")
    prob = inputs.Problem("heat", 3, 4, 2)
    mats, cons, lay = inputs.reference_inputs(prob)
    p = np.random.default_rng(9).normal(size=prob.n_multipliers)
    with dualop.prepare(mats, cons, lay, CFG, device=0) as op:
        op.preprocess()
        q_host = op.apply(p)
        pd = torch.from_numpy(p).cuda()
        qd = torch.full_like(pd, np.nan)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            op.apply_device(pd, qd)          # current (side) stream
            out = qd.cpu().numpy()
        assert np.array_equal(out, q_host)
        qd.fill_(np.nan)
        op.apply_device(pd, qd, stream=torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(qd.cpu().numpy(), q_host)


def _single(prob, s):
    """One-subdomain view with multipliers renumbered 0..m-1 (ConstraintSet.restricted_to)."""
    m = prob.gids[s].shape[0]
    mat = inputs.Csr((m, prob.n_dofs), np.arange(m + 1, dtype=np.int64), prob.bcol[s], prob.bval[s])
    cons = inputs.ConstraintSet(m, np.zeros(m), [inputs.SubdomainConstraints(np.arange(m, dtype=np.int64), mat)])
    lay = inputs.ClusterLayout([inputs.Cluster(0, np.array([0]), np.arange(m), [np.arange(m)])], m)
    return cons, lay


@pytest.mark.parametrize("ordering", ["rcm", "interface_last"])
def test_c3_subdomain_checksums_match_reference(ordering):
    """A full c3 interior subdomain (n=9261, m=2522) against the reference's own
    F~ (numba factorization + dense-storage assembly, checksums in the fixture)."""
    g = load_golden("c3_sub21")
    prob = inputs.Problem(*inputs.CONFIGS["c3"])
    s = int(g["sub_index"])
    k, _, q = prob.subdomain_system(s)
    mats = [inputs.DenseSym(inputs.regularized_dense(k, q))]
    cons, lay = _single(prob, s)
    with dualop.prepare(mats, cons, lay, CFG, ordering=ordering) as op:
        if ordering == "rcm":
            np.testing.assert_array_equal(op._subs[0].perm, g["perm"])
        op.preprocess()
        f = _full(op.local_operator(0))
    for name, got in (("Fv", f @ g["v"]), ("F_diag", np.diag(f)), ("F_row0", f[0])):
        ref = g[name]
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref), name
    assert abs(np.linalg.norm(f) - float(g["F_fro"])) <= 1e-10 * float(g["F_fro"])


def test_c2_apply_and_pcpg_match_reference():
    """Config 2 (512 subdomains x 729 DOFs, 103,807 multipliers): q = F p and
    the PCPG iteration count (80) of the reference."""
    g = load_golden("heat3d_c2")
    prob = inputs.Problem(*inputs.CONFIGS["c2"])
    assert prob.n_multipliers == int(g["n_multipliers"])
    mats, cons, lay = inputs.reference_inputs(prob, dense=True)
    with dualop.prepare(mats, cons, lay, CFG, workers=8) as op:
        op.preprocess()
        q = op.apply(g["p"])
        assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])
        kernels, forces, cl = [], [], []
        for s in range(prob.n_sub):
            k, f, qk = prob.subdomain_system(s)
            kernels.append(qk)
            forces.append(f)
            cl.append((prob.gids[s], prob.bcol[s], prob.bval[s]))
        gm, e, d, coarse = ora.assemble_dual_system(kernels, forces, cl, prob.n_multipliers, prob.c,
                                                    op.solve_local)
        lam, it = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
    assert it == int(g["pcpg_iterations"]) == 80
    ref = g["pcpg_lambda"]
    assert np.linalg.norm(lam - ref) <= 1e-9 * np.linalg.norm(ref)


def test_c4_interior_subdomain_matches_oracle():
    """Config 4 (3D elasticity, n = 10125) largest-m subdomain (m = 3873): the
    device F~ against the oracle's dense-storage path (factor_to_dense + BLAS
    dtrsm + dsyrk, the reference's call sequence) on the same host factor."""
    prob = inputs.Problem(*inputs.CONFIGS["c4"])
    s = int(np.argmax(prob.m_per_subdomain()))
    k, _, q = prob.subdomain_system(s)
    mats = [inputs.DenseSym(inputs.regularized_dense(k, q))]
    cons, lay = _single(prob, s)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        f = op.local_operator(0)
        sub = op._subs[0]
        up, ui = ora.dense_pattern(sub.n)
        fo = ora.assemble_explicit_local(up, ui, sub.values, sub.n, sub.iperm, prob.bcol[s], prob.bval[s],
                                         storage="dense")
    assert f.shape == (3873, 3873)
    assert np.linalg.norm(f - fo) <= 1e-10 * np.linalg.norm(fo)


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("ordering", ["rcm", "interface_last"])
def test_implicit_device_apply_matches_reference(case, ordering):
    """Implicit strategy on the device (two block sweeps over the assembly's
    scaled factor) vs the reference's implicit apply (dualop.py:504-521) and
    vs the explicit apply (test_dualop.py:215-224 bar: 1e-11)."""
    g = load_golden(case)
    prob, mats, cons, lay = _golden_problem(g)
    with dualop.prepare(mats, cons, lay, CFG, ordering=ordering) as op:
        op.preprocess()
        qi = op.apply_implicit(g["p"])
        qe = op.apply(g["p"])
        qi2 = op.apply_implicit(g["p"])
    assert np.array_equal(qi, qi2)
    assert np.linalg.norm(qi - g["q_implicit"]) <= 1e-11 * np.linalg.norm(g["q_implicit"])
    assert np.linalg.norm(qi - qe) <= 1e-11 * np.linalg.norm(qe)


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("factorization", ["host", "device"])
def test_implicit_strategy_through_the_drop_in(case, factorization):
    """DualOpConfig(strategy="implicit") (the reference's default,
    dualop.py:59): preprocess keeps only the block-scaled factor (no F~, no
    X), apply runs the device sweeps and gives the reference's implicit q
    (test_dualop.py:215-224 bar 1e-11); local_operator is None like the
    reference's; the reference's PCPG takes the same iteration count."""
    g = load_golden(case)
    prob, mats, cons, lay = _golden_problem(g)
    cfg = dualop.DualOpConfig(strategy="implicit")
    kw = {}
    if factorization == "device":
        ks, qs = [], []
        for s in range(prob.n_sub):
            k, _, q = prob.subdomain_system(s)
            ks.append(k)
            qs.append(q)
        kw = dict(factorization="device", stiffness=ks, kernels=qs)
        mats = [inputs.ShapeOnly(m.shape) for m in mats]
    with dualop.prepare(mats, cons, lay, cfg, **kw) as op:
        op.preprocess()
        assert op.stats()["flops_trsm_exec"] == 0.0
        q = op.apply(g["p"])
        assert op.local_operator(0) is None
        qk, fk = [], []
        for s in range(prob.n_sub):
            _, f, qb = prob.subdomain_system(s)
            qk.append(qb)
            fk.append(f)
        cons_o = [(prob.gids[s], prob.bcol[s], prob.bval[s]) for s in range(prob.n_sub)]
        gm, e, d, coarse = ora.assemble_dual_system(qk, fk, cons_o, prob.n_multipliers, prob.c, op.solve_local)
        _, it = ora.pcpg(gm, e, d, coarse, op.apply, tol=1e-9)
    assert np.linalg.norm(q - g["q_implicit"]) <= 1e-11 * np.linalg.norm(g["q_implicit"])
    assert it in expected_iterations(case, g)


def test_schur_oracle_strategy_keeps_the_cap():
    """strategy="schur_oracle": the reference's dense oracle semantics --
    SizeCapError above schur_cap DOFs (dualop.py:533-534), otherwise the
    reference's F~ (served by the device assembly)."""
    g = load_golden("heat2d_3x2")
    prob, mats, cons, lay = _golden_problem(g)
    cfg = dualop.DualOpConfig(strategy="schur_oracle")
    with dualop.prepare(mats, cons, lay, cfg, schur_cap=10) as op:
        with pytest.raises(dualop.SizeCapError):
            op.preprocess()
    with dualop.prepare(mats, cons, lay, cfg) as op:
        op.preprocess()
        q = op.apply(g["p"])
    assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])


@pytest.mark.parametrize("sb", [None, 1, 2, 3])
@pytest.mark.parametrize("warps", [1, 3, 5, 6, 7, 8])
def test_apply_any_warp_count_matches_reference(warps, sb, monkeypatch):
    """The apply kernel with any warp count per CTA and any super-block edge
    (None: one compact block per subdomain; 1-3 tiles: many off-diagonal
    super-blocks and segments on this small case) gives the reference's q."""
    monkeypatch.setenv("FETI_APPLY_WARPS", str(warps))
    if sb is not None:
        monkeypatch.setenv("FETI_APPLY_SB", str(sb))
    g = load_golden(SMALL_CASES[-1])
    prob, mats, cons, lay = _golden_problem(g)
    with dualop.prepare(mats, cons, lay, CFG) as op:
        op.preprocess()
        q = op.apply(g["p"])
    assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])


def test_apply_without_multiplier_limit():
    """Two subdomains with m = 15,500 and 2,100 multipliers (the round-1
    kernel capped m at ~14.5k: (NW+1) M doubles of shared memory) through
    the apply kernels, via the C-ABI's explicit-tile entry
    (feti_set_preconditioner + feti_precond_apply run the same SYMV + gather/
    scatter + ordered reduction as feti_apply): q = sum_i B~_i^T P_i B~_i p
    against numpy (symv_upper semantics, _kernels.py:274-287)."""
    lib = _lib.load()
    ctx = C.c_void_p()
    _lib.check(lib.feti_create(0, C.byref(ctx)))
    rng = np.random.default_rng(21)
    n_mult = 17000
    sizes = (15500, 2100)
    try:
        _lib.check(lib.feti_set_strategy(ctx, _lib.FETI_STRATEGY_IMPLICIT))   # no F~/X workspace needed
        subs = []
        for m in sizes:
            n = m + 3
            gids = np.sort(rng.choice(n_mult, size=m, replace=False)).astype(np.int64)
            first = rng.permutation(n)[:m].astype(np.int64)
            sign = rng.choice([-1.0, 1.0], size=m)
            slot = C.c_int64()
            _lib.check(lib.feti_add_subdomain(ctx, n, m, _lib.i64ptr(first), _lib.f64ptr(sign), _lib.i64ptr(gids),
                                              None, None, n * (n + 1) // 2, C.byref(slot)))
            subs.append((slot.value, m, gids))
        _lib.check(lib.feti_finalize(ctx, n_mult))
        mats = []
        for slot, m, gids in subs:
            a = rng.standard_normal((m, m))
            a = np.ascontiguousarray(a + a.T)
            _lib.check(lib.feti_set_preconditioner(ctx, slot, _lib.f64ptr(a)))
            mats.append((a, gids))
            del a
        p = rng.standard_normal(n_mult)
        q = np.empty(n_mult)
        _lib.check(lib.feti_precond_apply(ctx, _lib.f64ptr(p), _lib.f64ptr(q)))
        qr = np.zeros(n_mult)
        for a, gids in mats:
            qr[gids] += a @ p[gids]
        assert np.linalg.norm(q - qr) <= 1e-12 * np.linalg.norm(qr)
    finally:
        lib.feti_destroy(ctx)


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("factorization", ["host", "device", "sparse"])
def test_trsm_path_matches_reference(case, factorization):
    """config.path="trsm" (the reference's default path, dualop.py:472-479):
    the second triangular solve Y = L^-T X on the device (transposed trailing
    tiles, backward DMMA chains) and the row gather F = B~ Y instead of the
    SYRK.  Every F~_i and q against the reference (north-star bar 1e-10) on
    the three factor routes; F~ agrees with the SYRK path to rounding."""
    g = load_golden(case)
    prob, mats, cons, lay = _golden_problem(g)
    kw = {}
    if factorization != "host":
        ks, qs = [], []
        for s in range(prob.n_sub):
            k, _, q = prob.subdomain_system(s)
            ks.append(k)
            qs.append(q)
        kw = dict(factorization=factorization, stiffness=ks, kernels=qs, device=0)
        mats = [inputs.ShapeOnly(m.shape) for m in mats]
    fs = {}
    for path in ("trsm", "syrk"):
        with dualop.prepare(mats, cons, lay, dualop.DualOpConfig(strategy="explicit", path=path), **kw) as op:
            op.preprocess()
            fs[path] = [op.local_operator(s) for s in range(prob.n_sub)]
            q = op.apply(g["p"])
            if path == "trsm":
                assert op.stats()["flops_syrk_exec"] == 0.0
                assert np.linalg.norm(q - g["q_explicit"]) <= 1e-10 * np.linalg.norm(g["q_explicit"])
    for s in range(prob.n_sub):
        m = prob.gids[s].shape[0]
        ref = np.zeros((m, m))
        ref[np.triu_indices(m)] = g[f"s{s}_F_upper"]
        f = fs["trsm"][s]
        assert np.all(np.tril(f, -1) == 0.0)
        assert np.linalg.norm(f - ref) <= 1e-10 * np.linalg.norm(ref), (case, s)
        assert np.linalg.norm(f - fs["syrk"][s]) <= 1e-12 * np.linalg.norm(ref)
