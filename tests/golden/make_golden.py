"""Generate golden fixtures by running the UNMODIFIED reference (tfeti) here.

This script only runs in the build container, where /root/reference exists.
It imports the reference read-only (no-write recipe of SURVEY.md §8c):

    cd /tmp && NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python /root/repo/tests/golden/make_golden.py <case> [...]

The reference calls ``DualOperator._temp`` (dualop.py:331, 448) which it never
defines (only ``_temp_group``, dualop.py:164-187); the 4-line shim below adds
it from outside, exactly as SURVEY.md §0.3 describes.  Nothing in the
reference tree is modified.

Fixtures written to tests/golden/<case>.npz (small problems keep full F~_i;
large ones keep only size-independent checksums):

* per subdomain: n, m, gids (multiplier_ids), B~ rows as (col, val) with one
  nonzero per row (decomposition.py:184-207), the reference symbolic
  permutation (sparse.py:340-415), the stiffness K (CSR) for the
  input-generator parity check, F~_i upper triangle (dualop.py:427-485)
* q = F p for p = default_rng(0).normal(n_mult) through DualOperator.apply
  (dualop.py:348-380), explicit and implicit
* PCPG through solver.run_steps (solver.py:404-449): iterations, lambda,
  u_global, for explicit/syrk
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tfeti.dualop as d

    if not hasattr(d.DualOperator, "_temp"):
        def _temp(self, shape, order="C"):
            region, arrays = self._temp_group([(tuple(shape), order)])
            return region, arrays[0]

        d.DualOperator._temp = _temp
    import tfeti

    return tfeti


def _sub_arrays(cons, i):
    sc = cons.per_subdomain[i]
    ip, ix, dt = sc.matrix.row_arrays()
    assert np.all(np.diff(ip) == 1), "B~ rows carry exactly one nonzero"
    return sc.multiplier_ids.astype(np.int64), ix.astype(np.int64), dt.astype(np.float64)


def _upper_packed(f):
    iu = np.triu_indices(f.shape[0])
    return f[iu]


def small_case(name, physics, dim, cells, subs, clusters=1, pcpg=True, keep_f=True):
    tfeti = _import_reference()
    from tfeti import dualop as dop
    from tfeti import sparse as sp

    t0 = time.time()
    prob = tfeti.build_problem(physics, dim, cells, subs, n_clusters=clusters)
    subp = prob.subdomain_problems()
    cons = prob.constraints
    n_mult = cons.n_multipliers
    out = {
        "physics": np.array(physics), "dim": np.array(dim), "cells": np.array(cells),
        "subs": np.array(subs), "clusters": np.array(clusters),
        "n_multipliers": np.array(n_mult), "c": cons.c.astype(np.float64),
        "n_sub": np.array(prob.n_subdomains),
    }
    cfg = dop.DualOpConfig(strategy="explicit", path="syrk")
    kregs = [s.stiffness_reg for s in subp]
    with dop.prepare(kregs, cons, prob.layout, cfg) as state:
        state.preprocess()
        p = np.random.default_rng(0).normal(size=n_mult)
        out["p"] = p
        out["q_explicit"] = state.apply(p).copy()
        for i in range(prob.n_subdomains):
            gids, bcol, bval = _sub_arrays(cons, i)
            out[f"s{i}_gids"] = gids
            out[f"s{i}_bcol"] = bcol
            out[f"s{i}_bval"] = bval
            out[f"s{i}_perm"] = state._subs[i].symbolic.perm.astype(np.int64)
            out[f"s{i}_factor_nnz"] = np.array(state._subs[i].symbolic.nnz)
            k = subp[i].stiffness
            out[f"s{i}_k_indptr"] = k.indptr
            out[f"s{i}_k_indices"] = k.indices
            out[f"s{i}_k_data"] = k.data
            out[f"s{i}_force"] = subp[i].force
            out[f"s{i}_kernel"] = subp[i].kernel
            if keep_f:
                out[f"s{i}_F_upper"] = _upper_packed(state.local_operator(i))
    with dop.prepare(kregs, cons, prob.layout, dop.DualOpConfig(strategy="implicit")) as st2:
        st2.preprocess()
        out["q_implicit"] = st2.apply(out["p"]).copy()
    if pcpg:
        rep = tfeti.run_steps(prob, 1, config=cfg, tol=1e-9)[0]
        out["pcpg_iterations"] = np.array(rep.iterations)
        out["pcpg_lambda"] = rep.lam
        out["pcpg_u_global"] = rep.u_global
        out["pcpg_residual"] = np.array(rep.residual)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: {prob.n_subdomains} subdomains x {prob.dofs_per_subdomain} dofs, "
          f"{n_mult} multipliers, {time.time() - t0:.1f}s", flush=True)


def big_case(name, physics, dim, cells, subs):
    """Large problem: per-subdomain metadata + apply checksum + PCPG result."""
    tfeti = _import_reference()
    from tfeti import dualop as dop

    t0 = time.time()
    prob = tfeti.build_problem(physics, dim, cells, subs)
    cons = prob.constraints
    n_mult = cons.n_multipliers
    out = {"physics": np.array(physics), "dim": np.array(dim), "cells": np.array(cells),
           "subs": np.array(subs), "n_multipliers": np.array(n_mult),
           "n_sub": np.array(prob.n_subdomains), "c": cons.c}
    ms = np.array([sc.multiplier_ids.shape[0] for sc in cons.per_subdomain])
    out["m_per_sub"] = ms
    # gids flattened (CSR by subdomain) and B~ column/value per row
    out["gids_ptr"] = np.concatenate([[0], np.cumsum(ms)])
    g, bc, bv = [], [], []
    for i in range(prob.n_subdomains):
        a, b, c = _sub_arrays(cons, i)
        g.append(a), bc.append(b), bv.append(c)
    out["gids"] = np.concatenate(g)
    out["bcol"] = np.concatenate(bc)
    out["bval"] = np.concatenate(bv)
    print(f"{name}: build {time.time() - t0:.1f}s", flush=True)
    cfg = dop.DualOpConfig(strategy="explicit", path="syrk", forward_storage="dense",
                           forward_order="col", rhs_order="row")
    rep = tfeti.run_steps(prob, 1, config=cfg, tol=1e-9, workers=os.cpu_count())[0]
    out["pcpg_iterations"] = np.array(rep.iterations)
    out["pcpg_lambda"] = rep.lam
    out["pcpg_residual"] = np.array(rep.residual)
    out["pcpg_u_norm"] = np.array(rep.u_norm)
    print(f"{name}: pcpg {rep.iterations} it, {time.time() - t0:.1f}s", flush=True)
    subp = prob.subdomain_problems()
    with dop.prepare([s.stiffness_reg for s in subp], cons, prob.layout, cfg,
                     workers=os.cpu_count()) as state:
        state.preprocess()
        p = np.random.default_rng(0).normal(size=n_mult)
        out["p"] = p
        out["q_explicit"] = state.apply(p).copy()
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: done {time.time() - t0:.1f}s", flush=True)


def c3_subdomain(name="c3_sub21", sub_index=21, physics="heat", dim=3, cells=20, subs=4):
    """One c3-sized subdomain through the reference's own factorization and
    assembly (numba chol_numeric ~6 min).  Keeps checksums of F~_i only."""
    tfeti = _import_reference()
    from tfeti import decomposition as dc
    from tfeti import dualop as dop
    from tfeti import mesh as mm
    from tfeti import solver as sl
    from tfeti import sparse as sp

    t0 = time.time()
    mesh = mm.generate_mesh(dim, cells * subs, physics)
    dirichlet = mm.dirichlet_dofs(mesh, "x=0")
    part = dc.partition(mesh, subs)
    cons = dc.build_constraints(part, dirichlet)
    print(f"{name}: partition+constraints {time.time() - t0:.1f}s", flush=True)
    sub = part.subdomains[sub_index]
    k = mm.assemble_system(sub.mesh).stiffness
    kernel = sl.build_kernel(physics, sub.mesh)
    kreg = sp.regularize(k, kernel)
    sym = sp.symbolic_factorize(kreg)
    print(f"{name}: regularize+symbolic {time.time() - t0:.1f}s nnz={sym.nnz}", flush=True)
    fac = sp.numeric_factorize(sym, kreg)
    print(f"{name}: numeric {time.time() - t0:.1f}s", flush=True)
    sc = cons.per_subdomain[sub_index]
    cfg = dop.DualOpConfig(strategy="explicit", path="syrk", forward_storage="dense",
                           forward_order="col", rhs_order="row")
    t1 = time.time()
    f = dop.assemble_explicit_local(fac, sc.matrix, cfg)
    t_asm = time.time() - t1
    full = f + np.triu(f, 1).T
    m = full.shape[0]
    v = np.random.default_rng(7).normal(size=m)
    gids, bcol, bval = _sub_arrays(cons, sub_index)
    out = {
        "n": np.array(kreg.shape[0]), "m": np.array(m), "gids": gids, "bcol": bcol, "bval": bval,
        "perm": sym.perm, "factor_nnz": np.array(sym.nnz),
        "v": v, "Fv": full @ v, "F_diag": np.diag(full).copy(), "F_row0": full[0].copy(),
        "F_fro": np.array(np.linalg.norm(full)), "F_trace": np.array(np.trace(full)),
        "t_assemble_dense_s": np.array(t_asm), "n_multipliers": np.array(cons.n_multipliers),
        "k_indptr": k.indptr, "k_indices": k.indices, "k_data": k.data,
        "sub_index": np.array(sub_index),
    }
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: done {time.time() - t0:.1f}s (assembly {t_asm:.2f}s)", flush=True)


CASES = {
    "heat2d_3x2": lambda: small_case("heat2d_3x2", "heat", 2, 3, 2, clusters=2),
    "heat2d_c1": lambda: small_case("heat2d_c1", "heat", 2, 16, 4, clusters=4),
    "heat3d_4x2": lambda: small_case("heat3d_4x2", "heat", 3, 4, 2, clusters=2),
    "elast2d_4x2": lambda: small_case("elast2d_4x2", "elasticity", 2, 4, 2),
    "elast3d_4x2": lambda: small_case("elast3d_4x2", "elasticity", 3, 4, 2, clusters=2),
    "heat3d_c2": lambda: big_case("heat3d_c2", "heat", 3, 8, 8),
    "c3_sub21": lambda: c3_subdomain(),
}

if __name__ == "__main__":
    names = sys.argv[1:] or [k for k in CASES if k not in ("heat3d_c2", "c3_sub21")]
    for nm in names:
        CASES[nm]()
