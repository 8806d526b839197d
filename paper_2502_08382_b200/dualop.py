"""Drop-in explicit dual operator on B200 (replaces tfeti.dualop for that path).

Mirrors the object interface of the reference's ``DualOperator``
(pkg/src/tfeti/dualop.py:114-419) -- constructor, ``prepare`` /
``preprocess`` / ``apply`` lifecycle, ``solve_local``, ``local_operator``,
counters, context manager -- for ``strategy="explicit"``.  The reference's
solver (solver.py:195-272, 404-449) and bench (bench.py:229-246) drive it
unchanged through duck typing.

Where the work runs:

* ``prepare`` (dualop.py:212-269): symbolic stage on the host (RCM
  ordering, or an explicit one), B~ permutation as first-row indices,
  registration with the device context, device allocation.
* ``preprocess`` (dualop.py:301-327): numeric factorization on the host
  (LAPACK, threaded; timed separately by the caller), asynchronous factor
  upload, then the device assembly TRSM+SYRK of every F~_i
  (assemble_explicit_local, dualop.py:427-501) through the C-ABI.
* ``apply`` (dualop.py:348-388): one batched packed-SYMV kernel fused with
  the B~ gather/scatter plus an ordered reduction, on the device.

There is no CPU fallback: without the CUDA library every entry point raises.
"""

from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, fields

import numpy as np

from . import _lib
from . import factor as fct
from . import sparse_route as spr

STRATEGIES = ("implicit", "explicit", "schur_oracle")
PATHS = ("trsm", "syrk")
STORAGES = ("sparse", "dense")
ORDERS = ("row", "col")
STAGINGS = ("per_subdomain", "cluster_wide")
ORDERINGS = ("rcm", "interface_last")

SpdError = fct.SpdError


class LifecycleError(RuntimeError):
    """Operation called out of the prepare -> preprocess -> apply order (dualop.py:47-48)."""


class PoolCapacityError(MemoryError):
    """Device memory (or the caller's pool budget) cannot hold the operator (pool.py)."""


class SingularFactorError(ArithmeticError):
    """A triangular factor carries a zero diagonal entry (sparse.py:42-43)."""


class SizeCapError(ValueError):
    """schur_oracle on a subdomain above ``schur_cap`` DOFs (dualop.py:51-52, 533-534)."""


class _Shape:
    """Shape-only stand-in for K_reg on the device-factor routes (never densified)."""

    def __init__(self, shape):
        self.shape = tuple(int(v) for v in shape)


def _multiplier_owners(constraints):
    """(first, second) owning subdomain of every multiplier (-1: a Dirichlet
    row has one owner)."""
    nm = int(constraints.n_multipliers)
    first = np.full(nm, -1, np.int64)
    second = np.full(nm, -1, np.int64)
    for s, sc in enumerate(constraints.per_subdomain):
        g = np.asarray(sc.multiplier_ids, np.int64)
        taken = first[g] >= 0
        second[g[taken]] = s
        first[g[~taken]] = s
    return first, second


def _problem_like(x) -> bool:
    """A ``SubdomainProblem`` (solver.py:100-106) or anything carrying the
    unregularized ``stiffness`` and its ``kernel`` basis."""
    return hasattr(x, "stiffness") and hasattr(x, "kernel")


@dataclass(frozen=True)
class DualOpConfig:
    """Same fields and validation as the reference (dualop.py:55-82).

    ``strategy``: "explicit" assembles F~_i on the device; "implicit" keeps
    only the block-scaled factor and runs two triangular sweeps per apply on
    the device (apply_implicit_local, dualop.py:504-521); "schur_oracle" is
    the reference's dense test oracle for F~ (dualop.py:524-549) -- it keeps
    the oracle's size cap and is served by the explicit device assembly (the
    same F~ to rounding, strategy invariance test_dualop.py:297-308).
    ``path``: "syrk" forms F~ = X^T X; "trsm" (the reference's default) runs
    the second triangular solve Y = L^-T X and the row gather B~ Y on the
    device like the reference (dualop.py:472-479) -- the same F~_i to
    roundoff (test_dualop.py:143-149) at about twice the flops; bench.py uses
    "syrk".  The storage/order knobs select
    CPU kernel variants in the reference; the device has one tiled layout, so
    they are accepted and have no effect on the result (all variants agree to
    <=1e-12, test_dualop.py:160-176).
    """

    strategy: str = "implicit"
    path: str = "trsm"
    forward_storage: str = "sparse"
    backward_storage: str = "sparse"
    forward_order: str = "row"
    backward_order: str = "row"
    rhs_order: str = "row"
    staging: str = "per_subdomain"

    def __post_init__(self):
        checks = (
            ("strategy", STRATEGIES), ("path", PATHS),
            ("forward_storage", STORAGES), ("backward_storage", STORAGES),
            ("forward_order", ORDERS), ("backward_order", ORDERS),
            ("rhs_order", ORDERS), ("staging", STAGINGS),
        )
        for name, allowed in checks:
            if getattr(self, name) not in allowed:
                raise ValueError(f"{name} must be one of {allowed}, got {getattr(self, name)!r}")

    def replace(self, **kw) -> "DualOpConfig":
        vals = {f.name: getattr(self, f.name) for f in fields(self)}
        vals.update(kw)
        return DualOpConfig(**vals)


def _raise_from(err: _lib.FetiError):
    msg = str(err)
    if err.code == _lib.FETI_ERR_LIFECYCLE:
        raise LifecycleError(msg) from None
    if err.code == _lib.FETI_ERR_CAPACITY:
        raise PoolCapacityError(msg) from None
    if err.code == _lib.FETI_ERR_SINGULAR:
        raise SingularFactorError(msg) from None
    if err.code == _lib.FETI_ERR_ARG:
        raise ValueError(msg) from None
    raise RuntimeError(msg) from None


def _call(rc):
    try:
        _lib.check(rc)
    except _lib.FetiError as err:
        _raise_from(err)


def _constraint_rows(sc, n):
    """(local dof, value) of the single nonzero of each B~_i row."""
    mat = sc.matrix
    if hasattr(mat, "row_arrays"):
        ip, ix, dt = mat.row_arrays()
    else:
        m = mat.tocsr()
        ip, ix, dt = m.indptr, m.indices, m.data
    ip = np.asarray(ip, np.int64)
    if mat.shape[1] != n:
        raise ValueError("constraint matrix width does not match the factor")
    if np.any(np.diff(ip) != 1):
        raise ValueError("each B~ row must carry exactly one nonzero (decomposition.py:184-207)")
    return np.asarray(ix, np.int64), np.asarray(dt, np.float64)


class _Sub:
    __slots__ = ("index", "n", "m", "gids", "bcol", "bval", "perm", "iperm", "slot", "values", "pinned",
                 "cluster", "fix", "diagpos", "kcache", "npos")


class DualOperator:
    """Lifecycle-managed explicit dual operator on one B200 (one cluster = one GPU).

    Parameters follow the reference (dualop.py:124-126); extra keywords:

    * ``device``: CUDA device index (default: current torch device or 0)
    * ``ordering``: ``"rcm"`` reproduces the reference's symbolic permutation;
      ``"interface_last"`` orders constrained DOFs last (same F~ to rounding,
      far less forward-solve work)
    * ``subdomains``: restrict the operator to these subdomain indices (the
      ones of this rank's cluster); ``apply`` then returns this rank's
      contribution, summed across ranks by :mod:`.distributed`
    * ``pinned``: stage host factors in page-locked memory (default True)
    * ``perms``: explicit per-subdomain orderings (mapping or sequence indexed
      by subdomain), as ``symbolic_factorize(ordering=<array>)`` accepts
      (sparse.py:368-371); overrides ``ordering``
    * ``matrices`` may also be ``SubdomainProblem``-like objects (attributes
      ``stiffness`` and ``kernel``, solver.py:100-106): the operator then
      takes K_i and its kernel basis from them and defaults to the sparse
      route (``prepare_from_problems``)
    * ``factorization``: ``"host"`` (LAPACK on the host, the factor is
      uploaded) or ``"device"``: K_reg = K + rho Q Q^T is formed from the
      unregularized sparse ``stiffness[i]`` and the kernel basis
      ``kernels[i]`` and factored on the GPU (DMMA blocked Cholesky); the
      factor never crosses PCIe.  With the reference's dense K_reg the RCM
      ordering is the reversed natural order, which device mode uses.
      ``"sparse"``: the sparse-factor route (sparse_route.py): K_s = K +
      rho E E^T with fixing DOFs E is factored on the GPU into block-sparse
      tiles (constrained DOFs last, interior onion-ordered) and the exact
      rank-2r correction recovers the reference's F~_i; the dense K_reg is
      never formed, so ``matrices`` may be shape-only stand-ins.
    """

    def __init__(self, matrices, constraints, layout, config: DualOpConfig, pool=None, workers: int = 1,
                 schur_cap: int = 2000, device: int | None = None, ordering: str = "rcm",
                 subdomains=None, pinned: bool = True, perms=None, factorization: str | None = None,
                 stiffness=None, kernels=None, sparse_ordering: str = "auto", forces=None):
        matrices = list(matrices)
        if len(matrices) != len(constraints.per_subdomain):
            raise ValueError("one stiffness matrix per subdomain required")
        if matrices and all(_problem_like(x) for x in matrices):
            # SubdomainProblem inputs: K_i and ker K_i straight from the caller
            stiffness = [x.stiffness for x in matrices] if stiffness is None else stiffness
            kernels = [x.kernel for x in matrices] if kernels is None else kernels
            if forces is None and all(hasattr(x, "force") for x in matrices):
                forces = [x.force for x in matrices]
            factorization = factorization or "sparse"
            if factorization != "sparse":
                forces = None
            matrices = ([x.stiffness_reg for x in matrices] if factorization == "host"
                        else [_Shape(x.stiffness.shape) for x in matrices])
        factorization = factorization or "host"
        if ordering not in ORDERINGS:
            raise ValueError(f"ordering must be one of {ORDERINGS}")
        self.matrices = list(matrices)
        self.constraints = constraints
        self.layout = layout
        self.config = config
        self.pool = pool
        self.workers = max(1, int(workers))
        self.schur_cap = int(schur_cap)
        self.n_subdomains = len(self.matrices)
        self.n_multipliers = int(constraints.n_multipliers)
        self.ordering = ordering
        self.pinned = bool(pinned)
        self.device = device
        self.perms = perms
        if factorization not in ("host", "device", "sparse"):
            raise ValueError("factorization must be 'host', 'device' or 'sparse'")
        self.factorization = factorization
        self.stiffness = None if stiffness is None else list(stiffness)
        self.kernels = None if kernels is None else list(kernels)
        if factorization in ("device", "sparse") and (self.stiffness is None or self.kernels is None):
            raise ValueError(f"{factorization} factorization needs stiffness= and kernels= per subdomain")
        # loads f_i: on the sparse route they are factored along (an appended
        # row) so that d = B~ K^+ f comes out of the device (dual_rhs)
        self.forces = None if forces is None else list(forces)
        self._forces_dev = None
        self.owned = (list(range(self.n_subdomains)) if subdomains is None
                      else sorted(int(s) for s in subdomains))
        if not (sparse_ordering in ("auto", "onion") or sparse_ordering.startswith(("dissection:", "faces:"))):
            raise ValueError("sparse_ordering must be 'auto', 'onion', 'dissection:<depth>' or 'faces:<depth>'")
        self.sparse_ordering = sparse_ordering
        self.sparse_recipe = None

        self.prepared = False
        self.step_ready = False
        self.symbolic_count = 0
        self.numeric_count = 0
        self.external_temp_allocs = 0
        self.persistent_bytes = 0

        self._subs: dict[int, _Sub] = {}
        self._ctx = None
        self._lib = _lib.load()
        self._executor = None
        self._upload_pool = None
        self._handed_over = False
        self.timings = {}

    # -- helpers -------------------------------------------------------------

    def _map(self, fn, items):
        items = list(items)
        if self.workers == 1 or len(items) <= 1:
            return [fn(x) for x in items]
        if self._executor is None:
            self._executor = ThreadPoolExecutor(max_workers=self.workers, thread_name_prefix="dualop")
        return list(self._executor.map(fn, items))

    def _gather_order(self):
        """Subdomains in the reference's gather order (dualop.py:375-379)."""
        order = []
        owned = set(self.owned)
        for cluster in self.layout.clusters:
            for s in cluster.subdomain_ids:
                if int(s) in owned:
                    order.append(int(s))
        missing = owned.difference(order)
        order.extend(sorted(missing))
        return order

    def _resolve_device(self):
        if self.device is not None:
            return int(self.device)
        try:
            import torch

            if torch.cuda.is_available():
                return torch.cuda.current_device()
        except Exception:  # noqa: BLE001 - torch is optional plumbing
            pass
        return 0

    def close(self):
        if self._executor is not None:
            self._executor.shutdown(wait=True)
            self._executor = None
        if getattr(self, "_upload_pool", None) is not None:
            self._upload_pool.shutdown(wait=True)
            self._upload_pool = None
        if self._ctx is not None:
            self._lib.feti_destroy(self._ctx)
            self._ctx = None
        for sub in self._subs.values():
            if sub.pinned is not None:
                sub.pinned.free()
                sub.pinned = None
                sub.values = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # -- lifecycle -----------------------------------------------------------

    def prepare(self) -> "DualOperator":
        """Symbolic stage, device registration and allocation, exactly once."""
        if self.prepared:
            raise LifecycleError("prepare was already called on this operator")
        order = self._gather_order()

        def symbolic(i):
            sub = _Sub()
            sub.index = i
            matrix = self.matrices[i]
            sub.n = int(matrix.shape[0])
            sc = self.constraints.per_subdomain[i]
            sub.gids = np.ascontiguousarray(sc.multiplier_ids, dtype=np.int64)
            sub.m = int(sub.gids.shape[0])
            sub.bcol, sub.bval = _constraint_rows(sc, sub.n)
            if self.perms is not None:
                sub.perm = np.ascontiguousarray(self.perms[i], dtype=np.int64)
                if sub.perm.shape != (sub.n,) or not np.array_equal(np.sort(sub.perm), np.arange(sub.n)):
                    raise ValueError(f"subdomain {i}: explicit ordering is not a permutation")
            elif self.factorization == "sparse":
                n, ip, ix, _ = fct.csr_arrays(self.stiffness[i])
                if n != sub.n:
                    raise ValueError("stiffness size does not match the subdomain")
                pieces = self._interface_pieces(i, sub.bcol) if self.sparse_recipe[0] == "faces" else None
                sub.perm, sub.iperm = spr.sparse_route_ordering(n, ip, ix, sub.bcol, self.sparse_recipe, pieces)
                sub.npos = int(sub.perm.shape[0])
            elif self.factorization == "device":
                base = np.arange(sub.n - 1, -1, -1, dtype=np.int64)   # RCM of the dense K_reg
                if self.ordering == "rcm":
                    sub.perm = base
                else:
                    mark = np.zeros(sub.n, bool)
                    mark[sub.bcol] = True
                    sub.perm = np.concatenate([base[~mark[base]], np.sort(np.flatnonzero(mark))])
            elif self.ordering == "rcm":
                sub.perm = fct.rcm_ordering(matrix)
            else:
                sub.perm = fct.interface_last_ordering(matrix, sub.bcol)
            if self.factorization != "sparse":
                sub.iperm = fct.inverse_permutation(sub.perm)
                sub.npos = sub.n
            sub.values = None
            sub.pinned = None
            sub.fix = None
            sub.diagpos = None
            sub.kcache = None
            if self.factorization == "sparse":
                sub.fix = spr.fixing_dofs(self._kernel_basis(i, sub.n))
            return sub

        if self.factorization == "sparse":
            # one ordering recipe for the operator, chosen on its subdomain with
            # the most multipliers by the tile flops it leaves (subdomains of one
            # problem are alike)
            self._owners = _multiplier_owners(self.constraints)
            i0 = max(order, key=lambda i: self.constraints.per_subdomain[i].multiplier_ids.shape[0])
            n0, ip0, ix0, _ = fct.csr_arrays(self.stiffness[i0])
            sc0 = self.constraints.per_subdomain[i0]
            bcol0, _ = _constraint_rows(sc0, n0)
            r0 = self._kernel_basis(i0, n0).shape[1]
            self.sparse_recipe = spr.choose_ordering(n0, ip0, ix0, bcol0, r0, self.sparse_ordering,
                                                     pieces=self._interface_pieces(i0, bcol0))
        subs = self._map(symbolic, order)
        ctx = C.c_void_p()
        _call(self._lib.feti_create(self._resolve_device(), C.byref(ctx)))
        self._ctx = ctx
        for sub in subs:
            first = np.ascontiguousarray(sub.iperm[sub.bcol], dtype=np.int64)
            slot = C.c_int64()
            _call(self._lib.feti_add_subdomain(
                ctx, sub.npos, sub.m, _lib.i64ptr(first), _lib.f64ptr(sub.bval), _lib.i64ptr(sub.gids),
                None, None, fct.packed_size(sub.npos), C.byref(slot)))
            sub.slot = slot.value
            self._subs[sub.index] = sub
        if self.pool is not None and hasattr(self.pool, "capacity") and self.factorization != "sparse":
            need = self.device_bytes_estimate()
            if need > int(self.pool.capacity):
                raise PoolCapacityError(
                    f"pool of {self.pool.capacity} bytes cannot hold the {need}-byte device operator")
        if self.config.strategy == "implicit":
            _call(self._lib.feti_set_strategy(ctx, _lib.FETI_STRATEGY_IMPLICIT))
        elif self.config.path == "trsm":
            # the reference's second solve + row gather (dualop.py:472-479)
            _call(self._lib.feti_set_path(ctx, _lib.FETI_PATH_TRSM))
        if self.factorization == "device":
            _call(self._lib.feti_enable_device_factorization(ctx))
        if self.factorization == "sparse":
            _call(self._lib.feti_enable_sparse_factorization(ctx))
            if self.forces is not None:
                _call(self._lib.feti_enable_dual_rhs(ctx))
            for sub in subs:
                n, ip, ix, _ = fct.csr_arrays(self.stiffness[sub.index])
                ip = np.ascontiguousarray(ip, np.int64)
                ix = np.ascontiguousarray(ix, np.int64)
                fix = np.ascontiguousarray(sub.fix, np.int64)
                _call(self._lib.feti_set_sparse_pattern(ctx, sub.slot, n, _lib.i64ptr(ip), _lib.i64ptr(ix),
                                                        _lib.i64ptr(sub.perm), fix.shape[0], _lib.i64ptr(fix)))
        _call(self._lib.feti_finalize(ctx, self.n_multipliers))
        st = self.stats()
        if self.pool is not None and hasattr(self.pool, "capacity") and self.factorization == "sparse":
            # the block-sparse plan is known only after finalize: the library's own byte count
            need = int(st["bytes_persistent"]) + int(st["bytes_temporary"])
            if need > int(self.pool.capacity):
                raise PoolCapacityError(
                    f"pool of {self.pool.capacity} bytes cannot hold the {need}-byte device operator")
        self.persistent_bytes = int(st["bytes_persistent"])
        self.symbolic_count = len(self._subs)
        self.prepared = True
        return self

    def _interface_pieces(self, i, bcol):
        """Subdomain i's interface faces/edges/corners: constrained DOFs grouped
        by the subdomains their multipliers glue them to."""
        gids = np.asarray(self.constraints.per_subdomain[i].multiplier_ids, np.int64)
        first, second = self._owners
        nb = np.where(first[gids] == i, second[gids], first[gids])
        return spr.interface_pieces(bcol, nb)

    def device_bytes_estimate(self) -> int:
        """Dense-tile routes: factor tile triangle + X panels + packed F~ (the
        sparse route's plan is only known after finalize; prepare() checks it
        against the library's byte count instead)."""
        tot = 0
        for sub in self._subs.values():
            T = -(-sub.n // 128)
            P = -(-sub.m // 128)
            T32 = -(-sub.m // 32)
            tot += (T * (T + 1) // 2 + P * T) * 128 * 128 * 8 + T32 * (T32 + 1) // 2 * 1024 * 8
        return tot

    def _factor_buffer(self, sub):
        if sub.values is None:
            n = fct.packed_size(sub.n)
            if self.pinned:
                sub.pinned = _lib.PinnedArray(n)
                sub.values = sub.pinned.array
            else:
                sub.values = np.empty(n)
        return sub.values

    def preprocess(self, matrices=None, stiffness=None, kernels=None, forces=None) -> None:
        """Numeric factorization (host, or device), then device assembly of every F~_i."""
        import time

        if not self.prepared:
            raise LifecycleError("preprocess before prepare")
        if matrices is not None:
            if len(matrices) != self.n_subdomains:
                raise ValueError("one stiffness matrix per subdomain required")
            matrices = list(matrices)
            if matrices and all(_problem_like(x) for x in matrices):
                stiffness = [x.stiffness for x in matrices] if stiffness is None else stiffness
                kernels = [x.kernel for x in matrices] if kernels is None else kernels
                if forces is None and all(hasattr(x, "force") for x in matrices):
                    forces = [x.force for x in matrices]
                matrices = ([x.stiffness_reg for x in matrices] if self.factorization == "host"
                            else [_Shape(x.stiffness.shape) for x in matrices])
            self.matrices = matrices
        if self.config.strategy == "schur_oracle":
            for sub in self._subs.values():
                if sub.n > self.schur_cap:
                    raise SizeCapError(f"subdomain of {sub.n} DOFs exceeds the dense oracle cap {self.schur_cap}")
        if self.factorization in ("device", "sparse"):
            if stiffness is not None:
                self.stiffness = list(stiffness)
            if kernels is not None:
                self.kernels = list(kernels)
            if forces is not None:
                self.forces = list(forces)
            self._preprocess_device()
            return

        t0 = time.perf_counter()

        def numeric(sub):
            try:
                fct.numeric_factorize_dense(self.matrices[sub.index], sub.perm, out=self._factor_buffer(sub))
            except fct.SpdError as err:
                raise SpdError(f"subdomain {sub.index}: {err}") from err
            return sub

        done = self._map(numeric, self._subs.values())
        t1 = time.perf_counter()
        for sub in done:
            self.set_factor(sub.index, sub.values)
        self.assemble()
        t2 = time.perf_counter()
        self.timings = {"host_factorization_s": t1 - t0, "upload_and_assembly_s": t2 - t1}
        self.numeric_count += len(done)

    def _kernel_basis(self, index: int, n: int, changed: list | None = None) -> np.ndarray:
        """Orthonormal kernel basis as regularize takes it (np.linalg.qr, sparse.py:445-449).

        Cached per subdomain while the caller hands over an unchanged basis
        (the kernel depends on the mesh only; run_steps rebuilds equal arrays);
        ``changed`` (a list) receives whether the basis differs from the cache."""
        src = self.kernels[index]
        sub = self._subs.get(index)
        if sub is not None and sub.kcache is not None and sub.kcache[2] is src:
            # the very object handed over last time: not re-compared (O(n r)
            # per subdomain and step; a changed basis comes as a new array)
            if changed is not None:
                changed.append(False)
            return sub.kcache[1]
        kern = np.asarray(src, dtype=np.float64).reshape(n, -1)
        if sub is not None and sub.kcache is not None and sub.kcache[0].shape == kern.shape \
                and np.array_equal(sub.kcache[0], kern):
            sub.kcache = (sub.kcache[0], sub.kcache[1], src)
            if changed is not None:
                changed.append(False)
            return sub.kcache[1]
        if kern.shape[1] == 0:
            q = np.zeros((n, 0))
        else:
            q = np.ascontiguousarray(np.linalg.qr(kern)[0])
        if sub is not None:
            sub.kcache = (kern.copy(), q, src)
        if changed is not None:
            changed.append(True)
        return q

    def _preprocess_device(self) -> None:
        import time

        t0 = time.perf_counter()
        keep = []          # host buffers the asynchronous copies read until assemble returns

        def hand_over(sub):
            n, ip, ix, dt = fct.csr_arrays(self.stiffness[sub.index])
            if n != sub.n:
                raise ValueError("stiffness size does not match the subdomain")
            q = self._kernel_basis(sub.index, n)
            # diagonal positions: the pattern is frozen after the first step
            # (symbolic once, dualop.py:212-269); equality checks are O(nnz)
            # (the reference refills values into a frozen pattern without
            # re-checking it either; the library verifies indptr)
            if sub.diagpos is None or not (sub.diagpos[0].shape == ip.shape and np.array_equal(sub.diagpos[0], ip)):
                rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
                sub.diagpos = (np.array(ip), None, np.flatnonzero(rows == ix))
            rho = float(dt[sub.diagpos[2]].sum()) / n                 # trace(K)/n (sparse.py:450)
            ip, ix, dt = (np.ascontiguousarray(ip, np.int64), np.ascontiguousarray(ix, np.int64),
                          np.ascontiguousarray(dt, np.float64))
            keep.append((dt, q))
            _call(self._lib.feti_set_stiffness(self._ctx, sub.slot, n, _lib.i64ptr(ip), _lib.i64ptr(ix),
                                               _lib.f64ptr(dt), ip[-1], _lib.f64ptr(q), q.shape[1], rho,
                                               _lib.i64ptr(sub.perm)))
            return sub

        subs = list(self._subs.values())
        if self.factorization == "sparse" and self._handed_over:
            # later steps of the sparse route: one batched call queues every
            # slot's K values (and any changed kernel basis) asynchronously;
            # rho = trace(K)/n is computed on the device (sparse.py:450)
            ns = len(subs)
            slots = np.empty(ns, np.int64)
            data = (C.c_void_p * ns)()
            qptr = (C.c_void_p * ns)()
            nnz = np.empty(ns, np.int64)
            for k, sub in enumerate(subs):
                n, _, _, dt = fct.csr_arrays(self.stiffness[sub.index])
                if dt.dtype != np.float64 or not dt.flags.c_contiguous:
                    dt = np.ascontiguousarray(dt, np.float64)
                changed = []
                q = self._kernel_basis(sub.index, n, changed)
                keep.append((dt, q))
                slots[k] = sub.slot
                data[k] = dt.ctypes.data
                nnz[k] = dt.shape[0]
                qptr[k] = q.ctypes.data if (changed[0] and q.shape[1] > 0) else None
            _call(self._lib.feti_set_stiffness_values(self._ctx, ns, _lib.i64ptr(slots), data,
                                                      _lib.i64ptr(nnz), qptr))
        elif self._handed_over and len(subs) > 1:
            # dense device route, later steps: per-slot hand-overs (host copies of
            # K values and Q; ctypes releases the GIL) on a thread pool
            if self._upload_pool is None:
                from concurrent.futures import ThreadPoolExecutor

                self._upload_pool = ThreadPoolExecutor(max_workers=min(8, len(subs)),
                                                       thread_name_prefix="feti-upload")
            list(self._upload_pool.map(hand_over, subs))
        else:
            for sub in subs:
                hand_over(sub)
            self._handed_over = True
        if self.factorization == "sparse" and self.forces is not None:
            self._hand_over_forces(subs, keep)
        t1 = time.perf_counter()
        self._factorize_and_assemble()
        del keep
        t2 = time.perf_counter()
        self.timings = {"stiffness_upload_s": t1 - t0, "device_factorization_and_assembly_s": t2 - t1,
                        "device_factorization_ms": self.stats()["ms_factorize"]}
        self.numeric_count += len(self._subs)

    def _hand_over_forces(self, subs, keep) -> None:
        """f' = (I - Q Q^T) f and Q^T f per slot (O(n r) on the host), factored
        along with K_s so the dual right-hand side needs no solve_local."""
        ns = len(subs)
        slots = np.empty(ns, np.int64)
        fptr = (C.c_void_p * ns)()
        qptr = (C.c_void_p * ns)()
        for k, sub in enumerate(subs):
            f = np.asarray(self.forces[sub.index], dtype=np.float64)
            q = self._kernel_basis(sub.index, sub.n)
            qtf = np.ascontiguousarray(q.T @ f)
            fp = np.ascontiguousarray(f - q @ qtf)
            keep.append((fp, qtf))
            slots[k] = sub.slot
            fptr[k] = fp.ctypes.data
            qptr[k] = qtf.ctypes.data if qtf.size else None
        _call(self._lib.feti_set_forces(self._ctx, ns, _lib.i64ptr(slots), fptr, qptr))
        self._forces_dev = list(self.forces)

    def _factorize_and_assemble(self) -> None:
        # the sparse route reports a non-SPD pivot from feti_assemble (it
        # checks the pivots once the overlapped factorization/assembly ended)
        for fn in (self._lib.feti_factorize, self._lib.feti_assemble):
            try:
                _lib.check(fn(self._ctx))
            except _lib.FetiError as err:
                self.step_ready = False
                if err.code == _lib.FETI_ERR_NOT_SPD:
                    slot = int(str(err).split()[1].rstrip(":"))
                    index = next(s.index for s in self._subs.values() if s.slot == slot)
                    msg = str(err).split(":", 1)[1].strip()
                    raise SpdError(f"subdomain {index}: {msg}") from None
                _raise_from(err)
        self.step_ready = True

    def preprocess_resident(self) -> None:
        """Refactor and reassemble from the stiffness values already resident on
        the device (the last preprocess's): the device-side step alone, as the
        bench's HBM-resident measurement times it."""
        if self.factorization not in ("device", "sparse") or not self._handed_over:
            raise LifecycleError("preprocess_resident needs a device-factor route after one preprocess")
        self._factorize_and_assemble()

    # -- lower-level entry points (used by preprocess, bench and tests) -------

    def set_factor(self, index: int, values, on_device: bool = False) -> None:
        """Hand over the factor values of one subdomain (reference layout)."""
        if not self.prepared:
            raise LifecycleError("preprocess before prepare")
        sub = self._subs[int(index)]
        if on_device:
            ptr, nnz = int(values.data_ptr()), int(values.numel())
            where = _lib.FETI_FACTOR_DEVICE
        else:
            arr = np.asarray(values)
            if arr.dtype != np.float64 or not arr.flags.c_contiguous:
                raise ValueError("factor values must be contiguous float64")
            if sub.values is not arr:
                sub.values = arr  # keep alive until the async copy completes
            ptr, nnz = arr.ctypes.data, arr.shape[0]
            where = _lib.FETI_FACTOR_HOST
        _call(self._lib.feti_set_factor(self._ctx, sub.slot, C.c_void_p(ptr), nnz, where))
        self.step_ready = False

    def assemble(self) -> None:
        """Device assembly of every F~_i from the factors handed over."""
        if not self.prepared:
            raise LifecycleError("preprocess before prepare")
        _call(self._lib.feti_assemble(self._ctx))
        self.step_ready = True

    # -- application ---------------------------------------------------------

    def apply(self, p, out=None):
        """q = sum_i gather_i(F_i scatter_i(p)) (dualop.py:348-380)."""
        if not self.step_ready:
            raise LifecycleError("apply before preprocess for the current values")
        p = np.ascontiguousarray(p, dtype=np.float64)
        if p.shape != (self.n_multipliers,):
            raise ValueError("dual vector has the wrong length")
        if out is None:
            out = np.zeros(self.n_multipliers)
        if out.dtype != np.float64 or out.shape != (self.n_multipliers,):
            raise ValueError("output vector has the wrong shape or dtype")
        if out.flags.c_contiguous:
            _call(self._lib.feti_apply(self._ctx, _lib.f64ptr(p), _lib.f64ptr(out)))
        else:
            tmp = np.empty(self.n_multipliers)
            _call(self._lib.feti_apply(self._ctx, _lib.f64ptr(p), _lib.f64ptr(tmp)))
            out[:] = tmp
        return out

    def apply_implicit(self, p, out=None):
        """Implicit strategy on the device: q = sum B~ K_reg^-1 B~^T p through
        the factor tiles of the last assembly (dualop.py:504-521 semantics)."""
        if not self.step_ready:
            raise LifecycleError("apply before preprocess for the current values")
        p = np.ascontiguousarray(p, dtype=np.float64)
        if p.shape != (self.n_multipliers,):
            raise ValueError("dual vector has the wrong length")
        if out is None:
            out = np.zeros(self.n_multipliers)
        _call(self._lib.feti_apply_implicit(self._ctx, _lib.f64ptr(p), _lib.f64ptr(out)))
        return out

    def apply_implicit_device(self, p, q, stream=None) -> None:
        if not self.step_ready:
            raise LifecycleError("apply before preprocess for the current values")
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(p.device).cuda_stream
        _call(self._lib.feti_apply_implicit_device(self._ctx, C.c_void_p(int(p.data_ptr())),
                                                   C.c_void_p(int(q.data_ptr())), C.c_void_p(int(stream))))

    def apply_device(self, p, q, stream=None) -> None:
        """q = F p on device tensors (torch CUDA float64), enqueued on ``stream``."""
        if not self.step_ready:
            raise LifecycleError("apply before preprocess for the current values")
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(p.device).cuda_stream
        _call(self._lib.feti_apply_device(self._ctx, C.c_void_p(int(p.data_ptr())),
                                          C.c_void_p(int(q.data_ptr())), C.c_void_p(int(stream))))

    # -- lumped preconditioner (solver.py:155-175) ------------------------------

    def set_lumped_preconditioner(self, stiffness=None) -> None:
        """Upload P_i = B~_i K_i B~_i^T (the unregularized K_i, as
        make_preconditioner("lumped") uses ``SubdomainProblem.stiffness``) for
        every owned subdomain; applied by the explicit apply's kernels."""
        if not self.prepared:
            raise LifecycleError("set_lumped_preconditioner before prepare")
        stiffness = self.stiffness if stiffness is None else list(stiffness)
        if stiffness is None:
            raise ValueError("the lumped preconditioner needs the stiffness matrices")
        from scipy.sparse import csr_matrix

        for sub in self._subs.values():
            n, ip, ix, dt = fct.csr_arrays(stiffness[sub.index])
            k = csr_matrix((dt, ix, ip), shape=(n, n))
            kb = k[sub.bcol][:, sub.bcol].toarray()
            pm = np.ascontiguousarray(sub.bval[:, None] * kb * sub.bval[None, :])
            _call(self._lib.feti_set_preconditioner(self._ctx, sub.slot, _lib.f64ptr(pm)))
        self._lumped = True

    def precond_apply(self, w, out=None):
        """M w = sum_i gather_i(B~_i K_i B~_i^T scatter_i(w)) on the device."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        if w.shape != (self.n_multipliers,):
            raise ValueError("dual vector has the wrong length")
        if out is None:
            out = np.zeros(self.n_multipliers)
        _call(self._lib.feti_precond_apply(self._ctx, _lib.f64ptr(w), _lib.f64ptr(out)))
        return out

    def precond_apply_device(self, w, out, stream=None) -> None:
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(w.device).cuda_stream
        _call(self._lib.feti_precond_apply_device(self._ctx, C.c_void_p(int(w.data_ptr())),
                                                  C.c_void_p(int(out.data_ptr())), C.c_void_p(int(stream))))

    # -- multi-GPU apply with the fused exchange (feti_exchange.cu) -----------

    def exchange_setup(self, rank: int, world: int) -> bytes:
        """Allocate this rank's receive slab; returns its CUDA IPC handle."""
        buf = C.create_string_buffer(_lib.FETI_IPC_HANDLE_BYTES)
        _call(self._lib.feti_exchange_setup(self._ctx, int(rank), int(world), buf))
        return buf.raw

    def exchange_connect(self, handles) -> None:
        """Open every rank's slab (handles in rank order, own included)."""
        blob = b"".join(bytes(h) for h in handles)
        _call(self._lib.feti_exchange_connect(self._ctx, blob))

    def apply_exchange_device(self, p, q, stream=None) -> None:
        """q = sum over ranks of B~^T F~ B~ p, exchanged over peer memory."""
        if not self.step_ready:
            raise LifecycleError("apply before preprocess for the current values")
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(p.device).cuda_stream
        _call(self._lib.feti_apply_exchange_device(self._ctx, C.c_void_p(int(p.data_ptr())),
                                                   C.c_void_p(int(q.data_ptr())), C.c_void_p(int(stream))))

    def exchange_status(self) -> None:
        _call(self._lib.feti_exchange_status(self._ctx))

    # -- K^+ access for the solver --------------------------------------------

    def solve_local(self, index: int, rhs, out=None):
        """x = K_reg^-1 rhs for one subdomain through its factor."""
        if not self.step_ready:
            raise LifecycleError("solve_local before preprocess")
        sub = self._subs[int(index)]
        if self.factorization in ("device", "sparse"):
            x = self.solve_local_many([index], [rhs])[0]
            if out is not None:
                out[:] = x
                return out
            return x
        return fct.solve_packed(sub.values, sub.perm, rhs, out=out)

    def solve_local_many(self, indices, rhs_list):
        """Batched solve_local (one device launch in device-factorization mode)."""
        if not self.step_ready:
            raise LifecycleError("solve_local before preprocess")
        subs = [self._subs[int(i)] for i in indices]
        if self.factorization not in ("device", "sparse"):
            return [fct.solve_packed(s.values, s.perm, r) for s, r in zip(subs, rhs_list)]
        slots = np.array([s.slot for s in subs], dtype=np.int64)
        b = np.ascontiguousarray(np.concatenate([np.asarray(r, dtype=np.float64) for r in rhs_list]))
        x = np.empty_like(b)
        _call(self._lib.feti_solve_many(self._ctx, slots.shape[0], _lib.i64ptr(slots), _lib.f64ptr(b),
                                        _lib.f64ptr(x)))
        out, off = [], 0
        for s in subs:
            out.append(x[off:off + s.n].copy())
            off += s.n
        return out

    def dual_rhs(self, forces) -> np.ndarray:
        """B~ K^+ f summed over the owned subdomains (the d of
        assemble_dual_system without the -c, solver.py:141-143)."""
        if not self.step_ready:
            raise LifecycleError("dual_rhs before preprocess")
        fd = self._forces_dev
        if fd is not None and len(fd) == len(forces) and all(
                a is b or (a is not None and b is not None and np.array_equal(a, b))
                for a, b in ((fd[s.index], forces[s.index]) for s in self._subs.values())):
            # the loads were factored along with K_s: d straight from the device
            d = np.empty(self.n_multipliers)
            _call(self._lib.feti_dual_rhs(self._ctx, None, _lib.f64ptr(d)))
            return d
        d = np.zeros(self.n_multipliers)
        subs = sorted(self._subs.values(), key=lambda s: s.index)
        kfs = self.solve_local_many([s.index for s in subs], [forces[s.index] for s in subs])
        for s, kf in zip(subs, kfs):
            d[s.gids] += s.bval * kf[s.bcol]
        return d

    def local_operator(self, index: int):
        """Host copy of F~_i: m x m, upper triangle, strictly lower = 0 (None
        for the implicit strategy, as the reference, dualop.py:399-401)."""
        if self.config.strategy == "implicit":
            return None
        if not self.step_ready:
            raise LifecycleError("local operator before preprocess")
        sub = self._subs[int(index)]
        out = np.empty((sub.m, sub.m))
        _call(self._lib.feti_local_operator(self._ctx, sub.slot, _lib.f64ptr(out)))
        return out

    def persistent_addresses(self):
        """Host addresses of the persistent factor buffers (stability checks)."""
        return tuple(int(s.values.ctypes.data) for s in self._subs.values() if s.values is not None)

    def stats(self) -> dict:
        st = _lib.FetiStats()
        _call(self._lib.feti_get_stats(self._ctx, C.byref(st)))
        return st.as_dict()


def prepare(matrices, constraints, layout, config, pool=None, workers=1, schur_cap=2000, **kw) -> DualOperator:
    """Build and prepare a dual operator (dualop.py:414-419)."""
    op = DualOperator(matrices, constraints, layout, config, pool=pool, workers=workers,
                      schur_cap=schur_cap, **kw)
    return op.prepare()


def prepare_from_problems(subproblems, constraints, layout, config, pool=None, workers=1, schur_cap=2000,
                          **kw) -> DualOperator:
    """``prepare`` on the reference's ``SubdomainProblem`` list
    (Problem.subdomain_problems, solver.py:100-106): the operator reads the
    sparse K_i and ker K_i from them and runs the sparse-factor route, so the
    dense K_reg = K + rho Q Q^T (sparse.py:445-454) is never needed.  Later
    steps pass the new subproblems to ``preprocess``."""
    return prepare(list(subproblems), constraints, layout, config, pool=pool, workers=workers,
                   schur_cap=schur_cap, **kw)
