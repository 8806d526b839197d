"""Benchmark/test input generation (NOT on the hot path).

A vectorised restatement of the reference's problem setup so that the GPU box,
which has no copy of the reference, can build the BASELINE configurations:

* structured meshes: mesh.py:106-172 (lexicographic (z,y,x) nodes, 2 triangles
  per square, 6 Kuhn tetrahedra per cube with the orientation swap)
* linear-simplex element stiffness and load: mesh.py:180-305
* box partition and Total-FETI constraints: decomposition.py:131-224 (gluing
  chains over ascending owners, then Dirichlet rows; multipliers numbered
  gluing first, then Dirichlet, each lexicographically)
* kernel bases and regularization K + rho Q Q^T: solver.py:52-87,
  sparse.py:427-454
* contiguous cluster layout: decomposition.py:227-243

tests/test_inputs.py checks every array against fixtures produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import permutations

import numpy as np

POISSON = 0.3


# ---------------------------------------------------------------------------
# light containers with the duck-typed surface the drop-in consumes
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class Csr:
    shape: tuple
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray

    def row_arrays(self):
        return self.indptr, self.indices, self.data

    @property
    def nnz(self):
        return int(self.indptr[-1])

    def to_dense(self):
        out = np.zeros(self.shape)
        rows = np.repeat(np.arange(self.shape[0]), np.diff(self.indptr))
        out[rows, self.indices] = self.data
        return out


@dataclass(eq=False)
class DenseSym:
    """Dense symmetric matrix (the reference's K_reg is dense, sparse.py:445-454)."""

    values: np.ndarray

    @property
    def shape(self):
        return self.values.shape

    def to_dense(self):
        return self.values


@dataclass(eq=False)
class ShapeOnly:
    """Stand-in stiffness when the factor is produced elsewhere (bench)."""

    shape: tuple


@dataclass(eq=False)
class SubdomainConstraints:
    multiplier_ids: np.ndarray
    matrix: Csr


@dataclass(eq=False)
class ConstraintSet:
    n_multipliers: int
    c: np.ndarray
    per_subdomain: list


@dataclass(eq=False)
class Cluster:
    index: int
    subdomain_ids: np.ndarray
    dual_ids: np.ndarray
    scatter: list


@dataclass(eq=False)
class ClusterLayout:
    clusters: list
    n_multipliers: int

    @property
    def n_clusters(self):
        return len(self.clusters)


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------


def _kuhn_tets():
    corner = {(dx, dy, dz): dx + 2 * dy + 4 * dz for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)}
    tets = []
    for axes in permutations(range(3)):
        path = [(0, 0, 0)]
        pos = [0, 0, 0]
        for a in axes:
            pos = list(pos)
            pos[a] = 1
            path.append(tuple(pos))
        tets.append([corner[v] for v in path])
    return tets


_KUHN = _kuhn_tets()


def structured_mesh(dim, cells, offset=None, divisor=None):
    """(nodes, elements) of a structured box, as mesh.py:106-172."""
    npts = cells + 1
    offset = np.zeros(dim, np.int64) if offset is None else np.asarray(offset, np.int64)
    div = cells if divisor is None else int(divisor)
    axes = [(offset[a] + np.arange(npts, dtype=np.int64)) / div for a in range(dim)]
    if dim == 2:
        iy, ix = np.meshgrid(np.arange(npts), np.arange(npts), indexing="ij")
        nodes = np.stack([axes[0][ix.ravel()], axes[1][iy.ravel()]], axis=1)
        cy, cx = np.meshgrid(np.arange(cells), np.arange(cells), indexing="ij")
        cx, cy = cx.ravel(), cy.ravel()
        n00 = cy * npts + cx
        n10 = n00 + 1
        n01 = n00 + npts
        n11 = n01 + 1
        tri = np.empty((cells * cells, 2, 3), np.int64)
        tri[:, 0] = np.stack([n00, n10, n11], 1)
        tri[:, 1] = np.stack([n00, n11, n01], 1)
        return nodes, tri.reshape(-1, 3)
    iz, iy, ix = np.meshgrid(np.arange(npts), np.arange(npts), np.arange(npts), indexing="ij")
    nodes = np.stack([axes[0][ix.ravel()], axes[1][iy.ravel()], axes[2][iz.ravel()]], axis=1)
    cz, cy, cx = np.meshgrid(np.arange(cells), np.arange(cells), np.arange(cells), indexing="ij")
    base = ((cz.ravel() * npts + cy.ravel()) * npts + cx.ravel())
    rel = np.array([(dz * npts + dy) * npts + dx for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)])
    ids = base[:, None] + rel[None, :]                      # (ncell, 8) by dx+2dy+4dz
    # orientation swap decided on the unit cube (the sign of the volume is
    # translation invariant); mesh.py:157-159
    unit = np.array([[dx, dy, dz] for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)], float)
    tets = np.empty((ids.shape[0], 6, 4), np.int64)
    for k, tet in enumerate(_KUHN):
        conn = list(tet)
        pts = unit[conn]
        if np.linalg.det(pts[1:] - pts[0]) / 6.0 < 0:
            conn[2], conn[3] = conn[3], conn[2]
        tets[:, k] = ids[:, conn]
    return nodes, tets.reshape(-1, 4)


# ---------------------------------------------------------------------------
# element stiffness and assembly (mesh.py:180-305)
# ---------------------------------------------------------------------------


def _moduli(dim, coefficient):
    e, nu = float(coefficient), POISSON
    lam = e * nu / ((1 + nu) * (1 - 2 * nu))
    mu = e / (2 * (1 + nu))
    if dim == 2:
        return np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
    return np.array([
        [lam + 2 * mu, lam, lam, 0, 0, 0], [lam, lam + 2 * mu, lam, 0, 0, 0],
        [lam, lam, lam + 2 * mu, 0, 0, 0], [0, 0, 0, mu, 0, 0], [0, 0, 0, 0, mu, 0],
        [0, 0, 0, 0, 0, mu]], dtype=np.float64)


def element_matrices(nodes, elements, physics, dim, coefficient=1.0):
    pts = nodes[elements]                               # (ne, dim+1, dim)
    jac = pts[:, 1:] - pts[:, :1]
    if dim == 2:
        meas = 0.5 * np.linalg.det(jac)
    else:
        meas = np.linalg.det(jac) / 6.0
    if np.any(meas == 0.0):
        raise ArithmeticError("zero-measure element")
    inv_jt = np.linalg.inv(np.swapaxes(jac, 1, 2))
    grads = np.empty((elements.shape[0], dim + 1, dim))
    grads[:, 1:] = inv_jt
    grads[:, 0] = -inv_jt.sum(axis=1)
    meas = np.abs(meas)
    if physics == "heat":
        ke = coefficient * meas[:, None, None] * (grads @ np.swapaxes(grads, 1, 2))
    else:
        nn = dim + 1
        if dim == 2:
            b = np.zeros((elements.shape[0], 3, 2 * nn))
            for a in range(nn):
                gx, gy = grads[:, a, 0], grads[:, a, 1]
                b[:, 0, 2 * a] = gx
                b[:, 1, 2 * a + 1] = gy
                b[:, 2, 2 * a] = gy
                b[:, 2, 2 * a + 1] = gx
        else:
            b = np.zeros((elements.shape[0], 6, 3 * nn))
            for a in range(nn):
                gx, gy, gz = grads[:, a, 0], grads[:, a, 1], grads[:, a, 2]
                c = 3 * a
                b[:, 0, c] = gx
                b[:, 1, c + 1] = gy
                b[:, 2, c + 2] = gz
                b[:, 3, c] = gy
                b[:, 3, c + 1] = gx
                b[:, 4, c + 1] = gz
                b[:, 4, c + 2] = gy
                b[:, 5, c] = gz
                b[:, 5, c + 2] = gx
        d = _moduli(dim, coefficient)
        ke = meas[:, None, None] * (np.swapaxes(b, 1, 2) @ d @ b)
    return 0.5 * (ke + np.swapaxes(ke, 1, 2)), meas


def from_coo(rows, cols, vals, shape):
    """Deduplicating COO -> CSR exactly as SparseCsr.from_coo (sparse.py:98-119)."""
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        keep = np.concatenate(([True], (np.diff(rows) != 0) | (np.diff(cols) != 0)))
        starts = np.flatnonzero(keep)
        summed = np.add.reduceat(vals, starts)
        rows, cols, vals = rows[starts], cols[starts], summed
    indptr = np.zeros(shape[0] + 1, np.int64)
    np.add.at(indptr, rows + 1, 1)
    np.cumsum(indptr, out=indptr)
    return Csr(tuple(shape), indptr, cols.astype(np.int64), vals.astype(np.float64))


def assemble(nodes, elements, physics, dim, coefficient=1.0):
    """Stiffness (CSR) and unit body-force load, as assemble_system (mesh.py:265-305)."""
    dpn = 1 if physics == "heat" else dim
    nverts = dim + 1
    n_dofs = nodes.shape[0] * dpn
    ke, meas = element_matrices(nodes, elements, physics, dim, coefficient)
    dofs = (elements[:, :, None] * dpn + np.arange(dpn)).reshape(elements.shape[0], -1)
    nd = dofs.shape[1]
    load = np.zeros(n_dofs)
    np.add.at(load, dofs.ravel(), np.repeat(meas / nverts, nd))
    rr = np.repeat(dofs, nd, axis=1)
    cc = np.tile(dofs, (1, nd))
    keep = rr <= cc
    rows = rr[keep]
    cols = cc[keep]
    vals = ke.reshape(ke.shape[0], -1)[keep]
    off = rows != cols
    k = from_coo(np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                 np.concatenate([vals, vals[off]]), (n_dofs, n_dofs))
    return k, load


def kernel_basis(physics, nodes, dim):
    """Orthonormal kernel basis with deterministic signs (solver.py:52-87)."""
    n_nodes = nodes.shape[0]
    if physics == "heat":
        basis = np.full((n_nodes, 1), 1.0)
    else:
        cols = []
        for c in range(dim):
            t = np.zeros((n_nodes, dim))
            t[:, c] = 1.0
            cols.append(t.ravel())
        if dim == 2:
            r = np.zeros((n_nodes, 2))
            r[:, 0] = -nodes[:, 1]
            r[:, 1] = nodes[:, 0]
            cols.append(r.ravel())
        else:
            for (a, b) in ((0, 1), (1, 2), (0, 2)):
                r = np.zeros((n_nodes, 3))
                r[:, a] = -nodes[:, b]
                r[:, b] = nodes[:, a]
                cols.append(r.ravel())
        basis = np.stack(cols, axis=1)
    q, _ = np.linalg.qr(basis)
    for j in range(q.shape[1]):
        lead = np.flatnonzero(np.abs(q[:, j]) > 1e-12)
        if lead.size and q[lead[0], j] < 0:
            q[:, j] = -q[:, j]
    return q


def regularized_dense(k: Csr, kernel: np.ndarray) -> np.ndarray:
    """Dense K + rho Q Q^T with rho = trace(K)/n (sparse.py:427-454)."""
    dense = k.to_dense()
    n = dense.shape[0]
    q, _ = np.linalg.qr(kernel)
    rho = np.trace(dense) / n
    shift = q @ q.T
    shift = 0.5 * (shift + shift.T)
    dense += rho * shift
    return dense


# ---------------------------------------------------------------------------
# partition, constraints, clusters (decomposition.py)
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class SubdomainInfo:
    index: int
    offset: np.ndarray
    dof_l2g: np.ndarray


class Problem:
    """A BASELINE configuration: ``Problem("heat", 3, 20, 4)`` is config 3."""

    def __init__(self, physics: str, dim: int, cells_per_subdomain: int, subdomains_per_side: int,
                 n_clusters: int = 1, coefficient: float = 1.0):
        if physics not in ("heat", "elasticity") or dim not in (2, 3):
            raise ValueError("physics in {heat, elasticity}, dim in {2, 3}")
        self.physics, self.dim = physics, dim
        self.cells, self.sps = int(cells_per_subdomain), int(subdomains_per_side)
        self.coefficient = float(coefficient)
        self.dpn = 1 if physics == "heat" else dim
        gcells = self.cells * self.sps
        npts = gcells + 1
        ln = self.cells + 1
        self.n_local_nodes = ln ** dim
        self.n_dofs_global = npts ** dim * self.dpn
        self.n_sub = self.sps ** dim
        # local node -> index tuple (x fastest)
        li = np.arange(self.n_local_nodes)
        lidx = [(li // ln ** a) % ln for a in range(dim)]
        self.subs = []
        for flat in range(self.n_sub):
            pos = np.unravel_index(flat, (self.sps,) * dim, order="C")
            pos = tuple(int(p) for p in reversed(pos))
            offset = np.array(pos, np.int64) * self.cells
            g = np.zeros(self.n_local_nodes, np.int64)
            for a in reversed(range(dim)):
                g = g * npts + (offset[a] + lidx[a])
            dof = (g[:, None] * self.dpn + np.arange(self.dpn)).ravel()
            self.subs.append(SubdomainInfo(flat, offset, dof))
        self._build_constraints(npts)
        self.layout = self.build_clusters(n_clusters)
        self._local_mesh = {}

    @property
    def n_dofs(self) -> int:
        return self.n_local_nodes * self.dpn

    def _build_constraints(self, npts):
        dim, dpn = self.dim, self.dpn
        n_loc = self.n_dofs
        subs = np.repeat(np.arange(self.n_sub, dtype=np.int64), n_loc)
        locs = np.tile(np.arange(n_loc, dtype=np.int64), self.n_sub)
        globs = np.concatenate([s.dof_l2g for s in self.subs])
        order = np.lexsort((subs, globs))          # by global dof, then subdomain
        globs, subs, locs = globs[order], subs[order], locs[order]
        same_next = globs[1:] == globs[:-1]
        # gluing: each adjacent owner pair of a shared dof is one multiplier,
        # numbered by global dof then chain position
        pair = np.flatnonzero(same_next)
        n_glue = pair.shape[0]
        mids_g = np.arange(n_glue, dtype=np.int64)
        rows_s = [subs[pair], subs[pair + 1]]
        rows_l = [locs[pair], locs[pair + 1]]
        rows_v = [np.ones(n_glue), -np.ones(n_glue)]
        rows_m = [mids_g, mids_g]
        # Dirichlet on x = 0: global nodes with x index 0, every owner
        gnode = globs // dpn
        on_face = (gnode % npts) == 0
        dl = np.flatnonzero(on_face)                 # already sorted by dof then subdomain
        mids_d = n_glue + np.arange(dl.shape[0], dtype=np.int64)
        rows_s.append(subs[dl])
        rows_l.append(locs[dl])
        rows_v.append(np.ones(dl.shape[0]))
        rows_m.append(mids_d)
        self.n_multipliers = int(n_glue + dl.shape[0])
        self.c = np.zeros(self.n_multipliers)
        s_all = np.concatenate(rows_s)
        l_all = np.concatenate(rows_l)
        v_all = np.concatenate(rows_v)
        m_all = np.concatenate(rows_m)
        o = np.lexsort((m_all, s_all))
        s_all, l_all, v_all, m_all = s_all[o], l_all[o], v_all[o], m_all[o]
        bounds = np.searchsorted(s_all, np.arange(self.n_sub + 1))
        self.gids, self.bcol, self.bval = [], [], []
        for s in range(self.n_sub):
            a, b = bounds[s], bounds[s + 1]
            self.gids.append(m_all[a:b].copy())
            self.bcol.append(l_all[a:b].copy())
            self.bval.append(v_all[a:b].copy())

    def constraints(self) -> ConstraintSet:
        per = []
        for s in range(self.n_sub):
            m = self.gids[s].shape[0]
            mat = Csr((m, self.n_dofs), np.arange(m + 1, dtype=np.int64), self.bcol[s], self.bval[s])
            per.append(SubdomainConstraints(self.gids[s], mat))
        return ConstraintSet(self.n_multipliers, self.c, per)

    def build_clusters(self, n_clusters: int) -> ClusterLayout:
        k = int(n_clusters)
        if k < 1 or self.n_sub % k:
            raise ValueError(f"{self.n_sub} subdomains not divisible into {n_clusters} clusters")
        per = self.n_sub // k
        clusters = []
        for ci in range(k):
            ids = np.arange(ci * per, (ci + 1) * per, dtype=np.int64)
            dual = np.unique(np.concatenate([self.gids[s] for s in ids]))
            scatter = [np.searchsorted(dual, self.gids[s]) for s in ids]
            clusters.append(Cluster(ci, ids, dual, scatter))
        return ClusterLayout(clusters, self.n_multipliers)

    def local_mesh(self, s: int):
        info = self.subs[s]
        key = tuple(info.offset)
        if key not in self._local_mesh:
            self._local_mesh = {key: structured_mesh(self.dim, self.cells, info.offset, self.cells * self.sps)}
        return self._local_mesh[key]

    def subdomain_system(self, s: int):
        """(K, load, kernel) of subdomain s (solver.py:358-371 without regularization)."""
        nodes, elems = self.local_mesh(s)
        k, load = assemble(nodes, elems, self.physics, self.dim, self.coefficient)
        q = kernel_basis(self.physics, nodes, self.dim)
        return k, load, q

    def kreg_dense(self, s: int) -> np.ndarray:
        k, _, q = self.subdomain_system(s)
        return regularized_dense(k, q)

    def m_per_subdomain(self) -> np.ndarray:
        return np.array([g.shape[0] for g in self.gids])


CONFIGS = {
    "c1": ("heat", 2, 16, 4),
    "c2": ("heat", 3, 8, 8),
    "c3": ("heat", 3, 20, 4),
    "c4": ("elasticity", 3, 14, 4),
    "c5": ("elasticity", 2, 128, 16),
}


def regularized_csr(k: Csr, kernel: np.ndarray) -> Csr:
    """K_reg as the reference builds it: dense shift, then CSR with the
    diagonal kept (sparse.py:445-454, SparseCsr.from_dense(keep_diagonal))."""
    dense = regularized_dense(k, kernel)
    n = dense.shape[0]
    mask = dense != 0.0
    mask[np.diag_indices(n)] = True
    r, c = np.nonzero(mask)
    ip = np.zeros(n + 1, np.int64)
    np.add.at(ip, r + 1, 1)
    np.cumsum(ip, out=ip)
    return Csr((n, n), ip, c.astype(np.int64), dense[r, c])


def reference_inputs(prob: "Problem", dense: bool = False):
    """(matrices, constraints, layout) in the shape the drop-in consumes."""
    mats = []
    for s in range(prob.n_sub):
        k, _, q = prob.subdomain_system(s)
        mats.append(DenseSym(regularized_dense(k, q)) if dense else regularized_csr(k, q))
    return mats, prob.constraints(), prob.layout
