"""Host side of the sparse-factor route (SURVEY.md §7 hard part 4, §8f row 2).

The reference regularizes every floating subdomain as K_reg = K + rho Q Q^T
(regularize, sparse.py:427-454).  The shift is dense, so the reference's
factor is a full triangle: 4.4 GB and ~1.2e13 flops per config-5 subdomain
(n = 33,282), which makes config 5 infeasible on its path.  This route keeps
the factor sparse and still returns the reference's F~_i exactly (to
rounding):

* fixing DOFs: K_s = K + rho E E^T with E = [e_f] on r DOFs chosen by a
  pivoted QR of Q^T (E^T Q is then well conditioned and nonsingular), so K_s
  is SPD with K's sparsity pattern;
* identity: K_reg^-1 = K^+ + rho^-1 Q Q^T and K^+ = Pi K_s^-1 Pi with
  Pi = I - Q Q^T, hence

      F~ = B K_s^-1 B^T - U1 U2^T - U2 U1^T + U1 (Q^T W + rho^-1 I) U1^T,
      W = K_s^-1 Q,  U1 = B Q,  U2 = B W;

* ordering: every constrained DOF last (so X = L^-1 P B^T lives in the
  trailing rows only) and the interior "onion" ordered -- reverse
  Cuthill-McKee levels grown from the constrained DOFs -- so that the
  interface rows of L fill only across the last interior layers.

The device does the rest (csrc/feti_sparse.cu): K_s is scattered into a
block-sparse 128x128 tile pool, factored left-looking on the FP64 tensor
pipe together with an appended block row P Q (which yields y = L^-1 P Q, so
Q^T W = y^T y and U2 = X^T y_b need no extra solves), then the unchanged
explicit assembly runs on the trailing interface block and a rank-2r update
of the packed F~ tiles applies the correction.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import breadth_first_order


def fixing_dofs(kernel: np.ndarray) -> np.ndarray:
    """r DOFs whose rows of Q are the most independent (pivoted QR of Q^T)."""
    q = np.asarray(kernel, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] == 0:
        return np.zeros(0, np.int64)
    _, _, piv = scipy.linalg.qr(q.T, mode="economic", pivoting=True)
    return np.sort(piv[: q.shape[1]].astype(np.int64))


def onion_interface_last(n: int, indptr, indices, interface) -> np.ndarray:
    """perm (position -> DOF): interior by decreasing graph distance from the
    interface (breadth-first from all interface DOFs, reversed), then the
    interface DOFs in ascending order."""
    interface = np.unique(np.asarray(interface, np.int64))
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    mark = np.zeros(n, bool)
    mark[interface] = True
    if interface.size == 0 or interface.size == n:
        return np.concatenate([np.flatnonzero(~mark), interface]).astype(np.int64)
    # graph with one extra vertex (index n) adjacent to every interface DOF
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    r = np.concatenate([rows, np.full(interface.size, n), interface])
    c = np.concatenate([ix, interface, np.full(interface.size, n)])
    g = csr_matrix((np.ones(r.size, np.int8), (r, c)), shape=(n + 1, n + 1))
    order = breadth_first_order(g, n, directed=False, return_predecessors=False)
    order = order[order != n]
    interior = order[~mark[order]]
    seen = np.zeros(n, bool)
    seen[interior] = True
    rest = np.flatnonzero(~mark & ~seen)          # disconnected from the interface
    return np.concatenate([rest, interior[::-1], interface]).astype(np.int64)


def regularization_shift(indptr, indices, data, n: int) -> float:
    """rho = trace(K) / n (sparse.py:450)."""
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    return float(np.asarray(data, np.float64)[rows == ix].sum()) / n


# ---------------------------------------------------------------------------
# tile-aligned dissection ordering (padded positions)
# ---------------------------------------------------------------------------

TILE_ROWS = 128


def _csr_graph(n, indptr, indices):
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    return csr_matrix((np.ones(ix.size, np.int8), (rows, ix)), shape=(n, n))


def _bfs_levels(g, src):
    ip, ix = g.indptr, g.indices
    lev = np.full(g.shape[0], -1, np.int64)
    lev[src] = 0
    front = np.array([src], np.int64)
    depth = 0
    while front.size:
        starts, ends = ip[front], ip[front + 1]
        nb = np.unique(np.concatenate([ix[a:b] for a, b in zip(starts, ends)]))
        nb = nb[lev[nb] < 0]
        depth += 1
        lev[nb] = depth
        front = nb
    return lev


def _dissect(g, ids, depth, min_size, sep_rule="mid"):
    """[(kind, dof array)] in elimination order: both halves, then the separator
    (a breadth-first level from a pseudo-peripheral vertex: the median level,
    or with sep_rule "minsep" the smallest level within 35-65 % of the DOFs)."""
    if depth == 0 or ids.size <= min_size:
        return [("leaf", ids)]
    from scipy.sparse.csgraph import connected_components

    sub = g[ids][:, ids].tocsr()
    nc, lab = connected_components(sub, directed=False)
    if nc > 1:
        out = []
        for cc in range(nc):
            out += _dissect(g, ids[lab == cc], depth, min_size, sep_rule)
        return out
    s = 0
    for _ in range(2):
        s = int(np.argmax(_bfs_levels(sub, s)))
    lev = _bfs_levels(sub, s)
    cnt = np.bincount(lev)
    cum = np.cumsum(cnt)
    mid = int(np.searchsorted(cum, ids.size / 2))
    if sep_rule == "minsep":
        cand = [lv for lv in range(1, cnt.size - 1) if 0.35 * ids.size <= cum[lv - 1] and cum[lv] - cnt[lv]
                <= 0.65 * ids.size]
        if cand:
            mid = min(cand, key=lambda lv: cnt[lv])
    return (_dissect(g, ids[lev < mid], depth - 1, min_size, sep_rule)
            + _dissect(g, ids[lev > mid], depth - 1, min_size, sep_rule) + [("sep", ids[lev == mid])])


def _onion_toward(g, region, boundary):
    """region's DOFs by decreasing breadth-first distance from `boundary`."""
    m = region.size
    sub = np.concatenate([region, boundary])
    h = g[sub][:, sub].tocsr()
    nb = boundary.size
    r = np.concatenate([np.full(nb, m + nb), np.arange(m, m + nb)])
    c = np.concatenate([np.arange(m, m + nb), np.full(nb, m + nb)])
    extra = csr_matrix((np.ones(2 * nb, np.int8), (r, c)), shape=(m + nb + 1, m + nb + 1))
    hh = h.tocoo()
    h2 = (extra + csr_matrix((hh.data, (hh.row, hh.col)), shape=(m + nb + 1, m + nb + 1))).tocsr()
    order = breadth_first_order(h2, m + nb, directed=False, return_predecessors=False)
    order = order[order < m]
    seen = np.zeros(m, bool)
    seen[order] = True
    return region[np.concatenate([np.flatnonzero(~seen), order[::-1]])]


def dissection_segments(n, indptr, indices, interface, depth=2, min_size=512, sep_rule="mid"):
    """Segments (DOF arrays) of a tile-aligned ordering: a `depth`-level
    dissection of the interior (leaves onion-ordered toward their own
    boundary), then the interface ordered by the segment each DOF touches
    first, so the interface rows coupled to a leaf share few tiles."""
    g = _csr_graph(n, indptr, indices)
    interface = np.unique(np.asarray(interface, np.int64))
    mark = np.zeros(n, bool)
    mark[interface] = True
    interior = np.flatnonzero(~mark)
    segs = []
    for kind, ids in _dissect(g, interior, depth, min_size, sep_rule):
        if ids.size == 0:
            continue
        if kind == "leaf":
            inleaf = np.zeros(n, bool)
            inleaf[ids] = True
            nbr = np.unique(g[ids].indices)
            segs.append(_onion_toward(g, ids, nbr[~inleaf[nbr]]))
        else:
            segs.append(ids)
    return _with_interface_last(segs, n, indptr, indices, interface)


def interface_pieces(bcol, neighbour):
    """The interface split into FETI "pieces" (faces, edges, corners): the
    constrained DOFs grouped by the set of subdomains their multipliers glue
    them to (-1 for a Dirichlet row).  `neighbour[j]` is the other owner of
    multiplier j (row j of B~, DOF bcol[j])."""
    bcol = np.asarray(bcol, np.int64)
    neighbour = np.asarray(neighbour, np.int64)
    if bcol.size == 0:
        return []
    o = np.lexsort((neighbour, bcol))
    d, nb = bcol[o], neighbour[o]
    keep = np.ones(d.size, bool)
    keep[1:] = (d[1:] != d[:-1]) | (nb[1:] != nb[:-1])
    d, nb = d[keep], nb[keep]
    starts = np.flatnonzero(np.r_[True, d[1:] != d[:-1]])
    ends = np.r_[starts[1:], d.size]
    groups = {}
    for a, b in zip(starts.tolist(), ends.tolist()):
        groups.setdefault(tuple(nb[a:b].tolist()), []).append(int(d[a]))
    return [np.array(v, np.int64) for _, v in sorted(groups.items())]


def _bfs_from_set(sub, starts):
    ip, ix = sub.indptr, sub.indices
    lev = np.full(sub.shape[0], -1, np.int64)
    lev[starts] = 0
    front = starts
    depth = 0
    while front.size:
        nb = np.unique(np.concatenate([ix[a:b] for a, b in zip(ip[front], ip[front + 1])]))
        nb = nb[lev[nb] < 0]
        depth += 1
        lev[nb] = depth
        front = nb
    return lev


def _face_split(g, ids, pieces, n):
    """Vertex separator of region `ids` as a breadth-first level grown from
    the region's DOFs next to one boundary piece (an interface face or an
    earlier separator): on a box those levels are planes parallel to the
    piece.  Among levels with 35-65 % of the DOFs before them, the smallest
    one (relative to ids^(2/3), to one decimal), ties broken toward the
    middle.  None if no piece touches the region."""
    sub = g[ids][:, ids].tocsr()
    pos = np.full(n, -1, np.int64)
    pos[ids] = np.arange(ids.size)
    unit = max(1.0, ids.size ** (2.0 / 3.0))
    best = None
    for piece in pieces:
        st = pos[np.unique(g[piece].indices)]
        st = np.unique(st[st >= 0])
        if st.size == 0:
            continue
        lev = _bfs_from_set(sub, st)
        if (lev < 0).any():
            continue
        cnt = np.bincount(lev)
        cum = np.cumsum(cnt)
        for lv in range(1, cnt.size - 1):
            if not (0.35 * ids.size <= cum[lv - 1] and cum[lv] - cnt[lv] <= 0.65 * ids.size):
                continue
            key = (round(10.0 * cnt[lv] / unit), abs(cum[lv - 1] - (ids.size - cnt[lv]) / 2.0))
            if best is None or key < best[0]:
                best = (key, lev, lv)
    if best is None:
        return None
    _, lev, lv = best
    return ids[lev < lv], ids[lev > lv], ids[lev == lv]


def _face_dissect(g, ids, depth, pieces, n, min_size=256):
    from scipy.sparse.csgraph import connected_components

    if depth == 0 or ids.size <= min_size:
        return [("leaf", ids)]
    nc, lab = connected_components(g[ids][:, ids], directed=False)
    if nc > 1:
        out = []
        for cc in range(nc):
            out += _face_dissect(g, ids[lab == cc], depth, pieces, n, min_size)
        return out
    parts = _face_split(g, ids, pieces, n)
    if parts is None:
        return [("leaf", ids)]
    a, b, sep = parts
    return (_face_dissect(g, a, depth - 1, pieces + [sep], n, min_size)
            + _face_dissect(g, b, depth - 1, pieces + [sep], n, min_size) + [("sep", sep)])


def face_dissection_segments(n, indptr, indices, interface, pieces, depth=3):
    """Like `dissection_segments`, but every separator is a breadth-first
    level grown from a boundary piece (`interface_pieces`, then the
    separators already cut): on the structured subdomains of the benchmark
    these are the axis planes a geometric dissection would cut, found from
    the graph and the gluing alone (c3: 20.5 -> 16.2 GF of 128-row tile
    products per subdomain, c4 47.2 -> 36.6, c5 10.7 -> 9.9)."""
    g = _csr_graph(n, indptr, indices)
    interface = np.unique(np.asarray(interface, np.int64))
    mark = np.zeros(n, bool)
    mark[interface] = True
    interior = np.flatnonzero(~mark)
    segs = []
    for kind, ids in _face_dissect(g, interior, depth, [np.asarray(p, np.int64) for p in pieces], n):
        if ids.size == 0:
            continue
        if kind == "leaf":
            inleaf = np.zeros(n, bool)
            inleaf[ids] = True
            nbr = np.unique(g[ids].indices)
            segs.append(_onion_toward(g, ids, nbr[~inleaf[nbr]]))
        else:
            segs.append(ids)
    return _with_interface_last(segs, n, indptr, indices, interface)


def _with_interface_last(segs, n, indptr, indices, interface):
    seg_of = np.full(n, len(segs), np.int64)
    for i, s in enumerate(segs):
        seg_of[s] = i
    key = np.full(interface.size, len(segs), np.int64)
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    for t, d in enumerate(interface):
        key[t] = seg_of[ix[ip[d]:ip[d + 1]]].min()
    return segs + [interface[np.lexsort((interface, key))]]


def padded_positions(segments):
    """perm_pos (position -> DOF, -1 for padding) with every segment starting
    at a 128-row tile boundary, and iperm (DOF -> position)."""
    npos = sum(-(-s.size // TILE_ROWS) * TILE_ROWS for s in segments)
    n = sum(s.size for s in segments)
    perm = np.full(npos, -1, np.int64)
    iperm = np.empty(n, np.int64)
    p = 0
    for s in segments:
        perm[p:p + s.size] = s
        iperm[s] = p + np.arange(s.size)
        p += -(-s.size // TILE_ROWS) * TILE_ROWS
    return perm, iperm


def tile_flops_estimate(n, indptr, indices, iperm, npos, kernel_dim, n_iface):
    """Tile flops of the block-sparse factorization for an ordering (the
    block symbolic of csrc/feti_sparse.cu sp_symbolic, in Python): used to
    pick the ordering."""
    TB = TILE_ROWS
    T = -(-npos // TB)
    ip = np.asarray(indptr, np.int64)
    ix = np.asarray(indices, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    bi, bj = iperm[rows] // TB, iperm[ix] // TB
    lo = bi > bj
    struct = [set() for _ in range(T)]
    for a, b in zip(bi[lo].tolist(), bj[lo].tolist()):
        struct[b].add(a)
    smin = (npos - -(-n_iface // TB) * TB) // TB
    for J in range(smin, T):
        struct[J].update(range(J + 1, T))
    ops = 0.0
    for k in range(T):
        s = struct[k]
        sn = len(s)
        ops += sn * (sn + 1) / 2 + sn + (sn + 2) / 16.0 * (kernel_dim > 0)
        if s:
            p = min(s)
            struct[p] |= (s - {p})
    return ops * 2.0 * TB ** 3


_ORDERING_CACHE = {}
_ORDERING_CACHE_MAX = 256


def _ordering_key(n, indptr, indices, interface, recipe, pieces):
    import hashlib

    h = hashlib.blake2b(digest_size=16)
    h.update(repr((int(n), tuple(recipe) if recipe else None)).encode())
    for a in (indptr, indices, np.unique(np.asarray(interface, np.int64))):
        h.update(np.ascontiguousarray(a, np.int64).tobytes())
        h.update(b"|")
    for piece in sorted((np.asarray(x, np.int64).tobytes() for x in (pieces or [])), key=lambda b: (len(b), b)):
        h.update(piece)
        h.update(b";")
    return h.hexdigest()


def sparse_route_ordering(n, indptr, indices, interface, recipe, pieces=None):
    """(perm_pos, iperm) for a recipe ("onion",), ("dissection", depth),
    ("dissection", depth, sep_rule) or ("faces", depth) (needs the
    subdomain's `interface_pieces`).  Subdomains with the same pattern,
    interface and pieces (most of a structured decomposition) share one
    computation."""
    key = _ordering_key(n, indptr, indices, interface, recipe, pieces)
    hit = _ORDERING_CACHE.get(key)
    if hit is None:
        hit = _sparse_route_ordering(n, indptr, indices, interface, recipe, pieces)
        if len(_ORDERING_CACHE) >= _ORDERING_CACHE_MAX:
            _ORDERING_CACHE.clear()
        _ORDERING_CACHE[key] = hit
    return hit[0].copy(), hit[1].copy()


def _sparse_route_ordering(n, indptr, indices, interface, recipe, pieces=None):
    if recipe is None or recipe[0] == "onion":
        perm = onion_interface_last(n, indptr, indices, interface)
        iperm = np.empty(n, np.int64)
        iperm[perm] = np.arange(n, dtype=np.int64)
        return perm, iperm
    if recipe[0] == "faces":
        if not pieces:
            raise ValueError("the 'faces' ordering needs the subdomain's interface pieces")
        return padded_positions(face_dissection_segments(n, indptr, indices, interface, pieces, int(recipe[1])))
    rule = recipe[2] if len(recipe) > 2 else "mid"
    return padded_positions(dissection_segments(n, indptr, indices, interface, depth=int(recipe[1]), sep_rule=rule))


def choose_ordering(n, indptr, indices, interface, kernel_dim, mode="auto", max_depth=4, pieces=None):
    """The recipe with the fewest estimated tile flops (mode "auto"), or the
    one named by `mode` ("onion", "dissection:<depth>", "faces:<depth>")."""
    if mode == "onion":
        return ("onion",)
    if mode.startswith("dissection:"):
        return ("dissection", int(mode.split(":", 1)[1]))
    if mode.startswith("faces:"):
        return ("faces", int(mode.split(":", 1)[1]))
    n_iface = np.unique(np.asarray(interface, np.int64)).size
    best, best_ops = ("onion",), None
    candidates = [("onion",)]
    if n >= 16 * TILE_ROWS:
        candidates += [("dissection", d) for d in range(1, max_depth + 1)]
        candidates += [("dissection", d, "minsep") for d in range(1, max_depth + 1)]
        if pieces:
            candidates += [("faces", d) for d in range(1, max_depth + 2)]
    for rec in candidates:
        perm, iperm = sparse_route_ordering(n, indptr, indices, interface, rec, pieces)
        ops = tile_flops_estimate(n, indptr, indices, iperm, perm.shape[0], kernel_dim, n_iface)
        if best_ops is None or ops < best_ops:
            best, best_ops = rec, ops
    return best
