"""Structured P2-tetrahedron Poisson operator by stencil replication (C5 setup).

BASELINE C5 needs the fine-level P2-tet stiffness matrix at 2M / 8M / 16M
DOFs.  The reference's assembler (fem.py:303-377) would need ~70 GB at 16M
DOFs (SURVEY.md finding 8), so this builds the same operator for the
*unperturbed* Kuhn grid (mesh.py:136-184) row by row:

* DOF numbering is the reference's: vertices ``(k*side + j)*side + i``, then
  edges in np.unique order of sorted vertex pairs (fem.py:212-218).  In the
  Kuhn triangulation every vertex v owns up to 7 "forward" edges
  v -> v + {x, y, xy, z, xz, yz, xyz}, whose index increments
  (1, side, side+1, side^2, ...) are already in that lexicographic order.
* Every interior row is a translate of one of 8 stencils (vertex + 7 edge
  types), read off a small assembled mesh; boundary DOFs become identity rows
  and their columns are dropped (symmetric Dirichlet elimination,
  fem.py:361-374).  Within a row the stencil order is site-independent, so
  rows come out sorted and canonical without a global sort.

Values equal ``fem.assemble_poisson`` on the same grid up to the summation
order of element contributions (tests/test_setup.py checks <= 1e-13).
"""

from __future__ import annotations

import numpy as np

from .sparse import CsrMatrix

# forward edge directions in lexicographic (index-increment) order
_DIRS = np.array([(1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1)],
                 dtype=np.int64)


def _site_of(dofs, n):
    """(base vertex (i,j,k), type 0..7) of DOFs on an n-grid (type 0 = vertex)."""
    side = n + 1
    nv = side ** 3
    i = np.empty((len(dofs), 3), dtype=np.int64)
    t = np.zeros(len(dofs), dtype=np.int64)
    v = dofs < nv
    vi = dofs[v]
    i[v] = np.column_stack([vi % side, (vi // side) % side, vi // (side * side)])
    e = dofs[~v] - nv
    base, typ = _edge_table(n)
    i[~v] = base[e]
    t[~v] = typ[e] + 1
    return i, t


def _edge_table(n):
    side = n + 1
    k, j, ii = np.meshgrid(np.arange(side), np.arange(side), np.arange(side), indexing="ij")
    verts = np.column_stack([ii.ravel(), j.ravel(), k.ravel()])
    exists = np.all(verts[:, None, :] + _DIRS[None, :, :] <= n, axis=2)  # (nv, 7)
    vb, tb = np.nonzero(exists)
    return verts[vb], tb


def _stencils():
    """Interior-row stencils [(di, dj, dk, type, value)] per DOF type, in column order."""
    from .fem import assemble_poisson, build_dofmap
    from .mesh import generate_simplex_grid
    n = 4
    m = generate_simplex_grid(3, n)
    dm = build_dofmap(m, 2)
    a = assemble_poisson(m, dm, None, dirichlet_all=False).a
    side = n + 1
    nv = side ** 3
    base = np.array([2, 2, 2])
    vid = (base[2] * side + base[1]) * side + base[0]
    ebase, etyp = _edge_table(n)
    out = []
    for typ in range(8):
        if typ == 0:
            row = vid
        else:
            row = nv + int(np.nonzero((ebase == base).all(axis=1) & (etyp == typ - 1))[0][0])
        lo, hi = a.row_offsets[row], a.row_offsets[row + 1]
        cols = a.col_indices[lo:hi]
        vals = a.values[lo:hi]
        site, t = _site_of(cols, n)
        out.append((site - base, t, vals))
    return out


def _is_boundary(site, typ, n):
    """Boundary DOF: vertex on a box face, or edge whose both endpoints lie on one face."""
    a = site
    b = site + np.where(typ[:, None] > 0, _DIRS[np.maximum(typ - 1, 0)], 0)
    on = np.zeros(len(site), dtype=bool)
    for ax in range(3):
        on |= (a[:, ax] == 0) & (b[:, ax] == 0)
        on |= (a[:, ax] == n) & (b[:, ax] == n)
    return on


def p2_tet_laplacian(n: int, chunk: int = 1 << 18) -> CsrMatrix:
    """Dirichlet-eliminated P2 Laplacian on the n^3 Kuhn grid of the unit cube."""
    side = n + 1
    nv = side ** 3
    # 3D stiffness entries scale with h: rescale the n=4 stencils to this grid
    sten = [(o, t, v * (4.0 / n)) for o, t, v in _stencils()]
    k, j, ii = np.meshgrid(np.arange(side), np.arange(side), np.arange(side), indexing="ij")
    verts = np.column_stack([ii.ravel(), j.ravel(), k.ravel()])
    exists = np.all(verts[:, None, :] + _DIRS[None, :, :] <= n, axis=2)
    n_edges_at = exists.sum(axis=1)
    eprefix = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(n_edges_at, out=eprefix[1:])
    rank = np.cumsum(exists, axis=1) - 1                 # rank of each type at a vertex
    ndof = nv + int(eprefix[-1])

    def dof_id(site, typ):
        vid = (site[:, 2] * side + site[:, 1]) * side + site[:, 0]
        out = vid.copy()
        e = typ > 0
        out[e] = nv + eprefix[vid[e]] + rank[vid[e], typ[e] - 1]
        return out

    def rows_for(sites, typ):
        """CSR pieces for DOFs at `sites` of one type (rows in the given order)."""
        off, ctyp, vals = sten[typ]
        S = len(vals)
        tarr = np.full(len(sites), typ, dtype=np.int64)
        bnd = _is_boundary(sites, tarr, n)
        nb = (sites[:, None, :] + off[None, :, :]).reshape(-1, 3)
        nbt = np.tile(ctyp, len(sites))
        inside = np.all((nb >= 0) & (nb <= n), axis=1)
        # neighbours of interior rows always exist; keep interior neighbours only
        keep = np.zeros(len(nb), dtype=bool)
        nbi = np.nonzero(inside)[0]
        keep[nbi] = ~_is_boundary(nb[nbi], nbt[nbi], n)
        keep = keep.reshape(len(sites), S)
        keep[bnd] = False
        cols = np.zeros(len(nb), dtype=np.int64)
        cols[keep.ravel()] = dof_id(nb[keep.ravel()], nbt[keep.ravel()])
        cols = cols.reshape(len(sites), S)
        v = np.broadcast_to(vals, (len(sites), S))
        counts = keep.sum(axis=1)
        ids = dof_id(sites, tarr)
        # boundary rows: identity
        counts[bnd] = 1
        c_out = np.where(keep, cols, -1)
        v_out = np.where(keep, v, 0.0)
        bi = np.nonzero(bnd)[0]
        c_out[bi, 0] = ids[bi]
        v_out[bi, 0] = 1.0
        sel = c_out >= 0
        return counts, c_out[sel], v_out[sel]

    counts_all, cols_all, vals_all = [], [], []
    for s0 in range(0, nv, chunk):          # vertex rows
        c, cc, vv = rows_for(verts[s0:s0 + chunk], 0)
        counts_all.append(c)
        cols_all.append(cc)
        vals_all.append(vv)
    for s0 in range(0, nv, chunk):          # edge rows, base-vertex major, type minor
        vb, tb = np.nonzero(exists[s0:s0 + chunk])
        sites = verts[s0 + vb]
        types = tb + 1
        # emit per type then restore (vertex, type) order
        order = np.lexsort((types, vb))
        sites, types = sites[order], types[order]
        pieces = []
        for typ in range(1, 8):
            m = types == typ
            if not np.any(m):
                continue
            c, cc, vv = rows_for(sites[m], typ)
            pieces.append((np.nonzero(m)[0], c, cc, vv))
        # interleave rows back into (vertex, type) order
        nrow = len(sites)
        cnt = np.zeros(nrow, dtype=np.int64)
        for idx, c, _, _ in pieces:
            cnt[idx] = c
        start = np.zeros(nrow + 1, dtype=np.int64)
        np.cumsum(cnt, out=start[1:])
        cc_all = np.empty(start[-1], dtype=np.int64)
        vv_all = np.empty(start[-1])
        for idx, c, cc, vv in pieces:
            pos = np.repeat(start[idx], c) + (np.arange(len(cc)) - np.repeat(np.cumsum(c) - c, c))
            cc_all[pos] = cc
            vv_all[pos] = vv
        counts_all.append(cnt)
        cols_all.append(cc_all)
        vals_all.append(vv_all)
    counts = np.concatenate(counts_all)
    ptr = np.zeros(ndof + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return CsrMatrix(ndof, ndof, ptr, np.concatenate(cols_all), np.concatenate(vals_all))
