"""Slab decomposition of a lattice PD problem across ranks.

Rank r owns the element rows (2D) / layers (3D) [y0, y1) of the slowest lattice
axis -- a contiguous range of element and node ids -- and the nodes of those
rows (the last rank also the far node row).  Its handle holds the slab plus a
halo of HALO_LO = R+1 = 4 element rows below and HALO_HI = R = 3 above, i.e. 4
node rows on each side: with a stencil radius of R = 3 element rows, that is
exactly what the forces of the elements touching the owned nodes need.  After
every fine step the predictor displacement of the 4 boundary node rows goes to
each neighbour (pmts_pd_set_halo + NCCL, or pmts_pd_get_rows / set_rows for a
host-mediated exchange).  Elements and nodes in the halo compute garbage near
the cut (truncated families) but are overwritten before anyone owned reads
them, so the owned results equal a single-domain run bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

HALO_LO = 4  # element rows below the slab (R + 1)
HALO_HI = 3  # element rows above the slab (R)
HALO_NODE_ROWS = 4


def split_rows(n_rows: int, nranks: int):
    base, extra = divmod(n_rows, nranks)
    out, y = [], 0
    for r in range(nranks):
        n = base + (1 if r < extra else 0)
        out.append((y, y + n))
        y += n
    return out


@dataclass
class Slab:
    rank: int
    nranks: int
    y0: int
    y1: int
    ya: int
    yb: int
    plane: int       # elements per row/layer
    nplane: int      # nodes per row/layer
    lattice: tuple   # local lattice dims
    elem_first: int  # global id of local element 0
    node_first: int  # global id of local node 0
    n_elems: int
    n_nodes: int
    own_elems: tuple  # local element range owned
    own_nodes: tuple  # local node range owned
    halo: tuple       # (peer_lo, send_lo, recv_lo, n_lo, peer_hi, send_hi, recv_hi, n_hi)

    def global_nodes(self, a, b):
        return self.node_first + a, self.node_first + b


def make_slab(lattice, dim: int, rank: int, nranks: int) -> Slab:
    nx, ny = lattice[0], lattice[1]
    nz = lattice[2] if dim == 3 else 1
    rows = nz if dim == 3 else ny
    plane = nx * ny if dim == 3 else nx
    nplane = (nx + 1) * (ny + 1) if dim == 3 else nx + 1
    y0, y1 = split_rows(rows, nranks)[rank]
    if y1 - y0 < HALO_NODE_ROWS:
        raise ValueError(f"slab of {y1 - y0} rows < {HALO_NODE_ROWS}: too many ranks")
    ya, yb = max(0, y0 - HALO_LO), min(rows, y1 + HALO_HI)
    loc_rows = yb - ya
    lat = (nx, ny, loc_rows) if dim == 3 else (nx, loc_rows, 1)
    last = rank == nranks - 1
    own_e = ((y0 - ya) * plane, (y1 - ya) * plane)
    own_n = ((y0 - ya) * nplane, (y1 - ya + (1 if last else 0)) * nplane)
    H = HALO_NODE_ROWS * nplane
    if rank > 0:
        lo = (rank - 1, (y0 - ya) * nplane, (y0 - HALO_NODE_ROWS - ya) * nplane, H)
    else:
        lo = (-1, 0, 0, 0)
    if not last:
        hi = (rank + 1, (y1 - HALO_NODE_ROWS - ya) * nplane, (y1 - ya) * nplane, H)
    else:
        hi = (-1, 0, 0, 0)
    return Slab(rank, nranks, y0, y1, ya, yb, plane, nplane, lat, ya * plane, ya * nplane,
                loc_rows * plane, (loc_rows + 1) * nplane, own_e, own_n, lo + hi)


def local_arrays(sc, slab: Slab) -> dict:
    """Cut the global scenario (pd.Scenario) down to the slab's local problem."""
    dim = sc.dim
    e0, e1 = slab.elem_first, slab.elem_first + slab.n_elems
    n0, n1 = slab.node_first, slab.node_first + slab.n_nodes
    conn = sc.conn[e0:e1] - n0
    assert conn.min() >= 0 and conn.max() < slab.n_nodes
    d0, d1 = n0 * dim, n1 * dim
    sel = (sc.bc_dofs >= d0) & (sc.bc_dofs < d1)
    return dict(dim=dim, nodes=sc.nodes[n0:n1], conn=np.ascontiguousarray(conn),
                mass=sc.mass[d0:d1], p_ext=sc.p_ext[d0:d1],
                bc_dofs=(sc.bc_dofs[sel] - d0).astype(np.int32), bc_vel=sc.bc_vel[sel],
                centroid=sc.centroid[e0:e1], volume=sc.volume[e0:e1])


def lattice_constants(sc):
    """Nominal lattice spacing and the reference element volume (global element 0),
    identical on every rank."""
    h = float(sc.nodes[1, 0] - sc.nodes[0, 0])
    return h, float(sc.volume[0])


def solver_for_slab(sc, slab: Slab, mode, device=0, **over):
    """PDSolver of the slab's local problem (no communication attached yet)."""
    from .pd import PDSolver

    la = local_arrays(sc, slab)
    ext = sc.cfg.get("ext", {})
    h, vol = lattice_constants(sc)
    kw = dict(dim=sc.dim, nodes=la["nodes"], conn=la["conn"], mass=la["mass"],
              p_ext=la["p_ext"], delta=sc.delta, dt=sc.dt, bc_dofs=la["bc_dofs"],
              bc_vel=la["bc_vel"], c0=sc.c0, l=sc.l, s_crit=sc.s_crit, gamma=sc.gamma,
              beta=sc.beta, mode=mode, device=device, lattice=slab.lattice,
              global_id_offset=slab.elem_first, owned_elems=slab.own_elems,
              lattice_h=h, lattice_vol=vol)
    if len(sc.notch_npts) and sc.notch_npts[0]:
        kw.update(notch_npts=sc.notch_npts, notch_pts=sc.notch_pts)
    if ext.get("micromodulus") == "constant":
        from . import capi

        kw.update(micromodulus=capi.MICRO_CONST, c_const=ext["c"], h=ext.get("h", 1.0))
    if ext.get("s_crit_spread"):
        kw.update(s_crit_spread=ext["s_crit_spread"], seed=int(ext.get("seed", 0)))
    kw.update(over)
    s = PDSolver(**kw)
    s.slab = slab
    return s
