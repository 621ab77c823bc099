"""Slab decomposition of a lattice PD problem across ranks.

Both 2D and 3D lattices are cut along y: 2D plates into x-slabs of element rows
(contiguous id ranges), 3D blocks into z-x slabs (north star: "sharded in z-x
slabs") -- the y element rows [y0, y1) of every z layer.  Rank r owns those
element rows and the y node rows [y0, y1) (the last rank also the far node
row).  Its handle holds the slab plus a halo of HALO_LO = R+1 = 4 element rows
below and HALO_HI = R = 3 above, i.e. 4 node rows on each side: with a stencil
radius of R = 3 element rows, that is exactly what the forces of the elements
touching the owned nodes need.  After every fine step the predictor
displacement of the 4 boundary node rows goes to each neighbour (pmts_pd_set_halo
+ NCCL, or pmts_pd_get_rows_layers / set_rows_layers for a host-mediated
exchange); in 3D a halo is one 4-row range per z node layer, which the library
packs into one message.  Elements and nodes in the halo compute garbage near
the cut (truncated families) but are overwritten before anyone owned reads them,
so the owned results equal a single-domain run bit for bit.

Local numbering keeps the global order (x fastest, then y, then z), so every
per-element and per-node gather runs in the single-domain order.  Global ids:
element l of a slab is (l // p_loc) p_glob + ya nx + l % p_loc with p = nx ny_loc
and nx ny (pmts_pd_desc.slab_plane) -- the per-bond hash keys and the break log
use them.  Only the rows the owned nodes need are computed: the node update runs
on the owned node rows, the 3D bond kernel on the element rows those nodes touch
(pmts_pd_desc.node_rows), so the redundant work per rank is the halo's ubar only.
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
    dim: int
    nx: int          # global elements along x, y, z (z = 1 in 2D)
    ny: int
    nz: int
    y0: int          # owned element rows [y0, y1) of the global lattice
    y1: int
    ya: int          # local element rows [ya, yb) (slab + halo)
    yb: int

    @property
    def nyl(self) -> int:
        return self.yb - self.ya

    @property
    def last(self) -> bool:
        return self.rank == self.nranks - 1

    @property
    def lattice(self) -> tuple:
        return (self.nx, self.nyl, self.nz) if self.dim == 3 else (self.nx, self.nyl, 1)

    @property
    def n_elems(self) -> int:
        return self.nx * self.nyl * self.nz

    @property
    def layers(self) -> int:
        """z node layers a halo range repeats over (1 in 2D)."""
        return self.nz + 1 if self.dim == 3 else 1

    @property
    def layer_stride(self) -> int:
        return (self.nx + 1) * (self.nyl + 1) if self.dim == 3 else 0

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.nyl + 1) * self.layers

    @property
    def elem_first(self) -> int:
        """pmts_pd_desc.global_id_offset: global id of local element 0."""
        return self.ya * self.nx

    @property
    def plane(self) -> tuple:
        """pmts_pd_desc.slab_plane: elements per z layer, local and global (3D)."""
        return (self.nx * self.nyl, self.nx * self.ny) if self.dim == 3 else (0, 0)

    @property
    def own_elems(self) -> tuple:
        """pmts_pd_desc.owned_elems: the owned local element range (in-layer in 3D)."""
        return ((self.y0 - self.ya) * self.nx, (self.y1 - self.ya) * self.nx)

    @property
    def node_rows(self) -> tuple:
        """Owned local y node rows [lo, hi) (pmts_pd_desc.node_rows)."""
        return (self.y0 - self.ya, self.y1 - self.ya + (1 if self.last else 0))

    @property
    def halo(self) -> tuple:
        """(peer_lo, send_lo, recv_lo, n_lo, peer_hi, send_hi, recv_hi, n_hi): first local
        node of layer 0 and nodes per layer of each range (pmts_pd_set_halo)."""
        NX = self.nx + 1
        H = HALO_NODE_ROWS * NX
        lo = ((self.rank - 1, (self.y0 - self.ya) * NX,
               (self.y0 - HALO_NODE_ROWS - self.ya) * NX, H) if self.rank > 0 else (-1, 0, 0, 0))
        hi = ((self.rank + 1, (self.y1 - HALO_NODE_ROWS - self.ya) * NX, (self.y1 - self.ya) * NX,
               H) if not self.last else (-1, 0, 0, 0))
        return lo + hi

    # -- id maps ---------------------------------------------------------------
    def _node_ijk(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        NX, NYL = self.nx + 1, self.nyl + 1
        return ids % NX, (ids // NX) % NYL, ids // (NX * NYL)

    def node_global(self, ids) -> np.ndarray:
        i, j, k = self._node_ijk(ids)
        return (k * (self.ny + 1) + j + self.ya) * (self.nx + 1) + i

    def elem_global(self, ids) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        pl = self.nx * self.nyl
        return (ids // pl) * (self.nx * self.ny) + self.elem_first + ids % pl

    def owns_elem(self, ids) -> np.ndarray:
        r = np.asarray(ids, dtype=np.int64) % (self.nx * self.nyl)
        e0, e1 = self.own_elems
        return (r >= e0) & (r < e1)

    def owned_nodes(self) -> np.ndarray:
        """Local ids of the owned nodes (ascending)."""
        _, j, _ = self._node_ijk(np.arange(self.n_nodes))
        r0, r1 = self.node_rows
        return np.nonzero((j >= r0) & (j < r1))[0]

    def local_nodes_global(self) -> np.ndarray:
        return self.node_global(np.arange(self.n_nodes))

    def local_elems_global(self) -> np.ndarray:
        return self.elem_global(np.arange(self.n_elems))

    def halo_nodes(self):
        """[(peer, send local ids, recv local ids)] with the layers expanded."""
        plo, slo, rlo, nlo, phi, shi, rhi, nhi = self.halo
        out = []
        for peer, s0, r0, n in ((plo, slo, rlo, nlo), (phi, shi, rhi, nhi)):
            if peer < 0:
                continue
            base = np.arange(n)
            lay = np.arange(self.layers)[:, None] * self.layer_stride
            out.append((peer, (s0 + lay + base).ravel(), (r0 + lay + base).ravel()))
        return out

    # back-compat for 2D callers: the owned node range is contiguous there
    @property
    def node_first(self) -> int:
        return int(self.node_global(0))


def make_slab(lattice, dim: int, rank: int, nranks: int) -> Slab:
    nx, ny = int(lattice[0]), int(lattice[1])
    nz = int(lattice[2]) if dim == 3 else 1
    y0, y1 = split_rows(ny, nranks)[rank]
    if y1 - y0 < HALO_NODE_ROWS:
        raise ValueError(f"slab of {y1 - y0} rows < {HALO_NODE_ROWS}: too many ranks")
    ya, yb = max(0, y0 - HALO_LO), min(ny, y1 + HALO_HI)
    return Slab(rank, nranks, dim, nx, ny, nz, y0, y1, ya, yb)


def redundancy(lattice, dim: int, nranks: int) -> dict:
    """Per-rank work over owned work at nranks (max over ranks): the bond kernel runs
    on the element rows the owned nodes touch, ubar on every local row."""
    worst = {"bond": 0.0, "ubar": 0.0}
    for r in range(nranks):
        s = make_slab(lattice, dim, r, nranks)
        own = s.y1 - s.y0
        r0, r1 = s.node_rows
        bond = min(s.nyl, r1) - max(0, r0 - 1)
        worst["bond"] = max(worst["bond"], bond / own)
        worst["ubar"] = max(worst["ubar"], s.nyl / own)
    return worst


def local_arrays(sc, slab: Slab) -> dict:
    """Cut the global scenario (pd.Scenario) down to the slab's local problem."""
    dim = sc.dim
    ge = slab.local_elems_global()
    gn = slab.local_nodes_global()
    g2l = np.full(sc.n_nodes, -1, dtype=np.int64)
    g2l[gn] = np.arange(len(gn))
    conn = g2l[sc.conn[ge]]
    assert conn.min() >= 0
    dofs = (gn[:, None] * dim + np.arange(dim)).ravel()
    d2l = np.full(sc.n_dof, -1, dtype=np.int64)
    d2l[dofs] = np.arange(len(dofs))
    bl = d2l[sc.bc_dofs]
    sel = bl >= 0
    return dict(dim=dim, nodes=sc.nodes[gn], conn=np.ascontiguousarray(conn, dtype=np.int32),
                mass=sc.mass[dofs], p_ext=sc.p_ext[dofs],
                bc_dofs=bl[sel].astype(np.int32), bc_vel=sc.bc_vel[sel],
                centroid=sc.centroid[ge], volume=sc.volume[ge], dofs=dofs)


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
              lattice_h=h, lattice_vol=vol, slab_plane=slab.plane,
              node_rows=slab.node_rows if sc.dim == 3 else (0, 0))
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
    s.local_dofs = la["dofs"]
    return s


def attach_nccl(s, uid: bytes):
    """Join the clique and install the slab's halo (layers in 3D) on handle s."""
    slab = s.slab
    s.comm_init(uid, slab.nranks, slab.rank)
    s.set_halo(*slab.halo)
    if slab.layers > 1:
        s.set_halo_layers(slab.layers, slab.layer_stride)


def host_exchange(handles):
    """Host-mediated halo exchange between slab handles of one process (the
    single-GPU emulation of several ranks; no kernel ever waits on another rank)."""
    msgs = []
    for h in handles:
        s = h.slab
        plo, slo, rlo, nlo, phi, shi, rhi, nhi = s.halo
        if plo >= 0:
            msgs.append((plo, handles[plo].slab.halo[6], nlo,
                         h.get_rows(slo, nlo, s.layers, s.layer_stride)))
        if phi >= 0:
            msgs.append((phi, handles[phi].slab.halo[2], nhi,
                         h.get_rows(shi, nhi, s.layers, s.layer_stride)))
    for dst, first, n, vals in msgs:
        t = handles[dst]
        t.set_rows(first, n, vals, t.slab.layers, t.slab.layer_stride)


def gather_owned(handles, n_dof_global: int, dim: int):
    """Owned u, v, a of every slab handle assembled into global arrays."""
    out = [np.full(n_dof_global, np.nan) for _ in range(3)]
    for h in handles:
        own = h.slab.owned_nodes()
        g = h.slab.node_global(own)
        loc = (own[:, None] * dim + np.arange(dim)).ravel()
        glb = (g[:, None] * dim + np.arange(dim)).ravel()
        for x, y in zip(out, h.state()):
            x[glb] = y[loc]
    return out
