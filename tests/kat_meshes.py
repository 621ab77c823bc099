"""Tiny meshes of the reference's own known-answer tests (proj/tests/test_perifem.cpp,
proj/tests/test_mesh.cpp), shared by the CPU oracle tests and the GPU tests."""
import numpy as np


def quads(nodes, conn):
    """Quad4 mesh with centroid = node mean and volume = area (exact for squares)."""
    nodes = np.array(nodes, dtype=np.float64)
    conn = np.array(conn, dtype=np.int32)
    cen = nodes[conn].mean(axis=1)
    p = nodes[conn]
    area = 0.5 * np.abs((p[:, 2, 0] - p[:, 0, 0]) * (p[:, 3, 1] - p[:, 1, 1]) -
                        (p[:, 3, 0] - p[:, 1, 0]) * (p[:, 2, 1] - p[:, 0, 1]))
    return dict(dim=2, nodes=nodes, conn=conn, centroid=cen, volume=area)


def disjoint_quads():
    """test_perifem.cpp:112-124: two unit quads, disjoint nodes, centroids 1 apart."""
    return quads([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [1, 0, 0], [2, 0, 0], [2, 1, 0], [1, 1, 0]], [[0, 1, 2, 3], [4, 5, 6, 7]])


def manufactured_quads():
    """test_perifem.cpp:147-157: xi = (3, 4)."""
    return quads([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [3, 4, 0], [4, 4, 0], [4, 5, 0], [3, 5, 0]], [[0, 1, 2, 3], [4, 5, 6, 7]])


def grid(nx, ny, h):
    """generate_structured-style 2D grid (mesh.hpp:170-219), i fastest."""
    nodes = [[i * h, j * h, 0.0] for j in range(ny + 1) for i in range(nx + 1)]
    nid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    conn = [[nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)]
            for j in range(ny) for i in range(nx)]
    return quads(nodes, conn)


def brute_force_pairs(cen, delta, notches=(), eps=None):
    """tests/support/oracles.hpp:66-93 restated: O(E^2) double loop."""
    from oracle import pyoracle as po  # noqa: F401  (same predicate set as the oracle)

    E = len(cen)
    d = np.sqrt(((cen[:, None, :] - cen[None, :, :]) ** 2).sum(-1))
    i, j = np.nonzero(np.triu(d <= delta, 1))
    pairs = np.stack([i, j], 1).astype(np.int32)
    if notches:
        keep = []
        for a, b in pairs:
            keep.append(not any(_seg_cross(cen[a], cen[b], n) for n in notches))
        pairs = pairs[np.array(keep, dtype=bool)] if len(pairs) else pairs
    return pairs


def _seg_cross(p1, p2, n):
    """Proper or touching intersection of segment p1p2 with notch segment n (2D)."""
    q1, q2 = np.array(n[:2]), np.array(n[3:5])
    r, s = p2[:2] - p1[:2], q2 - q1
    den = r[0] * s[1] - r[1] * s[0]
    qp = q1 - p1[:2]
    if abs(den) < 1e-30:
        return False
    t = (qp[0] * s[1] - qp[1] * s[0]) / den
    u = (qp[0] * r[1] - qp[1] * r[0]) / den
    tol = 1e-9
    return -tol <= t <= 1 + tol and -tol <= u <= 1 + tol


def pd_sys(mesh, pairs, s_crit=0.0, delta=1.5, l=0.375, c0=1e9, dt=1e-3, mass=None):
    """OraclePD / PDSolver inputs for a KAT mesh (test_pd: l = delta/4, c0 = 1e9)."""
    n_nodes = len(mesh["nodes"])
    M = np.ones(2 * n_nodes) if mass is None else mass
    return dict(dim=2, n_nodes=n_nodes, conn=mesh["conn"], centroid=mesh["centroid"],
                volume=mesh["volume"], pairs=np.array(pairs, dtype=np.int32).reshape(-1, 2),
                mass=M, p_ext=np.zeros(2 * n_nodes), delta=delta, l=l, c0=c0,
                s_crit=s_crit, dt=dt)
