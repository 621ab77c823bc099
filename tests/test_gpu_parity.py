"""GPU parity: the CUDA fine step (through the C ABI) against the oracle and the
reference's own outputs.

Deterministic mode: broken-bond set bit-exact vs the reference, u/v/a bitwise
equal to the matrix-free oracle and within 1e-12 relative L2 of the reference.
Fast mode: fields within 1e-9 relative L2 before crack initiation, >= 99.9% of
broken bonds agree afterwards (BASELINE.json north_star tolerances).
"""
import numpy as np
import pytest

import kat_meshes as km
from conftest import GOLDEN_SCENARIO, load_golden, oracle_sys
from oracle import pyoracle as po
from paper_2403_03605_b200 import capi
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario

pytestmark = pytest.mark.gpu

SMALL = ["mini", "block3d", "cfg1_200"]


def _solver(name, mode, **over):
    g = load_golden(name)
    sc = Scenario(cf.get(GOLDEN_SCENARIO[name]))
    s = PDSolver.from_scenario(sc, mode=mode, **over)
    return g, sc, s


def _pairs_index(pairs):
    return {(int(i), int(j)): q for q, (i, j) in enumerate(pairs)}


@pytest.mark.parametrize("name", list(GOLDEN_SCENARIO))
def test_device_neighbour_build_matches_reference(name):
    g, sc, s = _solver(name, capi.DETERMINISTIC)
    s.find_pe_pairs()
    assert np.array_equal(s.pairs(), g["pairs"])
    info = s.info()
    assert info["n_bonds"] == g["meta"]["n_pairs"]


@pytest.mark.parametrize("name", SMALL)
def test_deterministic_bitwise(name):
    g, sc, s = _solver(name, capi.DETERMINISTIC)
    s.find_pe_pairs()
    steps = g["meta"]["steps"]
    s.initial_acceleration(g["scale"][0])
    nb = s.step(g["scale"][1:steps + 1])
    u, v, a = s.state()
    # broken set and order == reference (update_bond_states order: step, then pe)
    log = s.break_log(len(g["pairs"]))
    idx = _pairs_index(g["pairs"])
    got = np.array([[st, idx[(i, j)]] for st, i, j in log], dtype=np.int64).reshape(-1, 2)
    assert nb == len(g["broken"])
    assert np.array_equal(got, g["broken"])
    # bitwise == matrix-free oracle (same summation order, no FMA)
    o = po.OraclePD(oracle_sys(g, sc), po.MF)
    o.init(g["scale"][0])
    o.step(g["scale"][1:steps + 1])
    ou, ov, oa = o.state()
    assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(a, oa)
    # reference: 1e-12 relative
    for x, ref in ((u, g["u"]), (v, g["v"]), (a, g["a"])):
        assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    e, n = s.damage_field()
    assert np.array_equal(e, g["damage_elem"]) and np.array_equal(n, g["damage_node"])
    assert np.array_equal(s.intact(), o.mu())


def test_deterministic_checkpoint_and_set_state():
    """Stepping in batches equals one batch; set_state resumes exactly."""
    g, sc, s = _solver("cfg1_200", capi.DETERMINISTIC)
    s.find_pe_pairs()
    s.initial_acceleration(g["scale"][0])
    s.step(g["scale"][1:21])
    s.step(g["scale"][21:51])
    u, v, a = s.state()
    assert np.linalg.norm(u - g["u_50"]) <= 1e-12 * np.linalg.norm(g["u_50"])
    s.set_state(u, v, a)
    s.step(g["scale"][51:201])
    u2, _, _ = s.state()
    assert np.linalg.norm(u2 - g["u"]) <= 1e-12 * np.linalg.norm(g["u"])


@pytest.mark.slow
def test_bp_coarse_deterministic():
    g, sc, s = _solver("bp_coarse_2000", capi.DETERMINISTIC)
    s.find_pe_pairs()
    s.initial_acceleration(g["scale"][0])
    nb = s.step(g["scale"][1:2001])
    log = s.break_log(1000)
    idx = _pairs_index(g["pairs"])
    got = np.array([[st, idx[(i, j)]] for st, i, j in log]).reshape(-1, 2)
    assert nb == 10 and np.array_equal(got, g["broken"])
    u, v, _ = s.state()
    assert np.linalg.norm(u - g["u"]) <= 1e-12 * np.linalg.norm(g["u"])


@pytest.mark.parametrize("path", ["lattice", "lattice-nopairs", "ell"])
@pytest.mark.parametrize("name", SMALL)
def test_fast_mode_tolerances(name, path):
    # lattice-nopairs: representative per-bond stencil constants (lattice_h = 0): the 2D
    # tile kernel with per-offset (not pair-symmetric) sums; ell: no lattice encoding
    over = {"lattice": {}, "lattice-nopairs": {"lattice_h": 0.0},
            "ell": {"lattice": (0, 0, 0)}}[path]
    path = "ell" if path == "ell" else "lattice"
    g, sc, s = _solver(name, capi.FAST, **over)
    s.find_pe_pairs()
    assert s.info()["path"] in ((1, 2) if path == "lattice" else (0,))
    steps = g["meta"]["steps"]
    s.initial_acceleration(g["scale"][0])
    br = g["broken"]
    first = int(br[0, 0]) if len(br) else steps + 1
    pre = min(first - 1, steps)
    # before crack initiation: 1e-9 relative L2 against the oracle at the same step
    o = po.OraclePD(oracle_sys(g, sc), po.MF)
    o.init(g["scale"][0])
    if pre > 0:
        s.step(g["scale"][1:pre + 1])
        o.step(g["scale"][1:pre + 1])
        u, v, _ = s.state()
        ou, ov, _ = o.state()
        assert np.linalg.norm(u - ou) <= 1e-9 * np.linalg.norm(ou)
        assert np.linalg.norm(v - ov) <= 1e-9 * np.linalg.norm(ov)
    s.step(g["scale"][pre + 1:steps + 1])
    # after: >= 99.9% agreement of the broken set (symmetric difference)
    mine = s.intact() == 0
    ref = np.zeros(len(g["pairs"]), dtype=bool)
    ref[g["broken"][:, 1]] = True
    if ref.sum():
        agree = 1.0 - np.logical_xor(mine, ref).sum() / max(ref.sum(), 1)
        assert agree >= 0.999, agree
        _crack_within_delta(g["pairs"], mine, ref, sc, tip=False)


def _plate(nx, ny):
    """The mini notched plate (horizontal tension) resized to nx x ny elements."""
    sc = cf.get("mini")
    dx = sc["mesh"]["spacing"]
    lx, ly = nx * dx, ny * dx
    sc["mesh"]["bounds"] = [0.0, 0.0, lx, ly]
    sc["mesh"]["notch1"] = [0.5 * lx, 0.5 * ly, 0.5 * lx, 0.25 * ly]
    sc["load"]["traction2"] = [lx - 1e-4, -1.0, lx + 1e-4, 1.0, 16e6, 0.0]
    return Scenario(sc)


@pytest.mark.parametrize("nx,ny", [(40, 16), (124, 62), (32, 31), (64, 93), (60, 35), (42, 20), (33, 65)])
def test_tile9_ragged_lattices_vs_oracle(nx, ny):
    """The TMA-staged tile kernel on lattices that are multiples of the 31 x 31 tile,
    smaller than one tile, and ragged (the TMA zero fill stands in for bounds checks
    at every domain edge): fields within 1e-9 of the matrix-free oracle before the
    first break, >= 99.9 % broken-set agreement after 120 steps."""
    sc = _plate(nx, ny)
    s = PDSolver.from_scenario(sc, mode=capi.FAST).find_pe_pairs()
    assert s.info()["path"] == 2
    pairs = s.pairs()
    o = po.OraclePD(dict(dim=2, n_nodes=sc.n_nodes, conn=sc.conn, centroid=sc.centroid,
                         volume=sc.volume, pairs=pairs, mass=sc.mass, p_ext=sc.p_ext,
                         delta=sc.delta, l=sc.l, c0=sc.c0, s_crit=sc.s_crit, dt=sc.dt), po.MF)
    s.initial_acceleration(sc.load_scale(0.0))
    o.init(sc.load_scale(0.0))
    scales = [sc.load_scale(i * sc.dt) for i in range(1, 121)]
    pre = o.state()
    first = None
    for i, x in enumerate(scales):
        br, _ = o.step([x])
        if len(br):
            first = i + 1
            break
        pre = o.state()
    k = (first - 1) if first else 120
    s.step(scales[:k])
    u, v, _ = s.state()
    assert np.linalg.norm(u - pre[0]) <= 1e-9 * np.linalg.norm(pre[0])
    assert np.linalg.norm(v - pre[1]) <= 1e-9 * np.linalg.norm(pre[1])
    if first:
        o.step(scales[first:])
        s.step(scales[k:])
        mine, ref = s.intact() == 0, o.mu() == 0
        assert 1.0 - np.logical_xor(mine, ref).sum() / max(ref.sum(), 1) >= 0.999
    if (nx, ny) == (40, 16):
        assert first is not None  # the notched mini plate cracks within 120 steps


@pytest.mark.parametrize("nx,ny", [(40, 16), (124, 62), (64, 93)])
def test_tile9_pairs_close_to_per_offset(nx, ny):
    """The pair-symmetric force (default) regroups the same terms: fields within
    1e-12 relative L2 of the per-offset sums (representative per-bond constants,
    lattice_h = 0) and the same broken bonds."""
    sc = _plate(nx, ny)
    out = {}
    for pairs in (True, False):
        over = {} if pairs else {"lattice_h": 0.0}
        s = PDSolver.from_scenario(sc, mode=capi.FAST, **over).find_pe_pairs()
        assert s.info()["path"] == 2
        s.initial_acceleration(sc.load_scale(0.0))
        nb = s.step([sc.load_scale(i * sc.dt) for i in range(1, 121)])
        out[pairs] = (nb, *s.state(), s.intact())
    a, b = out[True], out[False]
    assert a[0] == b[0]
    assert np.array_equal(a[4], b[4])
    for x, y in zip(a[1:4], b[1:4]):
        assert np.linalg.norm(x - y) <= 1e-12 * np.linalg.norm(y)


@pytest.mark.parametrize("nx,ny,steps", [(40, 16, 120), (124, 62, 300), (33, 65, 200), (64, 93, 200)])
def test_tile9_screen_is_exact(nx, ny, steps, monkeypatch):
    """The cold-tile break screen (default) only skips candidate tests the node-step
    bound proves cannot fire: u, v, a and the bond states are bitwise those of the
    candidate pass on every tile (pmts_pd_set_option PMTS_OPT_BREAK_SCREEN = 0)."""
    sc = _plate(nx, ny)
    out = {}
    for screen in (True, False):
        s = PDSolver.from_scenario(sc, mode=capi.FAST).find_pe_pairs()
        s.set_option(capi.OPT_BREAK_SCREEN, 1 if screen else 0)
        s.initial_acceleration(sc.load_scale(0.0))
        nb = s.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
        out[screen] = (nb, *s.state(), s.intact())
    a, b = out[True], out[False]
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)
    if (nx, ny) == (40, 16):
        assert a[0] > 0


@pytest.mark.parametrize("mode", [capi.FAST, capi.FAST_F32POS])
@pytest.mark.parametrize("nx,ny,steps", [(124, 62, 300), (190, 130, 700), (97, 160, 700)])
def test_tile9_clean_tiles_are_exact(nx, ny, steps, mode):
    """Clean tiles (default: a tile whose own and neighbouring bonds are all intact
    neither stages nor re-writes its bond states) change nothing: fields, bond states,
    broken counts and the damage field are bitwise those of staging every tile
    (PMTS_OPT_CLEAN_TILES = 0), through crack growth, and switching the option in the
    middle of a run recomputes the flags from the live bond states."""
    sc = _plate(nx, ny)
    scales = [sc.load_scale(i * sc.dt) for i in range(1, steps + 1)]
    out = {}
    for clean in ("on", "off", "toggle"):
        s = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
        s.set_option(capi.OPT_CLEAN_TILES, 0 if clean == "off" else 1)
        s.initial_acceleration(sc.load_scale(0.0))
        h = steps // 2
        nb = [s.step(scales[:h])]
        if clean == "toggle":
            s.set_option(capi.OPT_CLEAN_TILES, 0)
            nb.append(s.step(scales[h:h + 7]))
            s.set_option(capi.OPT_CLEAN_TILES, 1)
            nb.append(s.step(scales[h + 7:]))
            nb = [nb[0], nb[1] + nb[2]]
        else:
            nb.append(s.step(scales[h:]))
        out[clean] = (nb, *s.state(), s.intact(), *s.damage_field())
    assert sum(out["on"][0]) > 0
    for k in ("off", "toggle"):
        assert out["on"][0] == out[k][0]
        for x, y in zip(out["on"][1:], out[k][1:]):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["mini", "block3d"])
@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_step_tracked_reports_every_step(mode, name):
    """pmts_pd_step_tracked: per-step tracked displacements and broken counts equal
    single-step stepping (2D tile kernel, 3D lattice path, deterministic ELL)."""
    g, sc, s = _solver(name, mode)
    _, _, s2 = _solver(name, mode)
    s.find_pe_pairs()
    s2.find_pe_pairs()
    steps = 40
    dofs = np.array([1, 2 * (sc.n_nodes // 2), 2 * sc.n_nodes - 1], dtype=np.int32)
    s.initial_acceleration(g["scale"][0])
    s2.initial_acceleration(g["scale"][0])
    trk, nb = s.step_tracked(g["scale"][1:steps + 1], dofs)
    ref_nb = []
    for i in range(steps):
        ref_nb.append(s2.step(g["scale"][i + 1:i + 2]))
        u, _, _ = s2.state()
        assert np.array_equal(trk[i], u[dofs])
    assert list(nb) == ref_nb
    u1, v1, a1 = s.state()
    u2, v2, a2 = s2.state()
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2) and np.array_equal(a1, a2)


def _crack_within_delta(pairs, mine, ref, sc, tip):
    """North star (fast mode after cracking): the damage path within one horizon of the
    oracle's -- Hausdorff distance of the broken-bond midpoints, and the tip (largest x)
    of a crack growing from a left-edge notch."""
    from crack import broken_midpoints, crack_tip, hausdorff

    mm = broken_midpoints(pairs, mine, sc.centroid)
    mr = broken_midpoints(pairs, ref, sc.centroid)
    assert hausdorff(mm, mr) <= sc.delta
    if tip:
        assert np.linalg.norm(crack_tip(mm) - crack_tip(mr)) <= sc.delta


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_cfg4_small_impact_3d(mode):
    """BASELINE cfg4 physics at 20x20x10 (3D hex8, constant micromodulus, seeded
    impact velocity): deterministic bitwise vs the matrix-free oracle; fast mode
    (3D lattice stencil, 122 offsets) within the north-star tolerances."""
    sc = Scenario(cf.get("cfg4_small"))
    s = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    if mode == capi.FAST:
        assert s.info()["path"] == 1 and s.info()["stencil_size"] == 122
    pairs = po.find_pairs(3, sc.centroid, sc.volume, sc.delta)
    assert np.array_equal(s.pairs(), pairs)
    ext = sc.cfg["ext"]
    o = po.OraclePD(dict(dim=3, n_nodes=sc.n_nodes, conn=sc.conn, centroid=sc.centroid,
                         volume=sc.volume, pairs=pairs, mass=sc.mass, p_ext=sc.p_ext,
                         delta=sc.delta, s_crit=sc.s_crit, dt=sc.dt, micromodulus=1,
                         c_const=ext["c"]), po.MF)
    z = np.zeros(sc.n_dof)
    v0 = sc.initial_velocity()
    assert (v0 != 0).sum() > 0
    s.set_state(z, v0, z)
    o.set_state(z, v0, z)
    s.initial_acceleration(sc.load_scale(0.0))
    o.init(sc.load_scale(0.0))
    steps = sc.n_steps
    scales = sc.scales(1, steps)
    if mode == capi.DETERMINISTIC:
        nb = s.step(scales)
        br, _ = o.step(scales)
        u, v, a = s.state()
        ou, ov, oa = o.state()
        assert nb == len(br)
        assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(a, oa)
        assert np.array_equal(s.intact(), o.mu())
    else:
        s.step(scales[:20])
        o.step(scales[:20])
        u, v, _ = s.state()
        ou, ov, _ = o.state()
        assert np.linalg.norm(u - ou) <= 1e-9 * np.linalg.norm(ou)
        assert np.linalg.norm(v - ov) <= 1e-9 * np.linalg.norm(ov)
        s.step(scales[20:])
        o.step(scales[20:])
        mine, ref = s.intact() == 0, o.mu() == 0
        if ref.sum():
            assert 1.0 - np.logical_xor(mine, ref).sum() / ref.sum() >= 0.999
            _crack_within_delta(pairs, mine, ref, sc, tip=False)


@pytest.mark.parametrize("name,steps", [("cfg4_small", 100), ("cfg5_core_small", 200),
                                        ("block3d", 300)])
def test_lat3_screen_is_exact(name, steps, monkeypatch):
    """The 3D cold-tile break screen (per-tile node-edge maxima from the tiled ubar
    kernel) only skips break tests its bound proves cannot fire: fields, bond
    states and broken counts are bitwise those of the test on every tile."""
    sc = Scenario(cf.get(name))
    out = {}
    for screen in (True, False):
        s = PDSolver.from_scenario(sc, mode=capi.FAST).find_pe_pairs()
        s.set_option(capi.OPT_BREAK_SCREEN, 1 if screen else 0)
        assert s.info()["stencil_size"] == 122
        v0 = sc.initial_velocity()
        if v0.any():
            z = np.zeros(sc.n_dof)
            s.set_state(z, v0, z)
        s.initial_acceleration(sc.load_scale(0.0))
        nb = [s.step(sc.scales(i, 20)) for i in range(1, steps + 1, 20)]
        out[screen] = (nb, *s.state(), s.intact())
    a, b = out[True], out[False]
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_cfg5_core_small_notched_3d(mode):
    """BASELINE cfg5's PD core physics at 40x80x10 (0.25 mm, 3D polygon pre-notch
    through the thickness, 12 MPa horizon bands, constant micromodulus, dt 4 ns):
    device families == oracle pairs (notch cut included); deterministic bitwise vs
    the matrix-free oracle; fast mode within the north-star tolerances."""
    sc = Scenario(cf.get("cfg5_core_small"))
    s = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    if mode == capi.FAST:
        assert s.info()["path"] == 1 and s.info()["stencil_size"] == 122
    pairs = po.find_pairs(3, sc.centroid, sc.volume, sc.delta, sc.notches())
    assert np.array_equal(s.pairs(), pairs)
    assert len(pairs) < len(po.find_pairs(3, sc.centroid, sc.volume, sc.delta))  # the notch cuts
    ext = sc.cfg["ext"]
    o = po.OraclePD(dict(dim=3, n_nodes=sc.n_nodes, conn=sc.conn, centroid=sc.centroid,
                         volume=sc.volume, pairs=pairs, mass=sc.mass, p_ext=sc.p_ext,
                         delta=sc.delta, s_crit=sc.s_crit, dt=sc.dt, micromodulus=1,
                         c_const=ext["c"]), po.MF)
    s.initial_acceleration(sc.load_scale(0.0))
    o.init(sc.load_scale(0.0))
    scales = sc.scales(1, 120)
    if mode == capi.DETERMINISTIC:
        nb = s.step(scales)
        br, _ = o.step(scales)
        u, v, a = s.state()
        ou, ov, oa = o.state()
        assert nb == len(br)
        assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(a, oa)
        assert np.array_equal(s.intact(), o.mu())
    else:
        s.step(scales[:10])
        o.step(scales[:10])
        u, v, _ = s.state()
        ou, ov, _ = o.state()
        assert np.linalg.norm(u - ou) <= 1e-9 * np.linalg.norm(ou)
        assert np.linalg.norm(v - ov) <= 1e-9 * np.linalg.norm(ov)
        s.step(scales[10:])
        o.step(scales[10:])
        mine, ref = s.intact() == 0, o.mu() == 0
        if ref.sum():
            assert 1.0 - np.logical_xor(mine, ref).sum() / ref.sum() >= 0.999
            _crack_within_delta(pairs, mine, ref, sc, tip=True)


# ----- known-answer tests on the device (test_perifem.cpp) ------------------

def _kat_solver(mesh, pairs, s_crit, mode, delta=1.5, l=0.375):
    n = len(mesh["nodes"])
    s = PDSolver(dim=2, nodes=mesh["nodes"], conn=mesh["conn"], mass=np.full(2 * n, 1e300),
                 p_ext=np.zeros(2 * n), delta=delta, dt=1e-6, c0=1e9, l=l, s_crit=s_crit,
                 mode=mode)
    s.set_pairs(pairs)
    return s


def _u_move(mesh, elem, comp, val):
    u = np.zeros(2 * len(mesh["nodes"]))
    for nd in mesh["conn"][elem]:
        u[2 * nd + comp] = val
    return u


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_kat_threshold_inclusive_irreversible(mode):
    m = km.disjoint_quads()
    s_crit = 0.1
    s = _kat_solver(m, [[0, 1]], s_crit, mode)
    z = np.zeros(16)
    # v = a = 0 and a huge mass: the step's displacement is u itself, so the
    # device break test runs on exactly this u (driver_run.hpp:228-229)
    s.set_state(_u_move(m, 1, 0, s_crit - 1e-9), z, z)
    assert s.step([0.0]) == 0 and s.intact()[0] == 1
    s.set_state(_u_move(m, 1, 0, s_crit), z, z)
    if mode == capi.DETERMINISTIC:
        assert s.step([0.0]) == 1 and s.intact()[0] == 0
    else:  # squared test at exactly s_crit may round either way; go just above
        s.set_state(_u_move(m, 1, 0, s_crit * (1 + 1e-12)), z, z)
        assert s.step([0.0]) == 1 and s.intact()[0] == 0
    s.set_state(_u_move(m, 1, 0, 2 * s_crit), z, z)
    assert s.step([0.0]) == 0 and s.intact()[0] == 0


def test_kat_damage_half():
    m = km.grid(3, 1, 1.0)
    s = _kat_solver(m, [[0, 1], [1, 2]], 0.1, capi.DETERMINISTIC)
    z = np.zeros(2 * len(m["nodes"]))
    e, _ = s.damage_field()
    assert (e == 0).all()
    # stretch only the (0,1) bond: move element 0 left (its nodes are shared with
    # element 1 on one side, so use a displacement field that separates them)
    u = np.zeros_like(z)
    for nd in (0, 4):  # left edge nodes of element 0
        u[2 * nd] = -1.0
    s.set_state(u, z, z)
    s.step([0.0])
    e, _ = s.damage_field()
    assert e[1] == pytest.approx(0.5) and e[0] == pytest.approx(1.0) and e[2] == 0.0


def test_kat_no_fracture_when_s_crit_zero():
    m = km.disjoint_quads()
    s = _kat_solver(m, [[0, 1]], 0.0, capi.DETERMINISTIC)
    z = np.zeros(16)
    s.set_state(_u_move(m, 1, 0, 5.0), z, z)
    assert s.step([0.0]) == 0 and s.intact()[0] == 1


def test_device_notch_cases():
    m = km.grid(2, 1, 1.0)
    n = len(m["nodes"])

    def count(notch):
        s = PDSolver(dim=2, nodes=m["nodes"], conn=m["conn"], mass=np.ones(2 * n),
                     p_ext=np.zeros(2 * n), delta=1.01, dt=1e-6, c0=1.0, l=0.5,
                     notch_npts=[2], notch_pts=notch)
        return s.find_pe_pairs().info()["n_bonds"]

    assert count([1.0, -0.5, 0, 1.0, 1.5, 0]) == 0
    assert count([1.0, 2.0, 0, 1.0, 3.0, 0]) == 1
    assert count([1.0, 0.5, 0, 1.0, 2.0, 0]) == 0


def test_non_positive_mass_is_solver_error():
    m = km.disjoint_quads()
    with pytest.raises(capi.SolverError):
        PDSolver(dim=2, nodes=m["nodes"], conn=m["conn"], mass=np.zeros(16),
                 p_ext=np.zeros(16), delta=1.5, dt=1e-6, c0=1.0, l=0.5)


def test_implicit_pd_rejected():
    m = km.disjoint_quads()
    with pytest.raises(capi.ConfigError):
        PDSolver(dim=2, nodes=m["nodes"], conn=m["conn"], mass=np.ones(16),
                 p_ext=np.zeros(16), delta=1.5, dt=1e-6, c0=1.0, l=0.5, beta=0.25)


# ----- full-size (BASELINE cfg3) size-independent properties -----------------

@pytest.fixture(scope="module")
def cfg3():
    sc = Scenario(cf.get("cfg3"))
    return sc


def test_cfg3_families_match_oracle(cfg3):
    s = PDSolver.from_scenario(cfg3, mode=capi.FAST).find_pe_pairs()
    p = s.pairs()
    assert len(p) == 22_331_624  # SURVEY.md 8(a), reference find_pe_pairs at 2000x800
    ref = po.find_pairs(2, cfg3.centroid, cfg3.volume, cfg3.delta, cfg3.notches())
    assert np.array_equal(p, ref)


def test_cfg3_linearity_and_momentum(cfg3):
    """No fracture: the step is linear in (u, v, a, P) and internal forces are
    self-equilibrated (sum of K u over all dofs vanishes)."""
    s1 = PDSolver.from_scenario(cfg3, mode=capi.FAST, s_crit=0.0).find_pe_pairs()
    s2 = PDSolver.from_scenario(cfg3, mode=capi.FAST, s_crit=0.0).find_pe_pairs()
    sc = np.full(20, 1.0)
    s1.initial_acceleration(1.0)
    s2.initial_acceleration(2.0)
    s1.step(sc)
    s2.step(2.0 * sc)
    u1, v1, a1 = s1.state()
    u2, v2, a2 = s2.state()
    assert np.linalg.norm(u2 - 2 * u1) <= 1e-12 * np.linalg.norm(u2)
    # momentum: sum M a == sum P (internal forces cancel pairwise)
    P = cfg3.p_ext
    f_int = P - cfg3.mass * a1
    assert abs(f_int[0::2].sum()) <= 1e-9 * np.abs(f_int).sum()
    assert abs(f_int[1::2].sum()) <= 1e-9 * np.abs(f_int).sum()


def test_cfg3_screen_exact_over_baseline_horizon(cfg3, monkeypatch):
    """BASELINE cfg3 over its full 1000-step horizon (cracks start near step 700):
    the screened kernel's per-batch broken counts, bond states and fields are bitwise
    those of the unscreened candidate pass."""
    out = {}
    for screen, clean in ((True, True), (False, True), (True, False)):
        s = PDSolver.from_scenario(cfg3, mode=capi.FAST).find_pe_pairs()
        s.set_option(capi.OPT_BREAK_SCREEN, 1 if screen else 0)
        s.set_option(capi.OPT_CLEAN_TILES, 1 if clean else 0)
        s.initial_acceleration(cfg3.load_scale(0.0))
        nb = [s.step(cfg3.scales(i, 100)) for i in range(1, 1001, 100)]
        out[screen, clean] = (nb, *s.state(), s.intact())
    a = out[True, True]
    assert sum(a[0]) > 1000
    for b in (out[False, True], out[True, False]):  # (clean tiles off: every tile staged)
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(x, y)


# ----- fp32-position / fp64-accumulate variant (BASELINE cfg3, PMTS_FAST_F32POS) -----
# Tolerances of the variant (the north star states none for it): fields within
# 1e-5 relative L2 of the oracle before crack initiation, >= 99.9 % broken-set
# agreement afterwards (measured: <= 1.7e-6 and 100 % on every 2D fixture).
F32_TOL = 1e-5


@pytest.mark.parametrize("name", ["mini", "cfg1_200", "bp_coarse_2000"])
def test_f32pos_tolerances(name):
    g, sc, s = _solver(name, capi.FAST_F32POS)
    s.find_pe_pairs()
    assert s.info()["path"] == 2
    steps = g["meta"]["steps"]
    s.initial_acceleration(g["scale"][0])
    br = g["broken"]
    first = int(br[0, 0]) if len(br) else steps + 1
    pre = min(first - 1, steps)
    o = po.OraclePD(oracle_sys(g, sc), po.MF)
    o.init(g["scale"][0])
    s.step(g["scale"][1:pre + 1])
    o.step(g["scale"][1:pre + 1])
    u, v, _ = s.state()
    ou, ov, _ = o.state()
    assert 0 < np.linalg.norm(u - ou) <= F32_TOL * np.linalg.norm(ou)  # > 0: fp32 really ran
    assert np.linalg.norm(v - ov) <= F32_TOL * np.linalg.norm(ov)
    s.step(g["scale"][pre + 1:steps + 1])
    mine = s.intact() == 0
    ref = np.zeros(len(g["pairs"]), dtype=bool)
    ref[g["broken"][:, 1]] = True
    agree = 1.0 - np.logical_xor(mine, ref).sum() / max(ref.sum(), 1)
    assert agree >= 0.999, agree


@pytest.mark.parametrize("nx,ny,steps", [(124, 62, 300), (33, 65, 200)])
def test_f32pos_screen_is_exact(nx, ny, steps, monkeypatch):
    """The cold-tile screen of the fp32 variant (bound against its lowered fp32
    candidate thresholds) changes nothing: bitwise the candidate pass on every tile."""
    sc = _plate(nx, ny)
    out = {}
    for screen in (True, False):
        s = PDSolver.from_scenario(sc, mode=capi.FAST_F32POS).find_pe_pairs()
        s.set_option(capi.OPT_BREAK_SCREEN, 1 if screen else 0)
        s.initial_acceleration(sc.load_scale(0.0))
        nb = s.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
        out[screen] = (nb, *s.state(), s.intact())
    a, b = out[True], out[False]
    assert a[0] == b[0] and a[0] > 0
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name,over", [("block3d", {}), ("mini", {"lattice": (0, 0, 0)})])
def test_f32pos_needs_the_2d_tile_kernel(name, over):
    """Only the 2D lattice tile kernel has the fp32-position arithmetic: 3D and
    unstructured families are a ConfigError (status 2), never a silent fp64 run."""
    g, sc, s = _solver(name, capi.FAST_F32POS, **over)
    s.find_pe_pairs()
    s.initial_acceleration(g["scale"][0])
    with pytest.raises(capi.ConfigError, match="F32POS"):
        s.step(g["scale"][1:3])


def test_cfg3_f32pos_vs_fp64_over_1500_steps(cfg3):
    """BASELINE cfg3 through crack growth: the fp32-position variant against the
    fp64 kernel -- broken sets agree >= 99.9 % (measured 100 %), displacements
    within 1e-6 relative L2 (measured 9e-8)."""
    out = {}
    for mode in (capi.FAST, capi.FAST_F32POS):
        s = PDSolver.from_scenario(cfg3, mode=mode).find_pe_pairs()
        s.initial_acceleration(cfg3.load_scale(0.0))
        s.step(cfg3.scales(1, 1500))
        u, _, _ = s.state()
        out[mode] = (u, s.intact() == 0)
    (u0, b0), (u1, b1) = out[capi.FAST], out[capi.FAST_F32POS]
    assert b0.sum() > 10000
    assert 1.0 - np.logical_xor(b0, b1).sum() / b0.sum() >= 0.999
    assert np.linalg.norm(u1 - u0) <= 1e-6 * np.linalg.norm(u0)


@pytest.mark.parametrize("nx,ny,steps", [(124, 62, 200), (64, 93, 150), (60, 35, 150)])
def test_tile9_split_launch_bitwise(nx, ny, steps, monkeypatch):
    """The halo-overlap launch split (edge tile rows, then the interior while the
    exchange runs; forced on one GPU by PMTS_OPT_HALO_OVERLAP) is bitwise the single
    launch: same fields, bond states and per-step broken counts, tracked rows too."""
    sc = _plate(nx, ny)
    out = {}
    for split in (True, False):
        s = PDSolver.from_scenario(sc, mode=capi.FAST).find_pe_pairs()
        s.set_option(capi.OPT_HALO_OVERLAP, 1 if split else 0)
        s.initial_acceleration(sc.load_scale(0.0))
        nb = s.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
        trk, cnt = s.step_tracked([sc.load_scale(i * sc.dt) for i in range(steps + 1, steps + 21)],
                                  np.array([1, 2 * (sc.n_nodes // 2), 2 * sc.n_nodes - 1], np.int32))
        out[split] = (nb, *s.state(), s.intact(), trk, cnt)
    a, b = out[True], out[False]
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)


# ----- damage_field and the intact export on the lattice path (device) -------

@pytest.mark.parametrize("name,steps", [("mini", 80), ("cfg1", 1000), ("block3d", 100),
                                        ("cfg5_core_small", 150)])
def test_lattice_damage_and_intact_on_device(name, steps):
    """Fast mode on the lattice stencil (2D tile kernel: bond state at the lower end;
    3D: both ends): pmts_pd_get_intact and pmts_pd_damage run over the stencil bits
    on the device.  The oracle's damage_field (perifem.hpp:202-231) given the same
    bond states is bitwise the device's, element and node."""
    sc = Scenario(cf.get(name))
    s = PDSolver.from_scenario(sc, mode=capi.FAST).find_pe_pairs()
    assert s.info()["path"] in (1, 2)
    s.initial_acceleration(sc.load_scale(0.0))
    s.step(sc.scales(1, steps))
    pairs = s.pairs()
    mu = s.intact()
    assert len(mu) == len(pairs) and (mu == 0).sum() > 0
    ext = sc.cfg["ext"]
    sysd = dict(dim=sc.dim, n_nodes=sc.n_nodes, conn=sc.conn, centroid=sc.centroid,
                volume=sc.volume, pairs=pairs, mass=sc.mass, p_ext=sc.p_ext, delta=sc.delta,
                l=sc.l, c0=sc.c0, s_crit=sc.s_crit, dt=sc.dt)
    if ext.get("micromodulus") == "constant":
        sysd.update(micromodulus=1, c_const=ext["c"])
    o = po.OraclePD(sysd, po.MF)
    o.set_mu(mu)
    oe, on = o.damage()
    e, n = s.damage_field()
    assert np.array_equal(e, oe) and np.array_equal(n, on)
    assert e.max() > 0


# ----- edge cases: empty families, one element, empty batches ----------------

@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_no_bonds_steps_like_the_oracle(mode):
    """A horizon below the element spacing (no family has a member) and a single-element
    mesh: the neighbour build returns no pairs, stepping runs the free Newmark update
    under the loads, and the fields are the oracle's (bitwise in deterministic mode);
    an empty batch of steps changes nothing."""
    one = {"mesh.bounds": [0.0, 0.0, 1e-3, 1e-3], "mesh.notch1": None,
           "load.traction2": [1e-3 - 1e-4, -1.0, 1e-3 + 1e-4, 1.0, 16e6, 0.0]}
    for over in ({"pd.delta_factor": 0.4}, one):
        c = cf.get("mini", **over)
        sc = Scenario(c)
        s = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
        assert len(s.pairs()) == 0 and s.info()["n_bonds"] == 0
        assert len(s.intact()) == 0
        o = po.OraclePD(dict(dim=2, n_nodes=sc.n_nodes, conn=sc.conn, centroid=sc.centroid,
                             volume=sc.volume, pairs=np.zeros((0, 2), np.int32), mass=sc.mass,
                             p_ext=sc.p_ext, bc_dofs=sc.bc_dofs, bc_vel=sc.bc_vel,
                             delta=sc.delta, l=sc.l, c0=sc.c0, s_crit=sc.s_crit, dt=sc.dt),
                        po.MF)
        s.initial_acceleration(sc.load_scale(0.0))
        o.init(sc.load_scale(0.0))
        assert s.step([]) == 0
        assert s.step(sc.scales(1, 30)) == 0
        o.step(sc.scales(1, 30))
        u, v, a = s.state()
        ou, ov, oa = o.state()
        if mode == capi.DETERMINISTIC:
            assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(a, oa)
        else:
            assert np.linalg.norm(u - ou) <= 1e-12 * max(np.linalg.norm(ou), 1e-300)
        e, _ = s.damage_field()
        assert (e == 0).all()


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
def test_set_pairs_empty_and_break_log_empty(mode):
    """set_pairs with an empty list (the reference's find_pe_pairs may return none) and
    an empty break log."""
    m = km.disjoint_quads()
    s = _kat_solver(m, np.zeros((0, 2), np.int32), 0.1, mode)
    z = np.zeros(16)
    s.set_state(z, z, z)
    assert s.step([0.0, 0.0]) == 0
    if mode == capi.DETERMINISTIC:  # (the (step, i, j) log is a deterministic-mode record)
        assert len(s.break_log(10)) == 0
