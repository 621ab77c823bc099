"""Scenario definitions for the PD fine-step path.

Each scenario is a plain dict in the reference's own config vocabulary
(``[section] key = value``, reference: proj/include/perimts/config.hpp:18-177,
keys and defaults from proj/include/perimts/scenario.hpp:90-258).  The same
dict drives three consumers:

* ``render_cfg`` -- text for the reference's ``load_scenario`` (the oracle
  harness ``oracle/_ref/ref_driver`` and the bench's reference arm);
* ``paper_2403_03605_b200.scenario.build`` -- the native C++ setup behind the
  C-ABI (structured mesh, geometry, traction bands, lumped mass, loads);
* the tests, which pick small members for parity.

BASELINE-only extensions that the reference cannot express (constant
micromodulus c = 9E/(pi h delta^3) or 18K/(pi delta^4), per-bond s0 factor)
live under the ``ext`` key and are never rendered into reference configs.
"""
from __future__ import annotations

import copy
import math

# Material shared by BASELINE configs 1-5 (BASELINE.json configs[0]).
_E = 72e9
_RHO = 2440.0
_G0 = 3.8


def _plate2d(nx: int, ny: int, dx: float, *, E: float, rho: float, delta_factor: float,
             l_factor: float, s_crit: float, dt: float, steps: int, m: int = 1,
             notch=(-0.001, 0.02, 0.05, 0.02), traction: float = 12e6) -> dict:
    lx, ly = nx * dx, ny * dx
    return {
        "mesh": {"kind": "generated", "dim": 2, "bounds": [0.0, 0.0, lx, ly], "spacing": dx,
                 "notch1": list(notch) if notch else None},
        "material": {"E": E, "nu": 0.3333333333333333, "rho": rho,
                     "formulation": "plane_stress"},
        "pd": {"delta_factor": delta_factor, "l_factor": l_factor, "s_crit": s_crit},
        "load": {
            "traction1": [-0.01, ly - 1e-7, lx + 0.01, ly + 1e-7, 0.0, traction],
            "traction2": [-0.01, -1e-7, lx + 0.01, 1e-7, 0.0, -traction],
        },
        "time": {"dt_pd": dt, "m": m, "total_time": dt * m * round(steps / m),
                 "gamma_pd": 0.5, "beta_pd": 0.0},
        "run": {"mode": "pure_pd"},
        "output": {"interval": 0.0},
        "ext": {},
    }


def s0_2d(E: float, G0: float, delta: float) -> float:
    """BASELINE cfg1: s0 = sqrt(4 pi G0 / (9 E delta))."""
    return math.sqrt(4.0 * math.pi * G0 / (9.0 * E * delta))


def s0_3d(E: float, nu: float, G0: float, delta: float) -> float:
    """BASELINE cfg4: s0 = sqrt(5 G0 / (9 K delta)), K = E / (3 (1 - 2 nu))."""
    K = E / (3.0 * (1.0 - 2.0 * nu))
    return math.sqrt(5.0 * G0 / (9.0 * K * delta))


def scenarios() -> dict:
    s = {}
    # Reference-native twin of BASELINE cfg1 (SURVEY.md 8(c) fixture 1):
    # the shipped branching plate (coarse) run in pure-PD mode.
    s["bp_coarse"] = _plate2d(200, 80, 5e-4, E=65e9, rho=2235.0, delta_factor=3.03,
                              l_factor=10.0, s_crit=0.002689, dt=1e-8, steps=6000, m=10)
    # BASELINE cfg1 analog in the reference's own form (SURVEY.md 8(c) fixture 2):
    # exponential micromodulus with l = delta, s_crit = s0 from G0.
    d1 = 3.015 * 5e-4
    s["cfg1"] = _plate2d(200, 80, 5e-4, E=_E, rho=_RHO, delta_factor=3.015, l_factor=1.0,
                         s_crit=2.211e-4, dt=2.5e-8, steps=1000)
    # BASELINE cfg1 with its own constant micromodulus (extension, restatement only).
    s["cfg1_const"] = copy.deepcopy(s["cfg1"])
    s["cfg1_const"]["ext"] = {"micromodulus": "constant",
                              "c": 9.0 * _E / (math.pi * 1e-3 * d1 ** 3), "h": 1e-3}
    # BASELINE cfg3: 2000 x 800 at 0.05 mm, per-bond s0 factor U[0.95, 1.05].
    d3 = 3.015 * 5e-5
    s["cfg3"] = _plate2d(2000, 800, 5e-5, E=_E, rho=_RHO, delta_factor=3.015, l_factor=1.0,
                         s_crit=round(s0_2d(_E, _G0, d3), 7), dt=5e-9, steps=1000)
    s["cfg3"]["ext"] = {"micromodulus": "constant",
                        "c": 9.0 * _E / (math.pi * 1e-3 * d3 ** 3), "h": 1e-3,
                        "s_crit_spread": 0.05, "seed": 0x5eed5 + 3}
    # cfg3's own physics (constant micromodulus c h / r^3, per-bond s0 spread, the
    # same seed) on a 400 x 160 sub-plate at the same dx: 20 x 8 mm, the pre-crack
    # from the left edge to mid-width at mid-height, the same 12 MPa bands.  The
    # oracle finishes it in seconds; it cracks near step 150 (tests/test_gpu_cfg3_physics.py).
    s["cfg3_sub"] = _plate2d(400, 160, 5e-5, E=_E, rho=_RHO, delta_factor=3.015,
                             l_factor=1.0, s_crit=s["cfg3"]["pd"]["s_crit"], dt=5e-9,
                             steps=400, notch=(-0.001, 0.004, 0.01, 0.004))
    s["cfg3_sub"]["ext"] = copy.deepcopy(s["cfg3"]["ext"])
    # Reference-native analog of cfg3 (exponential kernel, scalar s_crit): the
    # form the reference arm and the deterministic path run at full size.
    s["cfg3_native"] = copy.deepcopy(s["cfg3"])
    s["cfg3_native"]["ext"] = {}
    # Bounded CPU sample of cfg3 for the reference arm / cpu_baseline: the same
    # dx, horizon, material and loading on a 500 x 200 sub-plate (25 x 10 mm,
    # notch scaled to the same fraction), reference-native kernel.
    s["cfg3_sample"] = _plate2d(500, 200, 5e-5, E=_E, rho=_RHO, delta_factor=3.015,
                                l_factor=1.0, s_crit=s["cfg3"]["pd"]["s_crit"], dt=5e-9,
                                steps=1000, notch=(-0.00025, 0.005, 0.0125, 0.005))
    # Miniature notched plate of the reference's driver test
    # (proj/tests/test_driver.cpp:296-333), horizontal tension.
    mini = _plate2d(40, 16, 1e-3, E=72e9, rho=2235.0, delta_factor=3.03, l_factor=10.0,
                    s_crit=0.0004, dt=5e-8, steps=80, notch=(0.02, 0.016, 0.02, 0.010))
    mini["load"] = {"traction1": [-1e-9, -1.0, 1e-9, 1.0, -16e6, 0.0],
                    "traction2": [0.0399, -1.0, 0.0401, 1.0, 16e6, 0.0]}
    s["mini"] = mini
    # Small 3D hex8 block (probe on 20x20x10): tension on top/bottom.
    d3d = 3.015 * 5e-4
    blk = {
        "mesh": {"kind": "generated", "dim": 3, "bounds": [0, 0, 0, 0.005, 0.005, 0.004],
                 "spacing": 5e-4, "notch1": None},
        "material": {"E": _E, "nu": 0.25, "rho": _RHO, "formulation": "three_d"},
        "pd": {"delta_factor": 3.015, "l_factor": 1.0,
               "s_crit": round(s0_3d(_E, 0.25, _G0, d3d), 7)},
        "load": {"traction1": [-1, -1, 0.004 - 1e-7, 1, 1, 0.004 + 1e-7, 0, 0, 12e6],
                 "traction2": [-1, -1, -1e-7, 1, 1, 1e-7, 0, 0, -12e6]},
        "time": {"dt_pd": 2e-8, "m": 1, "total_time": 2e-8 * 100, "gamma_pd": 0.5,
                 "beta_pd": 0.0},
        "run": {"mode": "pure_pd"},
        "output": {"interval": 0.0},
        "ext": {},
    }
    s["block3d"] = blk
    # BASELINE cfg4: 3D impact block 200 x 200 x 50 at 0.5 mm (2.0M hexes), constant
    # micromodulus c = 18K/(pi delta^4), s0 = sqrt(5 G0/(9 K delta)), 20 m/s +-5% seeded
    # initial velocity on a 10 x 10 mm patch of the top face (extension: the reference
    # has no initial-velocity hook), dt = 20 ns, 500 steps.
    K4 = _E / (3.0 * (1.0 - 2.0 * 0.25))
    c4 = {
        "mesh": {"kind": "generated", "dim": 3, "bounds": [0, 0, 0, 0.1, 0.1, 0.025],
                 "spacing": 5e-4, "notch1": None},
        "material": {"E": _E, "nu": 0.25, "rho": _RHO, "formulation": "three_d"},
        "pd": {"delta_factor": 3.015, "l_factor": 1.0,
               "s_crit": round(s0_3d(_E, 0.25, _G0, d3d), 7)},
        "load": {},
        "time": {"dt_pd": 2e-8, "m": 1, "total_time": 2e-8 * 500, "gamma_pd": 0.5,
                 "beta_pd": 0.0},
        "run": {"mode": "pure_pd"},
        "output": {"interval": 0.0},
        "ext": {"micromodulus": "constant", "c": 18.0 * K4 / (math.pi * d3d ** 4),
                "initial_velocity": {"lo": [0.045, 0.045, 0.025 - 1e-7],
                                     "hi": [0.055, 0.055, 0.025 + 1e-7],
                                     "comp": 2, "value": -20.0, "spread": 0.05,
                                     "seed": 0x5eed5 + 4}},
    }
    s["cfg4"] = c4
    # small 3D twin of cfg4 for tests (same physics, 20 x 20 x 10)
    c4s = copy.deepcopy(c4)
    c4s["mesh"]["bounds"] = [0, 0, 0, 0.01, 0.01, 0.005]
    c4s["ext"]["initial_velocity"].update(lo=[0.003, 0.003, 0.005 - 1e-7],
                                          hi=[0.007, 0.007, 0.005 + 1e-7])
    c4s["time"]["total_time"] = 2e-8 * 100
    s["cfg4_small"] = c4s
    # BASELINE cfg5's PD core as a pure-PD run -- the largest PD configuration (the
    # north star's scaling target): 100 x 200 x 10 mm at 0.25 mm (400 x 800 x 40 =
    # 12.8M hexes, 755M bonds), a 40 mm through-thickness pre-notch at mid-height
    # from the left edge, 12 MPa on the top / bottom faces (horizon bands), constant
    # micromodulus with nu = 1/4, dt = 4 ns; 2000 fine steps = cfg5's 100 coarse x m=20
    d5 = 3.015 * 2.5e-4
    K5 = _E / (3.0 * (1.0 - 2.0 * 0.25))
    c5 = {
        "mesh": {"kind": "generated", "dim": 3, "bounds": [0, 0, 0, 0.1, 0.2, 0.01],
                 "spacing": 2.5e-4,
                 "notch1": [-0.001, 0.1, -0.001, 0.04, 0.1, -0.001, 0.04, 0.1, 0.011,
                            -0.001, 0.1, 0.011]},
        "material": {"E": _E, "nu": 0.25, "rho": _RHO, "formulation": "three_d"},
        "pd": {"delta_factor": 3.015, "l_factor": 1.0,
               "s_crit": round(s0_3d(_E, 0.25, _G0, d5), 7)},
        "load": {"traction1": [-1, 0.2 - 1e-7, -1, 1, 0.2 + 1e-7, 1, 0, 12e6, 0],
                 "traction2": [-1, -1e-7, -1, 1, 1e-7, 1, 0, -12e6, 0]},
        "time": {"dt_pd": 4e-9, "m": 1, "total_time": 4e-9 * 2000, "gamma_pd": 0.5,
                 "beta_pd": 0.0},
        "run": {"mode": "pure_pd"},
        "output": {"interval": 0.0},
        "ext": {"micromodulus": "constant", "c": 18.0 * K5 / (math.pi * d5 ** 4)},
    }
    s["cfg5_core"] = c5
    c5s = copy.deepcopy(c5)  # small twin for tests: 10 x 20 x 2.5 mm at 0.25 mm
    c5s["mesh"]["bounds"] = [0, 0, 0, 0.01, 0.02, 0.0025]
    c5s["mesh"]["notch1"] = [-0.001, 0.01, -0.001, 0.004, 0.01, -0.001, 0.004, 0.01, 0.0035,
                             -0.001, 0.01, 0.0035]
    c5s["load"] = {"traction1": [-1, 0.02 - 1e-7, -1, 1, 0.02 + 1e-7, 1, 0, 12e6, 0],
                   "traction2": [-1, -1e-7, -1, 1, 1e-7, 1, 0, -12e6, 0]}
    c5s["time"]["total_time"] = 4e-9 * 200
    s["cfg5_core_small"] = c5s

    # --- coupled MTS --------------------------------
    # Miniature coupled strip: 30 x 10 elements at 1 mm, PD box = middle third
    # (full height, so no interior corners -- SURVEY F6), overlap one element,
    # traction on the right (FE) face, left face fixed.  Explicit FE (beta_fe =
    # 0, stable at 1 mm / 40 ns) and a dense interface (n_lambda <= 400).
    mts = {
        "mesh": {"kind": "generated", "dim": 2, "bounds": [0.0, 0.0, 0.03, 0.01],
                 "spacing": 1e-3, "notch1": None},
        "material": {"E": 65e9, "nu": 0.3333333333333333, "rho": 2235.0,
                     "formulation": "plane_stress"},
        "pd": {"delta_factor": 2.2, "l_factor": 8.0, "s_crit": 0.0},
        "region": {"pd_box1": [0.01, 0.0, 0.02, 0.01], "overlap_width_factor": 1.0,
                   "weight_kind": "cubic"},
        "load": {"traction1": [0.03 - 1e-7, -0.001, 0.03 + 1e-7, 0.011, 40e6, 0.0],
                 "fixed1": [-1e-7, -0.001, 1e-7, 0.011]},
        "time": {"dt_pd": 2e-8, "m": 2, "total_time": 2e-8 * 2 * 40, "gamma_fe": 0.5,
                 "beta_fe": 0.0, "gamma_pd": 0.5, "beta_pd": 0.0},
        "run": {"mode": "coupled_mts", "interface": "auto"},
        "output": {"interval": 0.0},
        "ext": {},
    }
    s["mts_mini"] = mts
    # implicit FE (Newmark beta 1/4: PCG solves), m = 4
    mi = copy.deepcopy(mts)
    mi["time"].update(beta_fe=0.25, m=4, total_time=2e-8 * 4 * 20)
    s["mts_mini_implicit"] = mi
    # fracture in the PD core: notch-free tension with a low critical stretch
    mf = copy.deepcopy(mts)
    mf["pd"]["s_crit"] = 2.5e-4
    mf["time"].update(total_time=2e-8 * 2 * 60)
    s["mts_mini_frac"] = mf
    # matrix-free interface (forced), implicit FE
    mm = copy.deepcopy(mi)
    mm["run"]["interface"] = "matrix_free"
    s["mts_mini_mfree"] = mm
    # 3D coupled bar (hex8): 12 x 4 x 4 elements at 1 mm, PD box the middle third,
    # tension on the +x face, -x face fixed, implicit FE
    m3 = {
        "mesh": {"kind": "generated", "dim": 3, "bounds": [0, 0, 0, 0.012, 0.004, 0.004],
                 "spacing": 1e-3, "notch1": None},
        "material": {"E": 65e9, "nu": 0.25, "rho": 2235.0, "formulation": "three_d"},
        "pd": {"delta_factor": 2.2, "l_factor": 8.0, "s_crit": 0.0},
        "region": {"pd_box1": [0.004, 0.0, 0.0, 0.008, 0.004, 0.004],
                   "overlap_width_factor": 1.0, "weight_kind": "linear"},
        "load": {"traction1": [0.012 - 1e-7, -0.001, -0.001, 0.012 + 1e-7, 0.005, 0.005,
                               30e6, 0.0, 0.0],
                 "fixed1": [-1e-7, -0.001, -0.001, 1e-7, 0.005, 0.005]},
        "time": {"dt_pd": 2e-8, "m": 2, "total_time": 2e-8 * 2 * 15, "gamma_fe": 0.5,
                 "beta_fe": 0.25, "gamma_pd": 0.5, "beta_pd": 0.0},
        "run": {"mode": "coupled_mts", "interface": "auto"},
        "output": {"interval": 0.0},
        "ext": {},
    }
    s["mts_bar3d"] = m3
    # the same bar 8 mm deep (8 element layers along z, the slowest axis): a 3D coupled
    # run that two PD shards can split (tests/test_gpu_mts_shards.py), with fracture
    m3t = copy.deepcopy(m3)
    m3t["mesh"]["bounds"] = [0, 0, 0, 0.012, 0.004, 0.008]
    m3t["region"]["pd_box1"] = [0.004, 0.0, 0.0, 0.008, 0.004, 0.008]
    m3t["load"] = {"traction1": [0.012 - 1e-7, -0.001, -0.001, 0.012 + 1e-7, 0.005, 0.009,
                                 30e6, 0.0, 0.0],
                   "fixed1": [-1e-7, -0.001, -0.001, 1e-7, 0.005, 0.009]}
    m3t["pd"]["s_crit"] = 1e-4
    m3t["time"]["total_time"] = 2e-8 * 2 * 40
    s["mts_bar3d_tall"] = m3t

    # BASELINE cfg2, conforming analog: the cfg1 plate and
    # material, PD band 100 x 20 mm in the middle, FE elsewhere -- both at 0.25 mm
    # (the reference cannot couple a non-matching 1 mm FE mesh), 2 mm gluing zones
    # with a linear weight, implicit FE (100 ns is beyond the explicit limit at
    # 0.25 mm), m = 10, 12 MPa traction on the top / bottom (FE) faces.
    for tag, dx in (("cfg2", 2.5e-4), ("cfg2_0p5", 5e-4)):
        dl = 3.015 * dx
        c2 = {
            "mesh": {"kind": "generated", "dim": 2, "bounds": [0.0, 0.0, 0.1, 0.04],
                     "spacing": dx, "notch1": [-0.001, 0.02, 0.05, 0.02]},
            "material": {"E": _E, "nu": 0.3333333333333333, "rho": _RHO,
                         "formulation": "plane_stress"},
            "pd": {"delta_factor": 3.015, "l_factor": 1.0, "s_crit": round(s0_2d(_E, _G0, dl), 7)},
            "region": {"pd_box1": [0.0, 0.01, 0.1, 0.03],
                       "overlap_width_factor": round(2e-3 / dx), "weight_kind": "linear"},
            "load": {"traction1": [-0.01, 0.04 - 1e-7, 0.11, 0.04 + 1e-7, 0.0, 12e6],
                     "traction2": [-0.01, -1e-7, 0.11, 1e-7, 0.0, -12e6]},
            "time": {"dt_pd": 1e-8, "m": 10, "total_time": 1e-7 * 200, "gamma_fe": 0.5,
                     "beta_fe": 0.25, "gamma_pd": 0.5, "beta_pd": 0.0},
            "run": {"mode": "coupled_mts", "interface": "auto"},
            "output": {"interval": 0.0},
            "ext": {},
        }
        s[tag] = c2
    # BASELINE cfg2 as written (non-matching meshes, an extension -- DESIGN.md 11): the
    # PD band at 0.25 mm, FE elsewhere on a 1 mm lattice, explicit central-difference
    # FE (beta_fe = 0, dt_fe = 100 ns < the 1 mm CFL limit), 2 mm linear gluing zones
    nm = copy.deepcopy(s["cfg2"])
    nm["mesh"]["fe_spacing"] = 1e-3
    nm["time"]["beta_fe"] = 0.0
    s["cfg2_nm"] = nm
    # convergence family for the non-matching coupling: a 30 x 10 mm strip, PD at
    # 0.25 mm in the middle third, 2 mm gluing zones, explicit FE, traction on the
    # top face (FE and PD parts loaded at once), bottom face fixed;
    # mesh.fe_spacing in {0.25, 0.5, 1} mm (tests)
    cv = {
        "mesh": {"kind": "generated", "dim": 2, "bounds": [0.0, 0.0, 0.03, 0.01],
                 "spacing": 2.5e-4, "notch1": None, "fe_spacing": 1e-3},
        "material": {"E": _E, "nu": 0.3333333333333333, "rho": _RHO,
                     "formulation": "plane_stress"},
        "pd": {"delta_factor": 3.015, "l_factor": 1.0, "s_crit": 0.0},
        "region": {"pd_box1": [0.01, 0.0, 0.02, 0.01], "overlap_width_factor": 8.0,
                   "weight_kind": "linear"},
        "load": {"traction1": [-0.001, 0.01 - 1e-7, 0.031, 0.01 + 1e-7, 0.0, 40e6],
                 "fixed1": [-0.001, -1e-7, 0.031, 1e-7]},
        "time": {"dt_pd": 1e-8, "m": 2, "total_time": 1e-8 * 2 * 40, "gamma_fe": 0.5,
                 "beta_fe": 0.0, "gamma_pd": 0.5, "beta_pd": 0.0},
        "run": {"mode": "coupled_mts", "interface": "auto"},
        "output": {"interval": 0.0},
        "ext": {},
    }
    s["mts_nm_strip"] = cv
    # BASELINE cfg5 (configs[4]) as a coupled run: 400 x 200 x 10 mm plate, the PD core
    # 100 x 200 x 10 mm in the middle at 0.25 mm (400 x 800 x 40 = 12.8M hexes), FE hex8 at
    # 1 mm elsewhere (non-matching), 2 mm linear gluing zones inside the
    # core's x faces, explicit central-difference FE (dt_fe = 80 ns), m = 20 (dt_pd = 4
    # ns), a 40 mm through-thickness pre-notch at mid-height from the core's left face,
    # 12 MPa on the top / bottom faces, 100 coarse steps.  The coupled model's kernel is
    # the reference's calibrated exponential one (its coupled integrator has no other).
    d5 = 3.015 * 2.5e-4
    c5m = {
        "mesh": {"kind": "generated", "dim": 3, "bounds": [0, 0, 0, 0.4, 0.2, 0.01],
                 "spacing": 2.5e-4, "fe_spacing": 1e-3,
                 "notch1": [0.15, 0.1, -0.001, 0.19, 0.1, -0.001, 0.19, 0.1, 0.011,
                            0.15, 0.1, 0.011]},
        "material": {"E": _E, "nu": 0.25, "rho": _RHO, "formulation": "three_d"},
        "pd": {"delta_factor": 3.015, "l_factor": 1.0,
               "s_crit": round(s0_3d(_E, 0.25, _G0, d5), 7)},
        "region": {"pd_box1": [0.15, 0.0, 0.0, 0.25, 0.2, 0.01],
                   "overlap_width_factor": 8.0, "weight_kind": "linear"},
        "load": {"traction1": [-1, 0.2 - 1e-7, -1, 1, 0.2 + 1e-7, 1, 0, 12e6, 0],
                 "traction2": [-1, -1e-7, -1, 1, 1e-7, 1, 0, -12e6, 0]},
        "time": {"dt_pd": 4e-9, "m": 20, "total_time": 8e-8 * 100, "gamma_fe": 0.5,
                 "beta_fe": 0.0, "gamma_pd": 0.5, "beta_pd": 0.0},
        "run": {"mode": "coupled_mts", "interface": "auto"},
        "output": {"interval": 0.0},
        "ext": {},
    }
    s["cfg5_mts"] = c5m
    # its small twin (tests): 20 x 10 x 2 mm plate, 8 mm PD core at 0.25 mm, FE 1 mm
    c5t = copy.deepcopy(c5m)
    c5t["mesh"]["bounds"] = [0, 0, 0, 0.02, 0.01, 0.002]
    c5t["mesh"]["notch1"] = [0.006, 0.005, -0.001, 0.009, 0.005, -0.001, 0.009, 0.005,
                             0.003, 0.006, 0.005, 0.003]
    c5t["region"]["pd_box1"] = [0.006, 0.0, 0.0, 0.014, 0.01, 0.002]
    c5t["load"] = {"traction1": [-1, 0.01 - 1e-7, -1, 1, 0.01 + 1e-7, 1, 0, 12e6, 0],
                   "traction2": [-1, -1e-7, -1, 1, 1e-7, 1, 0, -12e6, 0]}
    c5t["time"]["total_time"] = 8e-8 * 20
    s["cfg5_mts_small"] = c5t
    return s


def stacked(name: str, n: int) -> dict:
    """Weak-scaling variant of a 2D plate scenario: n copies of its height stacked
    (same dx, material, loads on the new top/bottom, notch at the new mid-height)."""
    sc = get(name)
    if n == 1:
        return sc
    m = sc["mesh"]
    if m["dim"] == 3:  # 3D blocks stack along z (the slab axis); the impact patch stays on top
        b = list(m["bounds"])
        ztop = b[5]
        lz = (b[5] - b[2]) * n
        b[5] = b[2] + lz
        m["bounds"] = b
        for k in [k for k in m if k.startswith("notch") and m[k]]:  # through the new thickness
            pts = list(m[k])
            for q in range(2, len(pts), 3):
                if pts[q] > ztop:
                    pts[q] = b[5] + (pts[q] - ztop)
            m[k] = pts
        iv = sc["ext"].get("initial_velocity")
        if iv:
            iv["lo"][2] = b[5] - 1e-7
            iv["hi"][2] = b[5] + 1e-7
        return sc
    x0, y0, x1, y1 = m["bounds"]
    ly = (y1 - y0) * n
    m["bounds"] = [x0, y0, x1, y0 + ly]
    if m.get("notch1"):
        a, b, c, d = m["notch1"]
        mid = y0 + 0.5 * ly
        m["notch1"] = [a, mid, c, mid]
    t = sc["load"]["traction1"]
    sc["load"]["traction1"] = [t[0], y0 + ly - 1e-7, t[2], y0 + ly + 1e-7, t[4], t[5]]
    return sc


def get(name: str, **over) -> dict:
    sc = copy.deepcopy(scenarios()[name])
    for k, v in over.items():
        sec, key = k.split(".", 1)
        sc[sec][key] = v
    return sc


def n_steps(sc: dict) -> int:
    return int(round(sc["time"]["total_time"] / sc["time"]["dt_pd"]))


def render_cfg(sc: dict) -> str:
    """Reference config text (proj/include/perimts/config.hpp format)."""
    out = []
    for sec in ("mesh", "material", "pd", "region", "load", "time", "run", "output"):
        if sec not in sc:
            continue
        out.append(f"[{sec}]")
        for k, v in sc[sec].items():
            if v is None:
                continue
            if isinstance(v, (list, tuple)):
                v = " ".join(repr(float(x)) for x in v)
            elif isinstance(v, float):
                v = repr(v)
            out.append(f"{k} = {v}")
        out.append("")
    return "\n".join(out)
