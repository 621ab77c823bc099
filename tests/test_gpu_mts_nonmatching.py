"""GPU: the coupled MTS run on non-matching FE / PD meshes (extension, SURVEY.md
8(f) row 4; see tests/test_mts_nonmatching.py for the host side).

* fe_spacing == spacing: the device run is bitwise the conforming run (which
  tests/test_gpu_mts.py pins to the reference's own coupled loop);
* PD fixed at 0.25 mm, FE at 0.5 and 1 mm: the PD fields converge to the
  conforming run as the FE lattice refines (no oracle exists for the
  non-matching model; tolerances measured and written here)."""
import numpy as np
import pytest

from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.mts import MtsSolver

pytestmark = pytest.mark.gpu


def _rel(x, r):
    return np.linalg.norm(x - r) / max(np.linalg.norm(r), 1e-300)


@pytest.mark.parametrize("name,steps", [("mts_mini", 40), ("mts_mini_frac", 60), ("mts_bar3d", 15)])
def test_unit_ratio_runs_bitwise_as_conforming(name, steps):
    out = {}
    for nm in (False, True):
        sc = cf.get(name)
        if nm:
            sc["mesh"]["fe_spacing"] = sc["mesh"]["spacing"]
        s = MtsSolver(sc)
        s.initialize()
        reps = s.macro_step(steps)
        out[nm] = (s.state("fe"), s.state("pd"), s.lam(), s.intact(),
                   [r["newly_broken"] for r in reps])
    a, b = out[False], out[True]
    for w in (0, 1):
        for x, y in zip(a[w], b[w]):
            assert np.array_equal(x, y)
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]) and a[4] == b[4]


def test_fe_refinement_converges_to_conforming():
    res = {}
    for fe in (2.5e-4, 5e-4, 1e-3):
        sc = cf.get("mts_nm_strip")
        sc["mesh"]["fe_spacing"] = fe
        s = MtsSolver(sc)
        s.initialize()
        reps = s.macro_step(40)
        assert max(r["continuity"] for r in reps) <= 1e-8
        res[fe] = s.state("pd")[0]
    ref = res[2.5e-4]
    assert np.linalg.norm(ref) > 0
    e_half, e_one = _rel(res[5e-4], ref), _rel(res[1e-3], ref)
    print(f"PD u relL2 vs conforming: FE 0.5 mm {e_half:.3e}, FE 1 mm {e_one:.3e}")
    assert e_half < e_one
    assert e_one < 0.06  # measured 0.040 (FE 0.5 mm: 0.033) after 40 macro steps


def test_3d_nonmatching_bar_runs():
    """3D hex8 (mts_bar3d) with the PD lattice at half the FE spacing: the device
    run holds velocity continuity at every macro step and stays bounded."""
    from test_mts_nonmatching import nonmatching

    s = MtsSolver(nonmatching("mts_bar3d", 2))
    s.initialize()
    reps = s.macro_step(15)
    assert max(r["continuity"] for r in reps) <= 1e-8
    u_fe, u_pd = s.state("fe")[0], s.state("pd")[0]
    assert np.isfinite(u_fe).all() and np.isfinite(u_pd).all() and np.abs(u_pd).max() > 0
    # the PD field at the overlap follows the FE interpolant (coupled, not detached)
    sy = s.system()
    rp, ci, w = sy["cpl_fe_rowptr"], sy["cpl_fe_col"], sy["cpl_fe_w"]
    gfe = np.array([np.dot(w[rp[r]:rp[r + 1]], s.state("fe")[1][ci[rp[r]:rp[r + 1]]])
                    for r in range(len(rp) - 1)])
    gpd = s.state("pd")[1][sy["pd_dof"]]
    assert np.abs(gfe - gpd).max() <= 1e-8 * max(1.0, np.abs(gpd).max())


@pytest.mark.parametrize("name,fe,steps", [("mts_nm_strip", 1e-3, 40), ("mts_nm_strip", 5e-4, 40),
                                           ("cfg2_nm", None, 5)])
def test_sparse_explicit_h_fe_bitwise_unit_columns(name, fe, steps):
    """An explicit FE side's H_FE built directly as a sparse product (the default, no
    n_lambda^2 scratch: what BASELINE cfg5's 1.8M multipliers need) is bitwise the
    unit-column construction: same multipliers, states and iteration counts."""
    out = {}
    for mode in ("sparse", "unit_columns"):
        sc = cf.get(name)
        if fe:
            sc["mesh"]["fe_spacing"] = fe
        sc["run"]["interface"] = "matrix_free"
        sc["run"]["interface_h_fe"] = mode
        s = MtsSolver(sc)
        s.initialize()
        reps = s.macro_step(steps)
        out[mode] = (s.lam(), s.state("fe"), s.state("pd"),
                     [(r["interface_iterations"], r["newly_broken"]) for r in reps])
    a, b = out["sparse"], out["unit_columns"]
    assert np.array_equal(a[0], b[0]) and a[3] == b[3]
    for w in (1, 2):
        for x, y in zip(a[w], b[w]):
            assert np.array_equal(x, y)
