"""GPU: the device setup (pd_setup.cu -- generated mesh, element geometry, lumped
masses, body-force bands) is bitwise the host restatement,
which tests/test_oracle_golden.py pins bitwise to the reference's own setup."""
import numpy as np
import pytest

from paper_2403_03605_b200 import capi
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario

pytestmark = pytest.mark.gpu

FIELDS = ["nodes", "conn", "centroid", "volume", "mass", "p_ext", "bc_dofs", "bc_vel"]
SCALARS = ["n_nodes", "n_elems", "delta", "l", "c0", "char_length", "dt", "s_crit", "load_ramp"]


@pytest.mark.parametrize("name", ["mini", "block3d", "cfg1", "bp_coarse", "cfg3", "cfg4"])
def test_device_setup_bitwise_equals_host(name):
    dev = Scenario(cf.get(name))
    host = Scenario(cf.get(name), host_setup=True)
    for f in SCALARS:
        assert getattr(dev, f) == getattr(host, f), f
    for f in FIELDS:
        a, b = getattr(dev, f), getattr(host, f)
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), f


@pytest.mark.parametrize("name", ["mini", "block3d"])
def test_device_geometry_in_handle(name):
    """pmts_pd_create computes centroids / volumes on the device: the deterministic
    families (they depend on every centroid bit) equal the host-setup oracle's."""
    from oracle import pyoracle as po

    sc = Scenario(cf.get(name))
    s = PDSolver.from_scenario(sc, mode=capi.DETERMINISTIC).find_pe_pairs()
    ref = po.find_pairs(sc.dim, sc.centroid, sc.volume, sc.delta, sc.notches())
    assert np.array_equal(s.pairs(), ref)
