"""The C-ABI library: loads, exports exactly what include/pmts_capi.h declares,
and fails loudly (no CPU fallback) when there is no device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, gpu_available
from paper_2403_03605_b200 import capi

HEADER = os.path.join(ROOT, "include", "pmts_capi.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(pmts_[a-z_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_symbols() == set(capi.SIGNATURES)


def test_library_exports_every_symbol():
    L = capi.lib()
    for name in header_symbols():
        assert hasattr(L, name), name


def test_abi_version_and_error_string():
    L = capi.lib()
    assert L.pmts_abi_version() == capi.ABI_VERSION == 2
    assert isinstance(L.pmts_last_error(), bytes)


def test_sm100a_cubin_embedded():
    """The .so carries sm_100a SASS (tcgen05-era target), no PTX-only fallback."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-device path")
def test_create_without_device_fails_loudly():
    d = capi.PDDesc()
    nodes = np.zeros((4, 3))
    conn = np.array([[0, 1, 2, 3]], np.int32)
    m = np.ones(8)
    d.dim, d.n_nodes, d.n_elems = 2, 4, 1
    d.node_xyz, d.elem_nodes, d.mass, d.p_ext = capi.ptr(nodes), capi.ptr(conn), capi.ptr(m), capi.ptr(m)
    d.delta, d.c0, d.l, d.dt = 1.0, 1.0, 0.5, 1e-3
    h = C.c_void_p()
    st = capi.lib().pmts_pd_create(C.byref(d), C.byref(h))
    assert st == capi.PMTS_ERR_INTERNAL
    assert b"no CUDA device" in capi.lib().pmts_last_error()


def test_config_errors_map_to_status_2():
    d = capi.PDDesc()
    d.dim = 5
    h = C.c_void_p()
    assert capi.lib().pmts_pd_create(C.byref(d), C.byref(h)) == capi.PMTS_ERR_CONFIG
    with pytest.raises(capi.ConfigError):
        capi.check(capi.lib().pmts_pd_create(C.byref(d), C.byref(h)))


def test_scenario_config_errors():
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.pd import Scenario

    sc = cf.get("mini")
    sc["mesh"]["spacing"] = 0.0013  # not a divisor of the extent (mesh.hpp:181-183)
    with pytest.raises(capi.ConfigError):
        Scenario(sc)


def test_mode_enum_matches_binding():
    """enum pmts_mode of the header (deterministic, fast, fp32-position variant) and
    the Python constants agree."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    vals = dict((k, int(v)) for k, v in re.findall(r"\b(PMTS_(?:DETERMINISTIC|FAST|FAST_F32POS))\s*=\s*(\d+)", text))
    assert vals == {"PMTS_DETERMINISTIC": capi.DETERMINISTIC, "PMTS_FAST": capi.FAST,
                    "PMTS_FAST_F32POS": capi.FAST_F32POS}
