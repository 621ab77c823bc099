import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle restatement and libpmts.so (nvcc cross-compiles without a GPU)."""
    from oracle import pyoracle

    pyoracle.build()
    from paper_2403_03605_b200 import _build

    _build.build()


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["meta"] = json.loads(str(d["meta"]))
    d["cfg"] = str(d["cfg"])
    return d


def oracle_sys(g: dict, scenario) -> dict:
    """OraclePD input dict from a golden fixture + the product's scenario setup."""
    m = g["meta"]
    ext = scenario.cfg.get("ext", {})
    sysd = dict(dim=int(m["dim"]), n_nodes=int(m["n_nodes"]), conn=scenario.conn,
                centroid=g["centroid"], volume=g["volume"], pairs=g["pairs"], mass=g["mass"],
                p_ext=g["p_ext"], bc_dofs=scenario.bc_dofs, bc_vel=scenario.bc_vel,
                delta=m["delta"], l=m["l"], c0=m["c0"], s_crit=m["s_crit"], dt=m["dt"],
                gamma=m["gamma"], beta=m["beta"])
    if ext.get("micromodulus") == "constant":
        sysd.update(micromodulus=1, c_const=ext["c"], h=ext.get("h", 1.0))
    if ext.get("s_crit_spread"):
        sysd.update(s_crit_spread=ext["s_crit_spread"], seed=int(ext.get("seed", 0)))
    return sysd


GOLDEN_SCENARIO = {"mini": "mini", "cfg1_200": "cfg1", "block3d": "block3d",
                   "bp_coarse_2000": "bp_coarse"}


def gpu_available() -> bool:
    try:
        import ctypes

        from paper_2403_03605_b200 import capi

        n = ctypes.c_int()
        capi.lib().pmts_device_count(ctypes.byref(n))
        return n.value > 0
    except Exception:
        return False
