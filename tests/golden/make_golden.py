"""Generate the golden vectors under tests/golden/ from the reference itself.

Runs oracle/_ref/ref_driver -- the reference's own pure-PD loop, compiled in
place from /root/reference/proj/include (see oracle/Makefile) -- on the
scenarios below and stores its inputs and outputs as compressed npz files.
The reference publishes no full-run goldens; these are the
fixtures 1-3 of that section plus a 3D hex8 block.  Re-run with:

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from paper_2403_03605_b200 import configs as cf  # noqa: E402

# coupled MTS fixtures (oracle/_ref/ref_mts_driver): name -> (scenario, macro steps, checkpoints)
MTS_FIXTURES = {
    "mts_mini": ("mts_mini", 40, (10,)),
    "mts_mini_implicit": ("mts_mini_implicit", 20, (5,)),
    "mts_mini_frac": ("mts_mini_frac", 60, (30,)),
    "mts_mini_mfree": ("mts_mini_mfree", 20, (5,)),
    "mts_bar3d": ("mts_bar3d", 15, (5,)),
}

# name -> (scenario, steps, checkpoints)
FIXTURES = {
    "mini": ("mini", 80, (40,)),
    "cfg1_200": ("cfg1", 200, (50,)),
    "block3d": ("block3d", 100, (50,)),
    "bp_coarse_2000": ("bp_coarse", 2000, ()),
}


def main(names=None):
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, (scen, steps, ck) in FIXTURES.items():
        if names and name not in names:
            continue
        sc = cf.get(scen)
        text = cf.render_cfg(sc)
        with tempfile.TemporaryDirectory() as tmp:
            run = po.run_ref(text, tmp, steps=steps, checkpoints=ck)
            d = po.load_ref_dump(tmp)
        arrays = {k: d[k] for k in ("centroid", "volume", "pairs", "mass", "p_ext", "a0",
                                    "scale", "u", "v", "a", "damage_elem", "damage_node",
                                    "xi_norm", "weight")}
        arrays["broken"] = d["broken"] if d["broken"] is not None else np.zeros((0, 2), np.int32)
        for k in ck:
            for f in ("u", "v", "a"):
                arrays[f"{f}_{k}"] = d[f"{f}_{k}"]
        meta = {k: d[k] for k in ("dim", "n_nodes", "n_elems", "n_pairs", "n_dof", "n_steps",
                                  "delta", "l", "c0", "s_crit", "dt", "gamma", "beta", "rho",
                                  "char_length", "nnz")}
        meta.update(scenario=scen, steps=steps, checkpoints=list(ck), run=run,
                    sha256_u=hashlib.sha256(d["u"].tobytes()).hexdigest())
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), cfg=np.array(text),
                            meta=np.array(json.dumps(meta)), **arrays)
        print(name, run)


def main_mts(names=None):
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, (scen, steps, ck) in MTS_FIXTURES.items():
        if names and name not in names:
            continue
        text = cf.render_cfg(cf.get(scen))
        with tempfile.TemporaryDirectory() as tmp:
            run = po.run_ref_mts(text, tmp, steps=steps, checkpoints=ck)
            d = po.load_ref_mts_dump(tmp)
        arrays = {k: v for k, v in d.items() if isinstance(v, np.ndarray)}
        meta = {k: v for k, v in d.items() if not isinstance(v, np.ndarray)}
        meta.update(scenario=scen, steps=steps, checkpoints=list(ck), run=run)
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), cfg=np.array(text),
                            meta=np.array(json.dumps(meta)), **arrays)
        print(name, run)


# system arrays of the full-size coupled fixture kept as sha256 only (tens of MB otherwise)
FULL_HASHED = ("fe_k_val", "fe_mass", "fe_p_ext", "pd_mass", "pd_p_ext", "fe_dof", "pd_dof",
               "pairs", "pe_weight")


def main_mts_full(steps=3):
    """BASELINE cfg2's conforming analog at full size (0.25 mm, n_lambda = 14,436) through
    the reference's own coupled loop (~10 minutes of reference setup): end states, the
    multipliers and the interface iteration counts, the assembled systems as sha256."""
    out_dir = os.path.dirname(os.path.abspath(__file__))
    text = cf.render_cfg(cf.get("cfg2"))
    with tempfile.TemporaryDirectory() as tmp:
        run = po.run_ref_mts(text, tmp, steps=steps)
        d = po.load_ref_mts_dump(tmp)
    arrays = {k: d[k] for k in ("fe_u", "fe_v", "pd_u", "pd_v", "lambda", "iterations")}
    meta = {k: v for k, v in d.items() if not isinstance(v, np.ndarray)}
    meta.update(scenario="cfg2", steps=steps, run=run,
                sha256={k: hashlib.sha256(np.ascontiguousarray(d[k]).tobytes()).hexdigest()
                        for k in FULL_HASHED})
    np.savez_compressed(os.path.join(out_dir, "mts_cfg2_full.npz"), cfg=np.array(text),
                        meta=np.array(json.dumps(meta)), **arrays)
    print("mts_cfg2_full", run)


if __name__ == "__main__":
    if sys.argv[1:] == ["mts_cfg2_full"]:
        main_mts_full()
        sys.exit(0)
    main([a for a in sys.argv[1:] if not a.startswith("mts")] or None)
    main_mts([a for a in sys.argv[1:] if a.startswith("mts")] or None)
