"""Crack-tip and crack-path measures for the north-star fast-mode check ("the
crack-tip path lies within one horizon" of the oracle's).  The reference's own
analog is the notch-tip test, proj/tests/test_driver.cpp:296-367 (first break
within 2.5 delta of the notch tip).

A bond is a segment between two element centroids; a broken bond is represented
by its midpoint.  The crack tip of a crack that grows in +x from a left-edge
pre-crack is the broken-bond midpoint of largest x; the crack path is the set
of broken-bond midpoints.
"""
from __future__ import annotations

import numpy as np


def broken_midpoints(pairs: np.ndarray, broken: np.ndarray, centroid: np.ndarray) -> np.ndarray:
    """Midpoints (n, 3) of the bonds whose mask entry is True."""
    b = np.nonzero(broken)[0]
    c = np.asarray(centroid).reshape(-1, 3)
    return 0.5 * (c[pairs[b, 0]] + c[pairs[b, 1]])


def crack_tip(mid: np.ndarray) -> np.ndarray:
    """Tip of a crack growing in +x: the midpoint of largest x (ties: lowest index)."""
    return mid[int(np.argmax(mid[:, 0]))]


def hausdorff(a: np.ndarray, b: np.ndarray) -> float:
    """Symmetric Hausdorff distance of two point sets (inf if exactly one is empty)."""
    if len(a) == 0 and len(b) == 0:
        return 0.0
    if len(a) == 0 or len(b) == 0:
        return float("inf")
    from scipy.spatial import cKDTree

    da, _ = cKDTree(b).query(a)
    db, _ = cKDTree(a).query(b)
    return float(max(da.max(), db.max()))


def agreement(mine: np.ndarray, ref: np.ndarray) -> float:
    """1 - |symmetric difference| / |ref broken| (1.0 when neither broke anything)."""
    n = int(ref.sum())
    if n == 0:
        return 1.0 if not mine.any() else 0.0
    return 1.0 - np.logical_xor(mine, ref).sum() / n
