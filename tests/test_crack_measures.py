"""CPU: the crack-tip / crack-path measures used by the fast-mode parity tests."""
import numpy as np

from crack import agreement, broken_midpoints, crack_tip, hausdorff


def test_crack_measures():
    cen = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]], dtype=float)
    pairs = np.array([[0, 1], [1, 2], [2, 3]], dtype=np.int32)
    a = np.array([True, True, False])
    b = np.array([True, True, True])
    ma, mb = broken_midpoints(pairs, a, cen), broken_midpoints(pairs, b, cen)
    assert np.allclose(ma[:, 0], [0.5, 1.5])
    assert crack_tip(ma)[0] == 1.5 and crack_tip(mb)[0] == 2.5
    assert hausdorff(ma, mb) == 1.0 and hausdorff(ma, ma) == 0.0
    assert agreement(a, b) == 1.0 - 1 / 3
    assert agreement(np.zeros(3, bool), np.zeros(3, bool)) == 1.0
