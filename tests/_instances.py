"""Small deterministic instances shared by oracle pins and GPU parity tests."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def worked_example():
    """SURVEY.md §8.c worked example (tests/golden/worked_example.json)."""
    with open(os.path.join(GOLDEN, "worked_example.json")) as f:
        g = json.load(f)
    X, Y, Z, T = g["grid"]
    C = g["width"]
    mx, my, mz, mt = g["modes"]
    x, y, z, t = np.meshgrid(np.arange(X), np.arange(Y), np.arange(Z), np.arange(T), indexing="ij")
    v = np.zeros((1, C, X, Y, Z, T))
    for c in range(C):
        v[0, c] = ((x + 2 * y + 3 * z + 5 * t + 3 * c) % 7) - 3
    R = np.zeros((C, C, 2 * mx, 2 * my, 2 * mz, mt), dtype=np.complex128)
    for i in range(C):
        for o in range(C):
            for a in range(2 * mx):
                for bb in range(2 * my):
                    for cc in range(2 * mz):
                        for d in range(mt):
                            re = (1 + i + 2 * o + a - bb + cc + d) / 8.0
                            im = (((3 * i + o + 2 * a + bb + cc * d) % 5) - 2) / 8.0
                            R[i, o, a, bb, cc, d] = re + 1j * im
    W = np.array(g["W"], dtype=np.float64)
    b = np.array(g["b"], dtype=np.float64)
    return dict(v=v, R=R, W=W, b=b, modes=(mx, my, mz, mt), grid=(X, Y, Z, T), expected=g["expected"])


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
