"""Pins of the network oracle (oracle/network.py) against things
other than itself: special cases with known results, closed forms of the loss
and of Adam, and central finite differences of the whole network's loss."""

import numpy as np
import pytest

from oracle import network as nw


def _params(Cin, C, T, K, modes, seed=0, bias_p=True):
    rng = np.random.default_rng(seed)
    mx, my, mz, mt = modes
    shp = (C, C, 2 * mx, 2 * my, 2 * mz, mt)
    return {
        "Wt": rng.standard_normal((T, 1)), "bt": rng.standard_normal(T),
        "Wc": rng.standard_normal((C, Cin)) / np.sqrt(Cin), "bc": rng.standard_normal(C) * 0.1,
        "R": [(rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / C for _ in range(K)],
        "W": [rng.standard_normal((C, C)) / np.sqrt(C) for _ in range(K)],
        "b": [rng.standard_normal(C) * 0.1 for _ in range(K)],
        "Wp": rng.standard_normal((1, C)) / np.sqrt(C), "bp": rng.standard_normal(1) * 0.1 if bias_p else None,
    }


def test_lift_special_cases():
    """Wt = 1, bt = 0, Wc = I, bc = 0: nu_0 is the input repeated along t;
    a constant input c gives Wc (Wt c + bt) + bc, worked by hand below."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((1, 2, 3, 2, 2, 1))
    T = 5
    nu0 = nw.lift(a, np.ones((T, 1)), np.zeros(T), np.eye(2), np.zeros(2))
    assert nu0.shape == (1, 2, 3, 2, 2, T)
    for t in range(T):
        assert np.array_equal(nu0[..., t], a[..., 0])
    # a = (1, 2) everywhere, Wt = (1, 2)^T, bt = (0, 1), Wc = [[1, 1], [2, -1]], bc = (3, 0):
    # a1 = (1, 2) at t=0 and (3, 5) at t=1 ->
    # nu0[0] = (1 + 2, 3 + 5) + 3 = (6, 11);  nu0[1] = (2 - 2, 6 - 5) + 0 = (0, 1)
    a = np.stack([np.ones((1, 1, 1)), 2 * np.ones((1, 1, 1))])[None][..., None]
    nu0 = nw.lift(a, np.array([[1.0], [2.0]]), np.array([0.0, 1.0]), np.array([[1.0, 1.0], [2.0, -1.0]]),
                  np.array([3.0, 0.0]))
    assert np.allclose(nu0[0, :, 0, 0, 0, :], [[6.0, 11.0], [0.0, 1.0]], rtol=0, atol=1e-14)


def test_project_special_cases():
    rng = np.random.default_rng(2)
    nu = rng.standard_normal((2, 4, 2, 3, 2, 3))
    for j in range(4):
        e = np.zeros((1, 4)); e[0, j] = 1.0
        assert np.array_equal(nw.project(nu, e)[:, 0], nu[:, j])
    u0 = nw.project(nu, rng.standard_normal((1, 4)))
    u1 = nw.project(nu, np.zeros((1, 4)) + 0.0, np.array([2.5]))
    assert np.all(u1 == 2.5) and u0.shape == (2, 1, 2, 3, 2, 3)


def test_rel_l2_closed_forms():
    y = np.random.default_rng(3).standard_normal((1, 1, 3, 2, 2, 4))
    assert nw.rel_l2(y, y) == 0.0
    assert abs(nw.rel_l2(np.zeros_like(y), y) - 1.0) < 1e-15
    assert abs(nw.rel_l2(2 * y, y) - 1.0) < 1e-15
    u = y + 0.3 * np.cos(np.arange(y.size)).reshape(y.shape)
    assert abs(nw.rel_l2(7.5 * u, 7.5 * y) - nw.rel_l2(u, y)) < 1e-14          # scale invariance
    assert abs(nw.rel_l2(np.array([3.0, 9.0]), np.array([0.0, 5.0])) - 1.0) < 1e-15   # ||(3,4)|| / 5


def test_adam_closed_forms():
    """Constant gradient: bias correction makes m^ = g and v^ = g^2 at every step,
    so p_n = p_0 - n lr g / (|g| + eps) exactly (Kingma & Ba, Alg. 1)."""
    p0 = np.array([1.0, -2.0, 0.5])
    g = np.array([0.3, -4.0, 1e-3])
    p, m, v = p0.copy(), np.zeros(3), np.zeros(3)
    for n in range(1, 6):
        p, m, v = nw.adam_step(p, g, m, v, n, lr=1e-2)
        assert np.allclose(p, p0 - n * 1e-2 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-13)
    # complex: real and imaginary parts are independent real problems
    pc, mc, vc = nw.adam_step(np.array([1 + 2j]), np.array([0.5 - 0.25j]), np.zeros(1, complex), np.zeros(1, complex), 1)
    pr, _, _ = nw.adam_step(np.array([1.0]), np.array([0.5]), np.zeros(1), np.zeros(1), 1)
    pi, _, _ = nw.adam_step(np.array([2.0]), np.array([-0.25]), np.zeros(1), np.zeros(1), 1)
    assert pc[0] == pr[0] + 1j * pi[0]


@pytest.mark.parametrize("bias_p", [True, False])
def test_network_gradients_match_finite_differences(bias_p):
    """Central differences of the whole network's relative-L2 loss (lift, two
    blocks -- the last without sigma -- projection) against network_bwd."""
    grid, modes, Cin, C, K = (6, 4, 4, 4), (2, 1, 1, 2), 2, 3, 2
    X, Y, Z, T = grid
    rng = np.random.default_rng(5)
    a = rng.standard_normal((1, Cin, X, Y, Z, 1))
    y = rng.standard_normal((1, 1, X, Y, Z, T))
    P = _params(Cin, C, T, K, modes, seed=6, bias_p=bias_p)
    loss, g = nw.network_bwd(a, y, P, modes)
    assert abs(loss - nw.rel_l2(nw.network_fwd(a, P, modes)[0], y)) < 1e-14
    eps = 1e-6

    def L(P2):
        return nw.rel_l2(nw.network_fwd(a, P2, modes)[0], y)

    def check(key, idx, k=None, imag=False):
        def get(P2):
            return P2[key][k] if k is not None else P2[key]
        Pp = {kk: ([x.copy() for x in vv] if isinstance(vv, list) else (None if vv is None else vv.copy()))
              for kk, vv in P.items()}
        Pm = {kk: ([x.copy() for x in vv] if isinstance(vv, list) else (None if vv is None else vv.copy()))
              for kk, vv in P.items()}
        h = 1j * eps if imag else eps
        get(Pp)[idx] += h
        get(Pm)[idx] -= h
        fd = (L(Pp) - L(Pm)) / (2 * eps)
        gg = (g[key][k] if k is not None else g[key])[idx]
        an = gg.imag if imag else gg.real
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (key, idx, k, imag, fd, an)

    check("Wt", (2, 0)); check("bt", (1,)); check("Wc", (1, 0)); check("bc", (2,))
    check("Wp", (0, 1))
    if bias_p:
        check("bp", (0,))
    for k in range(K):
        check("W", (0, 2), k); check("b", (1,), k)
        check("R", (1, 0, 1, 0, 1, 1), k); check("R", (2, 2, 0, 1, 0, 0), k, imag=True)
