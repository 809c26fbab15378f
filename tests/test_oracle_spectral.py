"""Pins of the fp64 oracle (oracle/spectral.py) against things other than itself.

Each test names the pin of DESIGN.md "Oracle pins" (P1-P13) it implements.  None
of them re-calls an oracle helper to produce its expected value: expectations
come from brute-force sums written here, numpy.fft (an independent library),
closed forms, textbook constants, or finite differences.
"""

import math

import numpy as np
import pytest

from oracle import spectral as sp
from tests._instances import rel_l2, worked_example

RNG = np.random.default_rng(1234)


def _rand_problem(B, C, grid, modes, seed=0):
    rng = np.random.default_rng(seed)
    X, Y, Z, T = grid
    mx, my, mz, mt = modes
    v = rng.standard_normal((B, C, X, Y, Z, T))
    R = rng.standard_normal((C, C, 2 * mx, 2 * my, 2 * mz, mt)) + 1j * rng.standard_normal((C, C, 2 * mx, 2 * my, 2 * mz, mt))
    W = rng.standard_normal((C, C))
    b = rng.standard_normal(C)
    return v, R, W, b


def _full_index(n, m):
    return list(range(m)) + list(range(n - m, n))


# ---------------------------------------------------------------- P1 brute force
@pytest.mark.parametrize("grid,modes", [((4, 4, 4, 4), (1, 2, 1, 2)),
                                        ((6, 5, 4, 8), (2, 2, 1, 3)),
                                        ((4, 6, 8, 5), (2, 3, 4, 3))])
def test_p1_forward_equals_brute_force_4d_dft(grid, modes):
    X, Y, Z, T = grid
    v, _, _, _ = _rand_problem(1, 2, grid, modes, seed=1)
    got = sp.forward_modes(v, modes)
    xs = np.stack(np.meshgrid(np.arange(X), np.arange(Y), np.arange(Z), np.arange(T), indexing="ij"), -1)
    kxs, kys, kzs = (_full_index(n, m) for n, m in zip(grid[:3], modes[:3]))
    for c in range(2):
        for a, kx in enumerate(kxs):
            for bq, ky in enumerate(kys):
                for cq, kz in enumerate(kzs):
                    for d in range(modes[3]):
                        ph = 2 * np.pi * (kx * xs[..., 0] / X + ky * xs[..., 1] / Y + kz * xs[..., 2] / Z + d * xs[..., 3] / T)
                        ref = np.sum(v[0, c] * np.exp(-1j * ph))
                        assert abs(got[0, c, a, bq, cq, d] - ref) <= 1e-12 * max(1.0, abs(ref)) * 50


def test_p1_inverse_equals_brute_force_sum():
    grid, modes = (6, 5, 4, 8), (2, 2, 1, 3)
    X, Y, Z, T = grid
    rng = np.random.default_rng(2)
    what = rng.standard_normal((1, 1, 4, 4, 2, 3)) + 1j * rng.standard_normal((1, 1, 4, 4, 2, 3))
    u = sp.inverse_modes(what, grid)
    kxs, kys, kzs = (_full_index(n, m) for n, m in zip(grid[:3], modes[:3]))
    N = X * Y * Z * T
    for (x, y, z, t) in [(0, 0, 0, 0), (5, 4, 3, 7), (2, 1, 3, 5), (3, 2, 0, 1)]:
        s = 0.0
        for a, kx in enumerate(kxs):
            for bq, ky in enumerate(kys):
                for cq, kz in enumerate(kzs):
                    for d in range(3):
                        c = 1.0 if d == 0 else 2.0            # T=8, mt=3: no Nyquist retained
                        s += (c * what[0, 0, a, bq, cq, d] * np.exp(2j * np.pi * (kx * x / X + ky * y / Y + kz * z / Z + d * t / T))).real
        assert abs(u[0, 0, x, y, z, t] - s / N) < 1e-13


# ---------------------------------------------------------------- P2 numpy.fft
def _layer_numpy_fft(v, R, W, b, modes):
    """The same block written with numpy's pocketfft rfftn / irfftn."""
    B, C, X, Y, Z, T = v.shape
    mx, my, mz, mt = modes
    Vf = np.fft.rfftn(v, axes=(2, 3, 4, 5))
    ix, iy, iz = (np.array(_full_index(n, m)) for n, m in zip((X, Y, Z), (mx, my, mz)))
    Vk = Vf[:, :, ix][:, :, :, iy][:, :, :, :, iz][..., :mt]
    Wk = np.einsum("bixyzt,ioxyzt->boxyzt", Vk, R)
    full = np.zeros((B, C, X, Y, Z, T // 2 + 1), dtype=np.complex128)
    full[np.ix_(range(B), range(C), ix, iy, iz, range(mt))] = Wk
    u = np.fft.irfftn(full, s=(X, Y, Z, T), axes=(2, 3, 4, 5))
    z = np.einsum("oi,bixyzt->boxyzt", W, v) + b[None, :, None, None, None, None] + u
    y = 0.5 * z * (1 + np.vectorize(math.erf)(z / math.sqrt(2)))
    return u, z, y


@pytest.mark.parametrize("grid,modes", [((8, 6, 8, 8), (2, 2, 3, 3)),
                                        ((8, 8, 8, 8), (4, 4, 4, 5)),    # full pass incl. Nyquist
                                        ((6, 10, 4, 6), (3, 2, 2, 4)),   # Nyquist kt = 3 retained
                                        ((16, 16, 16, 8), (4, 4, 4, 4))])
def test_p2_layer_matches_numpy_pocketfft(grid, modes):
    v, R, W, b = _rand_problem(2, 3, grid, modes, seed=3)
    u_ref, z_ref, y_ref = _layer_numpy_fft(v, R, W, b, modes)
    u = sp.spectral_conv(v, R, modes)
    y, z = sp.layer_fwd(v, R, W, b, modes)
    assert rel_l2(u, u_ref) < 1e-12
    assert rel_l2(z, z_ref) < 1e-12
    assert rel_l2(y, y_ref) < 1e-12


# ---------------------------------------------------------------- P3 Parseval
@pytest.mark.parametrize("grid", [(4, 6, 8, 8), (6, 4, 4, 7)])
def test_p3_parseval_half_spectrum(grid):
    X, Y, Z, T = grid
    modes = (X // 2, Y // 2, Z // 2, T // 2 + 1)
    v, _, _, _ = _rand_problem(1, 2, grid, modes, seed=4)
    vh = sp.forward_modes(v, modes)
    w = np.full(modes[3], 2.0)
    w[0] = 1.0
    if T % 2 == 0:
        w[T // 2] = 1.0
    lhs = np.sum(v ** 2)
    rhs = np.sum(w * np.abs(vh) ** 2) / (X * Y * Z * T)
    assert abs(lhs - rhs) <= 1e-12 * lhs


# ---------------------------------------------------------------- P4 closed form
@pytest.mark.parametrize("a,r", [((1, 5, 2, 1), 0.7 - 0.4j), ((6, 0, 5, 2), -1.3 + 0.2j), ((0, 1, 0, 3), 2.0j)])
def test_p4_single_cosine_closed_form(a, r):
    """v = cos theta(a, x), R[a] = r, other modes 0  =>  u = |r| cos(theta(a, x) + arg r)."""
    grid, modes = (8, 6, 8, 8), (2, 2, 3, 4)
    X, Y, Z, T = grid
    xs = np.meshgrid(np.arange(X), np.arange(Y), np.arange(Z), np.arange(T), indexing="ij")
    theta = 2 * np.pi * (a[0] * xs[0] / X + a[1] * xs[1] / Y + a[2] * xs[2] / Z + a[3] * xs[3] / T)
    v = np.cos(theta)[None, None]
    R = np.zeros((1, 1, 4, 4, 6, 4), dtype=np.complex128)
    j = [_full_index(n, m).index(k) for n, m, k in zip(grid[:3], modes[:3], a[:3])]
    R[0, 0, j[0], j[1], j[2], a[3]] = r
    u = sp.spectral_conv(v, R, modes)
    ref = abs(r) * np.cos(theta + np.angle(r))
    assert np.max(np.abs(u[0, 0] - ref)) < 1e-12


# ---------------------------------------------------------------- P5 identity = low-pass
def _gain(grid, modes):
    X, Y, Z, T = grid
    mx, my, mz, mt = modes
    inK = lambda j, n, m: (j < m) | (j >= n - m)
    jx, jy, jz, jt = np.meshgrid(np.arange(X), np.arange(Y), np.arange(Z), np.arange(T), indexing="ij")

    def cw(k):
        c = np.where(k == 0, 1.0, 2.0)
        if T % 2 == 0:
            c = np.where(k == T // 2, 1.0, c)
        return c

    def ind(jx, jy, jz, jt):
        return inK(jx, X, mx) & inK(jy, Y, my) & inK(jz, Z, mz) & (jt < mt)

    pos = cw(jt) * ind(jx, jy, jz, jt)
    njt = (-jt) % T
    neg = cw(njt) * ind((-jx) % X, (-jy) % Y, (-jz) % Z, njt)
    return 0.5 * (pos + neg)


@pytest.mark.parametrize("grid,modes", [((8, 6, 8, 8), (2, 2, 3, 3)), ((5, 6, 7, 6), (2, 1, 3, 4)), ((8, 8, 4, 10), (3, 4, 1, 6))])
def test_p5_identity_weights_are_exact_low_pass(grid, modes):
    X, Y, Z, T = grid
    C = 2
    v, _, _, _ = _rand_problem(1, C, grid, modes, seed=5)
    R = np.zeros((C, C, 2 * modes[0], 2 * modes[1], 2 * modes[2], modes[3]), dtype=np.complex128)
    for i in range(C):
        R[i, i] = 1.0
    u = sp.spectral_conv(v, R, modes)
    h = _gain(grid, modes)
    assert set(np.unique(h)).issubset({0.0, 0.5, 1.0})
    ref = np.fft.ifftn(h * np.fft.fftn(v, axes=(2, 3, 4, 5)), axes=(2, 3, 4, 5)).real
    assert rel_l2(u, ref) < 1e-12


def test_p5_boundary_mode_has_half_gain():
    """cos(2 pi m x / X) at kt=0: only -m is retained -> gain 1/2; cos(2 pi (m-1) x/X) -> 1."""
    grid, modes = (8, 4, 4, 4), (3, 2, 2, 2)
    X = grid[0]
    x = np.arange(X)[:, None, None, None] * np.ones(grid)
    R = np.zeros((1, 1, 6, 4, 4, 2), dtype=np.complex128)
    R[0, 0] = 1.0
    for k, gain in ((3, 0.5), (2, 1.0), (4, 0.0)):
        v = np.cos(2 * np.pi * k * x / X)[None, None]
        u = sp.spectral_conv(v, R, modes)
        assert np.max(np.abs(u - gain * v)) < 1e-13


# ---------------------------------------------------------------- P6 full pass
@pytest.mark.parametrize("grid", [(4, 6, 8, 8), (6, 4, 2, 10)])
def test_p6_full_pass_is_identity(grid):
    X, Y, Z, T = grid
    modes = (X // 2, Y // 2, Z // 2, T // 2 + 1)
    v, _, _, _ = _rand_problem(1, 2, grid, modes, seed=6)
    R = np.zeros((2, 2, X, Y, Z, modes[3]), dtype=np.complex128)
    R[0, 0] = R[1, 1] = 1.0
    assert rel_l2(sp.spectral_conv(v, R, modes), v) < 1e-12


def test_p6_mt_equal_half_T_is_not_full_pass():
    """Reading Q19: under the real FFT, mt = T/2 drops the Nyquist plane."""
    grid = (4, 4, 4, 8)
    v, _, _, _ = _rand_problem(1, 1, grid, (2, 2, 2, 4), seed=7)
    R = np.ones((1, 1, 4, 4, 4, 4), dtype=np.complex128)
    assert rel_l2(sp.spectral_conv(v, R, (2, 2, 2, 4)), v) > 0.05


# ---------------------------------------------------------------- P7 trivial
def test_p7_zero_weights():
    grid, modes = (8, 6, 8, 8), (2, 2, 3, 3)
    v, R, W, b = _rand_problem(1, 2, grid, modes, seed=8)
    assert np.max(np.abs(sp.spectral_conv(v, 0 * R, modes))) == 0.0
    y, z = sp.layer_fwd(v, 0 * R, 0 * W, 0 * b, modes)
    assert np.max(np.abs(y)) == 0.0


# ---------------------------------------------------------------- P8 linearity, shift
def test_p8_linearity_and_shift_equivariance():
    grid, modes = (8, 6, 8, 8), (2, 2, 3, 3)
    v, R, _, _ = _rand_problem(1, 2, grid, modes, seed=9)
    w, _, _, _ = _rand_problem(1, 2, grid, modes, seed=10)
    S = lambda a: sp.spectral_conv(a, R, modes)
    assert rel_l2(S(2.5 * v - 0.75 * w), 2.5 * S(v) - 0.75 * S(w)) < 1e-12
    for axis, s in ((2, 3), (3, 1), (4, 5), (5, 2)):
        assert rel_l2(S(np.roll(v, s, axis=axis)), np.roll(S(v), s, axis=axis)) < 1e-12


# ---------------------------------------------------------------- P9 adjoint
@pytest.mark.parametrize("grid,modes", [((8, 6, 8, 8), (2, 2, 3, 3)), ((6, 6, 6, 6), (3, 3, 3, 4)), ((4, 4, 4, 4), (1, 2, 1, 2))])
def test_p9_adjoint_identity(grid, modes):
    v, R, _, _ = _rand_problem(2, 3, grid, modes, seed=11)
    g, _, _, _ = _rand_problem(2, 3, grid, modes, seed=12)
    Sv = sp.spectral_conv(v, R, modes)
    STg = sp.spectral_conv_adjoint(g, R, modes)
    lhs = np.sum(Sv * g)
    rhs = np.sum(v * STg)
    assert abs(lhs - rhs) / (np.linalg.norm(Sv) * np.linalg.norm(g)) < 1e-12


# ---------------------------------------------------------------- P10 bilinear dR
def test_p10_bilinear_identity_for_dR():
    grid, modes = (8, 6, 8, 8), (2, 2, 3, 3)
    v, R, W, b = _rand_problem(2, 3, grid, modes, seed=13)
    g, Rp, _, _ = _rand_problem(2, 3, grid, modes, seed=14)
    _, dR, _, _ = sp.layer_bwd(v, g, R, W, b, modes, act="none")
    lhs = np.sum(g * sp.spectral_conv(v, Rp, modes))
    rhs = np.sum((np.conj(dR) * Rp).real)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs) * 10


# ---------------------------------------------------------------- P11 finite differences
def test_p11_finite_differences_through_gelu():
    grid, modes = (4, 6, 4, 6), (2, 2, 1, 3)
    v, R, W, b = _rand_problem(1, 2, grid, modes, seed=15)
    R = 0.3 * R
    dy, _, _, _ = _rand_problem(1, 2, grid, modes, seed=16)
    dv, dR, dW, db = sp.layer_bwd(v, dy, R, W, b, modes)
    L = lambda v_, R_, W_, b_: np.sum(dy * sp.layer_fwd(v_, R_, W_, b_, modes)[0])
    eps = 1e-6
    rng = np.random.default_rng(17)
    for _ in range(4):
        idx = tuple(rng.integers(0, s) for s in v.shape)
        e = np.zeros_like(v); e[idx] = eps
        fd = (L(v + e, R, W, b) - L(v - e, R, W, b)) / (2 * eps)
        assert abs(fd - dv[idx]) <= 1e-6 * max(1.0, abs(fd))
    for (o, i) in [(0, 1), (1, 1)]:
        e = np.zeros_like(W); e[o, i] = eps
        fd = (L(v, R, W + e, b) - L(v, R, W - e, b)) / (2 * eps)
        assert abs(fd - dW[o, i]) <= 1e-6 * max(1.0, abs(fd))
    e = np.zeros_like(b); e[1] = eps
    fd = (L(v, R, W, b + e) - L(v, R, W, b - e)) / (2 * eps)
    assert abs(fd - db[1]) <= 1e-6 * max(1.0, abs(fd))
    for _ in range(3):
        idx = tuple(rng.integers(0, s) for s in R.shape)
        e = np.zeros_like(R); e[idx] = eps
        fre = (L(v, R + e, W, b) - L(v, R - e, W, b)) / (2 * eps)
        fim = (L(v, R + 1j * e, W, b) - L(v, R - 1j * e, W, b)) / (2 * eps)
        assert abs(fre - dR[idx].real) <= 1e-6 * max(1.0, abs(fre))
        assert abs(fim - dR[idx].imag) <= 1e-6 * max(1.0, abs(fim))


# ---------------------------------------------------------------- P12 GELU
def test_p12_gelu_textbook_values_and_derivative():
    # Phi(1) = 0.8413447460685429 (standard normal CDF table value)
    assert abs(sp.gelu(np.array(1.0)) - 0.8413447460685429) < 1e-15
    assert abs(sp.gelu(np.array(-1.0)) + 0.15865525393145707) < 1e-15
    assert sp.gelu(np.array(0.0)) == 0.0
    z = np.linspace(-5, 5, 41)
    h = 1e-6
    fd = (sp.gelu(z + h) - sp.gelu(z - h)) / (2 * h)
    assert np.max(np.abs(fd - sp.gelu_prime(z))) < 1e-8


# ---------------------------------------------------------------- golden worked example
def test_golden_worked_example():
    ex = worked_example()
    u = sp.spectral_conv(ex["v"], ex["R"], ex["modes"])[0]
    y, _ = sp.layer_fwd(ex["v"], ex["R"], ex["W"], ex["b"], ex["modes"])
    y = y[0]
    e = ex["expected"]
    assert abs(u.sum() - e["sum_u"]) < 1e-12
    assert abs((u ** 2).sum() - e["sum_u2"]) < 1e-11
    assert abs(u[0, 0, 0, 0, 0] - e["u[0,0,0,0,0]"]) < 1e-13
    assert abs(u[1, 1, 2, 3, 1] - e["u[1,1,2,3,1]"]) < 1e-13
    assert abs(y.sum() - e["sum_y"]) < 1e-11
    assert abs(y[1, 3, 0, 2, 2] - e["y[1,3,0,2,2]"]) < 1e-13


def test_sampled_inverse_matches_full_inverse():
    grid, modes = (8, 6, 8, 8), (2, 2, 3, 3)
    rng = np.random.default_rng(18)
    what = rng.standard_normal((2, 3, 4, 4, 6, 3)) + 1j * rng.standard_normal((2, 3, 4, 4, 6, 3))
    u = sp.inverse_modes(what, grid)
    pts = np.stack([rng.integers(0, n, size=17) for n in grid], -1)
    us = sp.inverse_modes_at(what, grid, pts)
    ref = u[:, :, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    assert rel_l2(us, ref) < 1e-13
