"""fp64 oracle: the 4D spectral convolution, the DFNO block and their gradients.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy float64 /
complex128.  Every transform is an explicit DFT-matrix product; no FFT.

Notation:
  field v[b, c, x, y, z, t], NCXYZT, t fastest ............. P:182
  retained modes per spatial axis  K_d = {0..m-1} ∪ {n-m..n-1}   P:52 ("how
      many Fourier-modes to keep in each dimension"); reading Q2
  retained modes along t           K_t = {0..mt-1} (half spectrum of the real
      FFT along t); readings Q1, Q2
  retained index j in [0, 2m) -> global k = j if j < m else n - 2m + j
  theta(k, x) = 2*pi*(kx x/X + ky y/Y + kz z/Z + kt t/T)
  c(kt) = 1 if kt == 0 or (T even and kt == T/2) else 2        reading Q4
  N = X*Y*Z*T

Parity status: every public function here is pinned by tests/test_oracle_*.py
(brute force DFT, numpy.fft cross-check, Parseval, closed forms, identity
low-pass filter, full pass, adjoint, bilinear dR identity, finite differences).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf as _erf

__all__ = [
    "retained", "retained_t", "dft_rows", "c_weight", "check_modes",
    "forward_modes", "mix", "inverse_modes", "inverse_modes_at",
    "spectral_conv", "spectral_conv_adjoint", "gelu", "gelu_prime",
    "layer_fwd", "layer_bwd",
]


# ---------------------------------------------------------------------------
# retained sets (reading Q2) and the DFT matrices ("F")
# ---------------------------------------------------------------------------

def retained(n: int, m: int) -> np.ndarray:
    """Retained global indices along a spatial axis: {0..m-1} ∪ {n-m..n-1}.

    P:52: "the cutoff ... how many Fourier-modes to keep in each dimension";
    P:144 "R_phi is sparse, containing nonzero elements only in the
    low-frequency modes".  Reading Q2 (positive and negative low modes, 2m<=n).
    Retained index j -> k = j (j < m) else n - 2m + j.
    """
    if not (1 <= m and 2 * m <= n):
        raise ValueError(f"spatial modes need 1 <= m and 2m <= n (n={n}, m={m})")
    return np.concatenate([np.arange(m), np.arange(n - m, n)]).astype(np.int64)


def retained_t(T: int, mt: int) -> np.ndarray:
    """Retained indices along t for the real FFT: {0..mt-1}, mt <= T//2+1 (Q1, Q2)."""
    if not (1 <= mt <= T // 2 + 1):
        raise ValueError(f"time modes need 1 <= mt <= T//2+1 (T={T}, mt={mt})")
    return np.arange(mt, dtype=np.int64)


def dft_rows(n: int, ks: np.ndarray, sign: int) -> np.ndarray:
    """Rows k of the n-point DFT matrix: F[j, x] = exp(sign*2*pi*i*((k_j*x) mod n)/n).

    The integer product is reduced mod n before the angle is formed, so the
    fp64 phase error stays ~1e-16 for any n.  sign=-1: forward ("F nu");
    sign=+1: inverse (unnormalised; 1/N is applied once, reading Q3).
    """
    x = np.arange(n, dtype=np.int64)
    r = np.outer(np.asarray(ks, dtype=np.int64), x) % n
    return np.exp(sign * 2j * np.pi * r / n)


def c_weight(T: int, mt: int) -> np.ndarray:
    """c(kt) for kt in K_t: 1 at kt=0 and at the Nyquist kt=T/2 (T even), else 2.

    This is the half-spectrum weight of the real inverse transform with
    real-part semantics (reading Q4): the full spectrum of a real field holds
    both kt and -kt; storing only kt >= 0 counts the kt > 0 terms twice.
    """
    kt = retained_t(T, mt)
    c = np.full(kt.shape, 2.0)
    c[kt == 0] = 1.0
    if T % 2 == 0:
        c[kt == T // 2] = 1.0
    return c


def check_modes(grid, modes):
    X, Y, Z, T = (int(g) for g in grid)
    mx, my, mz, mt = (int(m) for m in modes)
    return retained(X, mx), retained(Y, my), retained(Z, mz), retained_t(T, mt)


def _apply(a: np.ndarray, F: np.ndarray, axis: int) -> np.ndarray:
    """out[..., j, ...] = sum_x F[j, x] * a[..., x, ...] along `axis`."""
    out = np.tensordot(a, F, axes=([axis], [1]))  # contracted axis -> last
    return np.moveaxis(out, -1, axis)


# ---------------------------------------------------------------------------
# S(v) = F^-1 (R_phi . F v)      P:48-52 (Eq. 3), distributed form P:119-123
# ---------------------------------------------------------------------------

def forward_modes(v: np.ndarray, modes) -> np.ndarray:
    """V̂[b, c, jx, jy, jz, jt] = sum_x v[b,c,x] exp(-i theta(k_j, x)), k_j in K.

    v: real [B, C, X, Y, Z, T].  Separable order t, z, y, x ("first
    taking an FFT along time, ... followed by a 2D FFT along the x and y
    dimensions"; reading Q10), each axis restricted to its retained rows
    (the low-pass mask of R_phi applied as a row selector).
    """
    v = np.asarray(v, dtype=np.float64)
    B, C, X, Y, Z, T = v.shape
    kx, ky, kz, kt = check_modes((X, Y, Z, T), modes)
    a = _apply(v.astype(np.complex128), dft_rows(T, kt, -1), 5)
    a = _apply(a, dft_rows(Z, kz, -1), 4)
    a = _apply(a, dft_rows(Y, ky, -1), 3)
    a = _apply(a, dft_rows(X, kx, -1), 2)
    return a


def mix(vhat: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Ŵ[b, o, k] = sum_i V̂[b, i, k] R[i, o, k] for every retained k.

    "R_phi . (F nu)": per-mode complex channel mixing with the learned
    weights.  R layout [C_in, C_out, 2mx, 2my, 2mz, mt] (reading Q5).
    """
    return np.einsum("bixyzt,ioxyzt->boxyzt", vhat, R)


def inverse_modes(what: np.ndarray, grid) -> np.ndarray:
    """u[b, o, x] = (1/N) Re sum_{k in K} c(kt) Ŵ[b, o, k] exp(+i theta(k, x)).

    "F^-1" of P:50 / "F_dist^T" of P:121 with the real inverse FFT along t
    (C2R, real-part semantics, readings Q1, Q4); zero-padding of the
    non-retained modes is implicit (they contribute nothing).
    """
    X, Y, Z, T = (int(g) for g in grid)
    B, C, nx, ny, nz, nt = what.shape
    mx, my, mz, mt = nx // 2, ny // 2, nz // 2, nt
    kx, ky, kz, kt = check_modes((X, Y, Z, T), (mx, my, mz, mt))
    a = _apply(what, dft_rows(X, kx, +1).T, 2)
    a = _apply(a, dft_rows(Y, ky, +1).T, 3)
    a = _apply(a, dft_rows(Z, kz, +1).T, 4)
    a = a * c_weight(T, mt)
    u = _apply(a, dft_rows(T, kt, +1).T, 5).real
    return u / float(X * Y * Z * T)


def inverse_modes_at(what: np.ndarray, grid, points: np.ndarray) -> np.ndarray:
    """inverse_modes evaluated only at `points` (int array [P, 4] of x,y,z,t).

    Returns u[b, o, p].  Same formula as inverse_modes, written as the direct
    sum over all retained modes for each requested point (for full-size
    configurations whose whole output the oracle cannot afford).
    """
    X, Y, Z, T = (int(g) for g in grid)
    B, C, nx, ny, nz, nt = what.shape
    kx, ky, kz, kt = check_modes((X, Y, Z, T), (nx // 2, ny // 2, nz // 2, nt))
    pts = np.asarray(points, dtype=np.int64)
    ex = np.exp(2j * np.pi * (np.outer(pts[:, 0], kx) % X) / X)   # [P, 2mx]
    ey = np.exp(2j * np.pi * (np.outer(pts[:, 1], ky) % Y) / Y)
    ez = np.exp(2j * np.pi * (np.outer(pts[:, 2], kz) % Z) / Z)
    et = np.exp(2j * np.pi * (np.outer(pts[:, 3], kt) % T) / T) * c_weight(T, nt)
    s = np.einsum("boxyzt,px,py,pz,pt->bop", what, ex, ey, ez, et, optimize=True)
    return s.real / float(X * Y * Z * T)


def spectral_conv(v: np.ndarray, R: np.ndarray, modes) -> np.ndarray:
    """S v = F^-1 (R_phi . F v) (Eq. 3; P:121 Eq. sconv_dist)."""
    B, C, X, Y, Z, T = v.shape
    return inverse_modes(mix(forward_modes(v, modes), R), (X, Y, Z, T))


def spectral_conv_adjoint(g: np.ndarray, R: np.ndarray, modes) -> np.ndarray:
    """S^T g under the real inner product: S with R^H[i, o, k] := conj(R[o, i, k]).

    The adjoint of each linear primitive is what reverse-mode AD replays
    ("its adjoint is also a repartitioning"); for S the
    derivation is in DESIGN.md (Backward).  Pinned by the adjoint test P9.
    """
    RH = np.conj(np.swapaxes(R, 0, 1))
    return spectral_conv(g, RH, modes)


# ---------------------------------------------------------------------------
# DFNO block  nu_{k+1} = sigma(W nu_k + S nu_k)     P:161, P:166 (Eq. dist_block)
# ---------------------------------------------------------------------------

def gelu(z: np.ndarray) -> np.ndarray:
    """sigma = GELU, exact erf form: z * Phi(z) = 0.5 z (1 + erf(z / sqrt 2)) (reading Q6)."""
    return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))


def gelu_prime(z: np.ndarray) -> np.ndarray:
    """d/dz GELU = Phi(z) + z phi(z)."""
    return 0.5 * (1.0 + _erf(z / math.sqrt(2.0))) + z * np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)


def _channel_linear(W: np.ndarray, v: np.ndarray) -> np.ndarray:
    """(W v)[b, o, x] = sum_i W[o, i] v[b, i, x]: the pointwise affine "W x" along
    the (undistributed) channel dimension, P:88-93 (Eq. affine, affine_bcast)."""
    return np.einsum("oi,bixyzt->boxyzt", W, v)


def layer_fwd(v, R, W, b, modes, act: str = "gelu"):
    """One DFNO block.  Returns (y, z) with z = W v + b + S v, y = sigma(z).

    P:166 (Eq. dist_block); bias optional (reading Q7, b=None means 0);
    act in {"gelu", "none"} (reading Q6).
    """
    v = np.asarray(v, dtype=np.float64)
    z = _channel_linear(np.asarray(W, np.float64), v) + spectral_conv(v, R, modes)
    if b is not None:
        z = z + np.asarray(b, np.float64)[None, :, None, None, None, None]
    y = gelu(z) if act == "gelu" else z.copy()
    return y, z


def layer_bwd(v, dy, R, W, b, modes, act: str = "gelu"):
    """Gradients of <dy, layer_fwd(v)> w.r.t. v, R, W, b.  Returns (dv, dR, dW, db).

      dz = dy * sigma'(z)
      dv = W^T dz + S^T dz                      (S^T as above)
      dW[o, i] = sum_{b,x} dz[b,o,x] v[b,i,x]   (broadcast adjoint = sum)
      db[o]    = sum_{b,x} dz[b,o,x]
      dR[i, o, k] = (c(kt)/N) sum_b conj(V̂[b,i,k]) Ĝ[b,o,k],  Ĝ = F dz on K
    Complex gradient convention dL/dRe + i dL/dIm (reading Q16).
    """
    v = np.asarray(v, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    W = np.asarray(W, np.float64)
    _, z = layer_fwd(v, R, W, b, modes, act)
    dz = dy * gelu_prime(z) if act == "gelu" else dy
    B, C, X, Y, Z, T = v.shape
    N = float(X * Y * Z * T)
    dW = np.einsum("boxyzt,bixyzt->oi", dz, v)
    db = dz.sum(axis=(0, 2, 3, 4, 5))
    vh = forward_modes(v, modes)
    gh = forward_modes(dz, modes)
    c = c_weight(T, modes[3])
    dR = np.einsum("bixyzt,boxyzt->ioxyzt", np.conj(vh), gh) * (c / N)
    dv = np.einsum("oi,boxyzt->bixyzt", W, dz) + spectral_conv_adjoint(dz, R, modes)
    return dv, dR, dW, db
