"""fp64 oracle of the whole DFNO network: lift, K blocks,
projection, relative-L2 loss, their gradients, and one Adam step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy float64.

Network (PAPER.md §"Full Network"):
  a1(x, t)  = (W_t a + b_t)(x, t)      time affine on an input with T = 1
  nu_0      = (W_c a1 + b_c)(x, t)     channel affine C_in -> C              P:140, P:156-157 (Eq. lift)
  nu_{k+1}  = sigma(W nu_k + S nu_k)   k = 0..K-1, DFNO block
  u         = W_p nu_K (+ b_p)         projection C -> 1
  L(u, y)   = ||u - y||_2 / ||y||_2    relative L2 misfit (p = 2)
Readings: N1a  W_t is [T, 1] and b_t [T] (a has a time axis of
size 1); N1b no sigma after the last block, as in the original FNO the
paper says it is identical to (Li et al.); N1c the projection bias is
optional (the paper writes none); N1d Adam as in Kingma & Ba (P:187,
lr 1e-3, beta1 0.9, beta2 0.999, eps 1e-8) with bias correction, applied to the
real and imaginary parts of R independently.
"""

from __future__ import annotations

import numpy as np

from . import spectral as sp

__all__ = ["lift", "project", "rel_l2", "network_fwd", "network_bwd", "adam_step"]


def lift(a, Wt, bt, Wc, bc):
    """nu_0[b, o, x, y, z, t] = sum_c Wc[o, c] (Wt[t, 0] a[b, c, x, y, z, 0] + bt[t]) + bc[o].

    P:139-140 (two affine maps, along t then along the channels)."""
    a = np.asarray(a, np.float64)
    assert a.shape[-1] == 1, "the network input has a time axis of size 1 (P:141)"
    a1 = np.asarray(Wt, np.float64)[:, 0][None, None, None, None, None, :] * a + \
        np.asarray(bt, np.float64)[None, None, None, None, None, :]
    nu0 = np.einsum("oc,bcxyzt->boxyzt", np.asarray(Wc, np.float64), a1)
    return nu0 + np.asarray(bc, np.float64)[None, :, None, None, None, None]


def project(nu, Wp, bp=None):
    """u[b, 0, x] = sum_o Wp[0, o] nu[b, o, x] (+ bp[0]): the channel projection."""
    u = np.einsum("po,boxyzt->bpxyzt", np.asarray(Wp, np.float64), np.asarray(nu, np.float64))
    if bp is not None:
        u = u + np.asarray(bp, np.float64)[None, :, None, None, None, None]
    return u


def rel_l2(u, y):
    """L(u, y) = ||u - y||_2 / ||y||_2 over the whole (global) tensor."""
    u = np.asarray(u, np.float64)
    y = np.asarray(y, np.float64)
    return float(np.sqrt(np.sum((u - y) ** 2)) / np.sqrt(np.sum(y ** 2)))


def network_fwd(a, params, modes):
    """Forward of the whole network.  params: dict with Wt, bt, Wc, bc, Wp, bp
    (bp may be None) and lists R, W, b of length K.  Returns (u, cache) where
    cache holds nu_0..nu_K for the backward."""
    K = len(params["R"])
    nus = [lift(a, params["Wt"], params["bt"], params["Wc"], params["bc"])]
    for k in range(K):
        act = "gelu" if k < K - 1 else "none"                       # reading N1b
        y, _ = sp.layer_fwd(nus[-1], params["R"][k], params["W"][k], params["b"][k], modes, act)
        nus.append(y)
    u = project(nus[-1], params["Wp"], params.get("bp"))
    return u, nus


def network_bwd(a, y_true, params, modes):
    """Loss and its gradient w.r.t. every parameter (same keys as params).

    dL/du = (u - y) / (||u - y|| ||y||); the projection and lift adjoints are
    the transposed affine maps with the broadcast adjoint summing over points
    (P:64); each block uses sp.layer_bwd (pinned in test_oracle_spectral)."""
    u, nus = network_fwd(a, params, modes)
    y_true = np.asarray(y_true, np.float64)
    d = u - y_true
    nd, ny = np.sqrt(np.sum(d * d)), np.sqrt(np.sum(y_true * y_true))
    loss = float(nd / ny)
    du = d / (nd * ny)
    g = {}
    Wp = np.asarray(params["Wp"], np.float64)
    g["Wp"] = np.einsum("bpxyzt,boxyzt->po", du, nus[-1])
    g["bp"] = du.sum(axis=(0, 2, 3, 4, 5)) if params.get("bp") is not None else None
    dnu = np.einsum("po,bpxyzt->boxyzt", Wp, du)
    K = len(params["R"])
    g["R"], g["W"], g["b"] = [None] * K, [None] * K, [None] * K
    for k in reversed(range(K)):
        act = "gelu" if k < K - 1 else "none"
        dnu, g["R"][k], g["W"][k], g["b"][k] = sp.layer_bwd(nus[k], dnu, params["R"][k], params["W"][k],
                                                             params["b"][k], modes, act)
    # lift adjoint: nu0 = Wc a1 + bc, a1 = Wt a + bt
    a = np.asarray(a, np.float64)
    Wt = np.asarray(params["Wt"], np.float64)[:, 0]
    a1 = Wt[None, None, None, None, None, :] * a + np.asarray(params["bt"], np.float64)[None, None, None, None, None, :]
    g["Wc"] = np.einsum("boxyzt,bcxyzt->oc", dnu, a1)
    g["bc"] = dnu.sum(axis=(0, 2, 3, 4, 5))
    da1 = np.einsum("oc,boxyzt->bcxyzt", np.asarray(params["Wc"], np.float64), dnu)
    g["Wt"] = np.einsum("bcxyzt,bcxyz->t", da1, a[..., 0])[:, None]
    g["bt"] = da1.sum(axis=(0, 1, 2, 3, 4))
    return loss, g


def adam_step(p, g, m, v, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """One Adam update (Kingma & Ba, Alg. 1; P:187 uses Adam with lr 1e-3).
    Complex arrays are updated as independent real and imaginary parts (N1d).
    Returns (p, m, v) new arrays."""
    def upd(p, g, m, v):
        m = beta1 * m + (1 - beta1) * g
        v = beta2 * v + (1 - beta2) * g * g
        mh = m / (1 - beta1 ** step)
        vh = v / (1 - beta2 ** step)
        return p - lr * mh / (np.sqrt(vh) + eps), m, v
    if np.iscomplexobj(p):
        pr, mr, vr = upd(p.real, g.real, m.real, v.real)
        pi, mi, vi = upd(p.imag, g.imag, m.imag, v.imag)
        return pr + 1j * pi, mr + 1j * mi, vr + 1j * vi
    return upd(np.asarray(p, np.float64), np.asarray(g, np.float64), np.asarray(m, np.float64),
               np.asarray(v, np.float64))
