"""Helpers for the -m gpu parity tests: run libfno on numpy inputs (fp32)."""

import numpy as np
import torch

import paper_2204_01205_b200 as fno

DEV = "cuda"


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(DEV)


def tc64(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex64))).to(DEV)


def np64(t):
    return t.detach().cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


def f32(a):
    """The fp32 values the GPU sees, promoted back to fp64 for the oracle."""
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return a.astype(np.complex64).astype(np.complex128)
    return a.astype(np.float32).astype(np.float64)


def make_plan(grid, C, modes, B=1, act="gelu", pgrid=(1, 1), comm=None):
    return fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, batch=B, pgrid=pgrid, act=act), comm)


def layer_fwd(plan, v, R, W, b, save=True):
    vt, Rt, Wt = t32(v), tc64(R), t32(W)
    bt = t32(b) if b is not None else None
    y = torch.empty_like(vt)
    z = torch.empty_like(vt) if save else None
    vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=DEV) if save else None
    fno.layer_fwd(plan, vt, Rt, Wt, bt, y, z, vh)
    torch.cuda.synchronize()
    return y, z, vh


def spectral_fwd(plan, v, R):
    vt, Rt = t32(v), tc64(R)
    u = torch.empty_like(vt)
    vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=DEV)
    fno.spectral_conv_fwd(plan, vt, Rt, u, vh)
    torch.cuda.synchronize()
    return u, vh
