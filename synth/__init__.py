"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no DFT, no mixing, no
activation): it only draws numbers.  Both the oracle and the CUDA path consume
exactly the arrays produced here (fp32, promoted to fp64 by the oracle).

Recipe:
  v   = smooth + 0.1 * N(0, 1) per channel.  smooth = sum of `n_waves` separable
        products of 1D cosines, cos(2 pi a x/X + p_x) cos(2 pi b y/Y + p_y) ...,
        amplitude ~ (1 + |k|^2)^-1, half of the wave numbers inside the retained
        set and half outside (so pass-band, stop-band and the +-m boundary are
        exercised).  shape="ns": isotropic (4D Navier-Stokes-shaped);
        shape="co2": x/y correlation length 4x the z one (layered permeability)
        and an amplitude ramp along t (plume growth).
  R   = complex uniform(-1, 1) * 1/(C_in C_out)      (SPEC init_model, reading Q17)
  W   = uniform(-sqrt(1/C), sqrt(1/C)), b likewise    (reading Q17)
  dy  = N(0, 1)
Seeds: 220401205 + 1000 * config_index + layer.
"""

from __future__ import annotations

import numpy as np

BASE_SEED = 220401205

# BASELINE.json configs (index -> parameters).  grid = global X, Y, Z, T.
CONFIGS = {
    1: dict(name="c1", grid=(16, 16, 16, 8), width=4, modes=(4, 4, 4, 4), layers=1, shape="ns"),
    2: dict(name="c2", grid=(64, 64, 64, 32), width=20, modes=(8, 8, 8, 8), layers=4, shape="ns"),
    3: dict(name="c3", grid=(64, 64, 64, 30), width=20, modes=(12, 12, 12, 12), layers=4, shape="co2"),
    4: dict(name="c4", grid=(64, 128, 128, 32), width=20, modes=(12, 12, 12, 12), layers=4, shape="ns"),
    5: dict(name="c5", grid=(256, 256, 256, 32), width=20, modes=(16, 16, 16, 16), layers=4, shape="ns"),
}


def seed_for(config_index: int, layer: int = 0, salt: int = 0) -> int:
    return BASE_SEED + 1000 * int(config_index) + int(layer) + 7919 * int(salt)


def _wave_numbers(rng, n, m, count, inside):
    if inside:
        k = rng.integers(0, m, size=count)            # inside the retained low band
    else:
        lo = min(m, n // 2)
        k = rng.integers(lo, n // 2 + 1, size=count) if lo <= n // 2 else np.zeros(count, int)
    sign = rng.choice([-1, 1], size=count)
    return k * sign


def field(shape, modes, seed: int, kind: str = "ns", n_waves: int = 8, noise: float = 0.1) -> np.ndarray:
    """Input field v [B, C, X, Y, Z, T] float32."""
    B, C, X, Y, Z, T = (int(s) for s in shape)
    mx, my, mz, mt = (int(m) for m in modes)
    rng = np.random.default_rng(seed)
    out = (noise * rng.standard_normal((B, C, X, Y, Z, T), dtype=np.float32))
    ax = [np.arange(n, dtype=np.float64) for n in (X, Y, Z, T)]
    for b in range(B):
        for c in range(C):
            acc = np.zeros((X, Y, Z, T), dtype=np.float64)
            for w in range(n_waves):
                inside = (w % 2 == 0)
                ks = [int(_wave_numbers(rng, n, m, 1, inside)[0])
                      for n, m in zip((X, Y, Z, T), (mx, my, mz, mt))]
                if kind == "co2":
                    ks[0] = ks[0] // 4 if abs(ks[0]) >= 4 else ks[0]
                    ks[1] = ks[1] // 4 if abs(ks[1]) >= 4 else ks[1]
                amp = 1.0 / (1.0 + sum(k * k for k in ks))
                ph = rng.uniform(0, 2 * np.pi, size=4)
                f = [np.cos(2 * np.pi * k * a / n + p) for k, a, n, p in zip(ks, ax, (X, Y, Z, T), ph)]
                acc += amp * (f[0][:, None, None, None] * f[1][None, :, None, None] * f[2][None, None, :, None] *
                              f[3][None, None, None, :])
            if kind == "co2":
                acc *= (0.25 + ax[3] / max(T - 1, 1))[None, None, None, :]
            out[b, c] += acc.astype(np.float32)
    return out


def field_torch(shape, modes, seed: int, kind: str = "ns", n_waves: int = 8, noise: float = 0.1, device="cuda"):
    """Same recipe as `field`, drawn on the device with torch (for bench-sized
    fields; a different random stream than the numpy version)."""
    import math

    import torch
    B, C, X, Y, Z, T = (int(s) for s in shape)
    mx, my, mz, mt = (int(m) for m in modes)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    out = noise * torch.randn((B, C, X, Y, Z, T), generator=g, device=device, dtype=torch.float32)
    rng = np.random.default_rng(seed)
    ax = [torch.arange(n, device=device, dtype=torch.float32) for n in (X, Y, Z, T)]
    ramp = (0.25 + ax[3] / max(T - 1, 1)) if kind == "co2" else None
    for b in range(B):
        for c in range(C):
            acc = torch.zeros((X, Y, Z, T), device=device, dtype=torch.float32)
            for w in range(n_waves):
                inside = (w % 2 == 0)
                ks = [int(_wave_numbers(rng, n, m, 1, inside)[0]) for n, m in zip((X, Y, Z, T), (mx, my, mz, mt))]
                if kind == "co2":
                    ks[0] = ks[0] // 4 if abs(ks[0]) >= 4 else ks[0]
                    ks[1] = ks[1] // 4 if abs(ks[1]) >= 4 else ks[1]
                amp = 1.0 / (1.0 + sum(k * k for k in ks))
                ph = rng.uniform(0, 2 * np.pi, size=4)
                f = [torch.cos(2 * math.pi * k * a / n + float(p)) for k, a, n, p in zip(ks, ax, (X, Y, Z, T), ph)]
                acc += amp * (f[0][:, None, None, None] * f[1][None, :, None, None] * f[2][None, None, :, None] *
                              f[3][None, None, None, :])
            if ramp is not None:
                acc *= ramp
            out[b, c] += acc
    return out


def spectral_weights(c_in: int, c_out: int, modes, seed: int, kz_range=None) -> np.ndarray:
    """R [C_in, C_out, 2mx, 2my, 2mz_or_local, mt] complex64 (global, then optionally
    sliced to a retained-kz block so every partition sees the same global weights)."""
    mx, my, mz, mt = (int(m) for m in modes)
    rng = np.random.default_rng(seed)
    shp = (c_in, c_out, 2 * mx, 2 * my, 2 * mz, mt)
    scale = 1.0 / (c_in * c_out)
    re = rng.uniform(-1.0, 1.0, size=shp).astype(np.float32)
    im = rng.uniform(-1.0, 1.0, size=shp).astype(np.float32)
    R = (scale * (re + 1j * im)).astype(np.complex64)
    if kz_range is not None:
        R = np.ascontiguousarray(R[:, :, :, :, kz_range[0]:kz_range[1], :])
    return R


def channel_weights(c: int, seed: int):
    """(W [C, C] float32, b [C] float32)."""
    rng = np.random.default_rng(seed)
    s = np.sqrt(1.0 / c)
    W = rng.uniform(-s, s, size=(c, c)).astype(np.float32)
    b = rng.uniform(-s, s, size=(c,)).astype(np.float32)
    return W, b


def cotangent(shape, seed: int) -> np.ndarray:
    """Upstream gradient dy [B, C, X, Y, Z, T] float32 ~ N(0, 1)."""
    return np.random.default_rng(seed).standard_normal(tuple(shape), dtype=np.float32)


def problem(config_index: int, batch: int = 1, grid=None, width=None, layer: int = 0, with_dy=True):
    """All inputs of one layer of config `config_index` (optionally shrunk grid/width)."""
    cfg = CONFIGS[config_index]
    X, Y, Z, T = grid if grid is not None else cfg["grid"]
    C = width if width is not None else cfg["width"]
    modes = cfg["modes"]
    s = seed_for(config_index, layer)
    v = field((batch, C, X, Y, Z, T), modes, s, cfg["shape"])
    R = spectral_weights(C, C, modes, s + 1)
    W, b = channel_weights(C, s + 2)
    dy = cotangent(v.shape, s + 3) if with_dy else None
    return dict(v=v, R=R, W=W, b=b, dy=dy, modes=modes, grid=(X, Y, Z, T))
