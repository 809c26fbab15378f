"""fp64 oracle: partitions, repartition and the x/y decomposition simulator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Partition = Cartesian worker grid, one entry per tensor dimension,
  row-major rank <-> coordinate (reading Q11), balanced blocks with the first
  n mod p blocks one longer (reading Q11; SPEC block_range).
* Repartition R_{P->Q}: "a high-dimensional generalization of all-to-all ...
  any worker may need to send or receive subtensors to or from any or all
  other workers"; its adjoint is R_{Q->P}.
* Decomposition simulator: the distributed spectral convolution S_dist
  (Eq. DFFT/sconv_dist) run on an explicit x/y worker grid with the
  index sets I_1 = {t, z} (local), one repartition to kz blocks, I_2 = {y, x}
  (reading Q10/Q12), R_phi applied only on the owner of each retained kz
  (P:125), then the adjoint chain back.  It uses only slicing and the
  single-axis DFT rows of oracle.spectral, so it checks the partition logic
  (boxes, kz ownership, exchange index maps) against the undecomposed oracle.

Parity status: pinned (tests/test_oracle_decomp.py: SPEC examples for
block_range / local boxes, tiling by brute-force membership, repartition ==
global slicing, round trip == identity, adjoint identity, simulator ==
undecomposed oracle for pgrids (1,1), (2,1), (2,2), (4,2), (3,3)).
"""

from __future__ import annotations

import numpy as np

from . import spectral as sp

__all__ = [
    "block_range", "rank_to_coords", "coords_to_rank", "local_box", "owned_kz",
    "transfer_plan", "repartition", "simulate_spectral_conv",
]


def block_range(n: int, p: int, i: int):
    """[start, stop) of block i of n items split over p workers (q = n//p, r = n%p;
    blocks 0..r-1 have q+1 items; start = i*q + min(i, r)); empty when p > n."""
    if not (0 <= i < p):
        raise ValueError("block index out of range")
    q, r = divmod(n, p)
    start = i * q + min(i, r)
    return start, start + q + (1 if i < r else 0)


def rank_to_coords(pgrid, rank: int):
    """Row-major rank -> worker coordinates (last dimension fastest)."""
    return tuple(int(c) for c in np.unravel_index(rank, tuple(pgrid)))


def coords_to_rank(pgrid, coords) -> int:
    return int(np.ravel_multi_index(tuple(coords), tuple(pgrid)))


def local_box(global_shape, pgrid, rank: int):
    """Per-dimension [lo, hi) of worker `rank`'s subtensor ("the location of
    its corresponding local subtensor in the global distributed tensor")."""
    if len(global_shape) != len(pgrid):
        raise ValueError("dimensionality mismatch")
    co = rank_to_coords(pgrid, rank)
    return [block_range(int(n), int(p), c) for n, p, c in zip(global_shape, pgrid, co)]


def owned_kz(mz: int, P: int, rank: int):
    """Retained-kz index block [lo, hi) owned by `rank` after the forward exchange:
    the 2mz retained kz planes split over all P ranks (reading Q12)."""
    return block_range(2 * mz, P, rank)


def transfer_plan(global_shape, src_pgrid, dst_pgrid):
    """All non-empty intersections (src_rank, dst_rank, box) of a source box with a
    destination box, sorted by (src, dst)."""
    if not (len(global_shape) == len(src_pgrid) == len(dst_pgrid)):
        raise ValueError("repartition needs partitions with the tensor's ndim (P:73)")
    nsrc = int(np.prod(src_pgrid))
    ndst = int(np.prod(dst_pgrid))
    plan = []
    for s in range(nsrc):
        sb = local_box(global_shape, src_pgrid, s)
        for d in range(ndst):
            db = local_box(global_shape, dst_pgrid, d)
            box = [(max(a[0], b[0]), min(a[1], b[1])) for a, b in zip(sb, db)]
            if all(lo < hi for lo, hi in box):
                plan.append((s, d, box))
    return plan


def repartition(src_locals, global_shape, src_pgrid, dst_pgrid):
    """R_{P->Q}: given every source worker's local block, return every destination
    worker's local block, moving each intersection box from its sender to its
    receiver.  The adjoint is repartition with the pgrids swapped."""
    ndst = int(np.prod(dst_pgrid))
    dtype = src_locals[0].dtype
    out = []
    for d in range(ndst):
        db = local_box(global_shape, dst_pgrid, d)
        out.append(np.zeros([hi - lo for lo, hi in db], dtype=dtype))
    for s, d, box in transfer_plan(global_shape, src_pgrid, dst_pgrid):
        sb = local_box(global_shape, src_pgrid, s)
        db = local_box(global_shape, dst_pgrid, d)
        src_sl = tuple(slice(lo - o[0], hi - o[0]) for (lo, hi), o in zip(box, sb))
        dst_sl = tuple(slice(lo - o[0], hi - o[0]) for (lo, hi), o in zip(box, db))
        out[d][dst_sl] = src_locals[s][src_sl]
    return out


def simulate_spectral_conv(v: np.ndarray, R: np.ndarray, modes, pgrid_xy):
    """S_dist v on an explicit (px, py) grid; returns the gathered u.

    v: global [B, C, X, Y, Z, T]; R: global [C, C, 2mx, 2my, 2mz, mt].
    Rank r = ix*py + iy holds the box block_range(X,px,ix) x block_range(Y,py,iy).
    """
    B, C, X, Y, Z, T = v.shape
    px, py = pgrid_xy
    P = px * py
    kx, ky, kz, kt = sp.check_modes((X, Y, Z, T), modes)
    mz2, mt = len(kz), len(kt)
    pg = (1, 1, px, py, 1, 1)
    boxes = [local_box(v.shape, pg, r) for r in range(P)]

    # stage I_1 = {t, z}: local transforms, truncated (reading Q9)
    slabs = []
    for r in range(P):
        (_, _), (_, _), (x0, x1), (y0, y1), _, _ = boxes[r]
        a = sp._apply(v[:, :, x0:x1, y0:y1].astype(np.complex128), sp.dft_rows(T, kt, -1), 5)
        a = sp._apply(a, sp.dft_rows(Z, kz, -1), 4)           # [B, C, Xl, Yl, 2mz, mt]
        slabs.append(a)

    # repartition x/y blocks -> kz blocks (all-to-all), then I_2 = {y, x}
    what_owned = []
    for d in range(P):
        k0, k1 = owned_kz(modes[2], P, d)
        plane = np.zeros((B, C, X, Y, k1 - k0, mt), dtype=np.complex128)
        for s in range(P):
            (_, _), (_, _), (x0, x1), (y0, y1), _, _ = boxes[s]
            plane[:, :, x0:x1, y0:y1] = slabs[s][:, :, :, :, k0:k1, :]
        a = sp._apply(plane, sp.dft_rows(Y, ky, -1), 3)
        a = sp._apply(a, sp.dft_rows(X, kx, -1), 2)            # V̂ on owned kz
        w = sp.mix(a, R[:, :, :, :, k0:k1, :])                 # R_phi on owners only
        g = sp._apply(w, sp.dft_rows(X, kx, +1).T, 2)
        g = sp._apply(g, sp.dft_rows(Y, ky, +1).T, 3)          # [B, C, X, Y, kz_loc, mt]
        what_owned.append(g)

    # adjoint repartition kz blocks -> x/y blocks, then inverse z, t
    u = np.zeros((B, C, X, Y, Z, T))
    c = sp.c_weight(T, mt)
    for r in range(P):
        (_, _), (_, _), (x0, x1), (y0, y1), _, _ = boxes[r]
        col = np.zeros((B, C, x1 - x0, y1 - y0, mz2, mt), dtype=np.complex128)
        for d in range(P):
            k0, k1 = owned_kz(modes[2], P, d)
            col[:, :, :, :, k0:k1, :] = what_owned[d][:, :, x0:x1, y0:y1]
        a = sp._apply(col, sp.dft_rows(Z, kz, +1).T, 4) * c
        u[:, :, x0:x1, y0:y1] = sp._apply(a, sp.dft_rows(T, kt, +1).T, 5).real / float(X * Y * Z * T)
    return u


def all_boxes_tile(global_shape, pgrid) -> bool:
    """Brute-force membership count: every global index lies in exactly one box."""
    count = np.zeros(tuple(global_shape), dtype=np.int64)
    for r in range(int(np.prod(pgrid))):
        box = local_box(global_shape, pgrid, r)
        count[tuple(slice(lo, hi) for lo, hi in box)] += 1
    return bool((count == 1).all())

