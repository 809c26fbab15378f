"""World-size-2 (and 4) CPU tests of the multi-rank logic over torch.distributed `gloo`.

Each rank asks libfno (host side, no GPU: `fno_comm_init_local`) for its x/y box
and its retained-kz ownership block, then runs the distributed spectral
convolution with the library's documented exchange layouts:
  send 1: [owner d][B][Xl][Yl][C][nkz_d][mt]   (pass A output)
  recv 1: [source s][B][Xl][Yl][C][nkz][mt]    (pass B input)
  send 2 / recv 2: the reverse
through real `dist.all_to_all_single` exchanges, with the fp64 oracle's per-axis
DFT rows as the local transforms.  The gathered result must equal the
undecomposed oracle (S_dist == S).  The dW/db cross-rank reduction
(all-gather + ascending-rank sum, reading Q14) must be bitwise identical on all
ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pg, grid, C, modes, B, q):
    import paper_2204_01205_b200 as fno
    import synth
    from oracle import decomp as dc
    from oracle import spectral as sp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Y, Z, T = grid
        mx, my, mz, mt = modes
        v = synth.field((B, C) + grid, modes, 99).astype(np.float64)
        R = synth.spectral_weights(C, C, modes, 100).astype(np.complex128)
        comm = fno.Comm.local(world, rank)
        plans = [fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, batch=B, pgrid=pg), fno.Comm.local(world, r),
                          allocate=False) for r in range(world)]
        boxes = [p.local_box() for p in plans]
        owned = [p.owned_modes() for p in plans]
        (x0, x1), (y0, y1), _, _ = boxes[rank]
        k0, k1 = owned[rank]
        Xl, Yl = x1 - x0, y1 - y0
        kx, ky, kz, kt = sp.check_modes(grid, modes)
        # ---- pass A equivalent: t, z transforms on the local box --------------
        a = sp._apply(v[:, :, x0:x1, y0:y1].astype(np.complex128), sp.dft_rows(T, kt, -1), 5)
        a = sp._apply(a, sp.dft_rows(Z, kz, -1), 4)                        # [B][C][Xl][Yl][2mz][mt]
        a = np.transpose(a, (0, 2, 3, 1, 4, 5))                            # [B][Xl][Yl][C][2mz][mt]
        send = np.concatenate([a[:, :, :, :, lo:hi, :].ravel() for lo, hi in owned])
        scounts = [B * Xl * Yl * C * (hi - lo) * mt for lo, hi in owned]
        rcounts = [B * Xl * Yl * C * (k1 - k0) * mt] * world
        recv = _a2a(send, scounts, rcounts)
        # ---- pass B equivalent on the owned kz block ----------------------------
        nkz = k1 - k0
        plane = np.zeros((B, C, X, Y, nkz, mt), dtype=np.complex128)
        off = 0
        for s in range(world):
            (sx0, sx1), (sy0, sy1), _, _ = boxes[s]
            n = rcounts[s]
            blk = recv[off:off + n].reshape(B, sx1 - sx0, sy1 - sy0, C, nkz, mt)
            plane[:, :, sx0:sx1, sy0:sy1] = np.transpose(blk, (0, 3, 1, 2, 4, 5))
            off += n
        if nkz:
            h = sp._apply(plane, sp.dft_rows(Y, ky, -1), 3)
            h = sp._apply(h, sp.dft_rows(X, kx, -1), 2)
            w = sp.mix(h, R[:, :, :, :, k0:k1, :])
            g = sp._apply(w, sp.dft_rows(X, kx, +1).T, 2)
            g = sp._apply(g, sp.dft_rows(Y, ky, +1).T, 3)                  # [B][C][X][Y][nkz][mt]
        else:
            g = plane
        send2 = np.concatenate([np.transpose(g[:, :, bx[0][0]:bx[0][1], bx[1][0]:bx[1][1]], (0, 2, 3, 1, 4, 5)).ravel()
                                for bx in boxes])
        recv2 = _a2a(send2, rcounts, scounts)
        # ---- pass C equivalent: inverse z, t on the local box --------------------
        col = np.zeros((B, Xl, Yl, C, 2 * mz, mt), dtype=np.complex128)
        off = 0
        for d, (lo, hi) in enumerate(owned):
            n = scounts[d]
            col[:, :, :, :, lo:hi, :] = recv2[off:off + n].reshape(B, Xl, Yl, C, hi - lo, mt)
            off += n
        col = np.transpose(col, (0, 3, 1, 2, 4, 5))
        a = sp._apply(col, sp.dft_rows(Z, kz, +1).T, 4) * sp.c_weight(T, mt)
        u_loc = sp._apply(a, sp.dft_rows(T, kt, +1).T, 5).real / float(X * Y * Z * T)
        parts = [None] * world
        dist.all_gather_object(parts, (boxes[rank], u_loc))
        # ---- dW/db style reduction: all-gather + ascending-rank fixed-order sum ---
        part = np.random.default_rng(rank).standard_normal(C * C + C).astype(np.float32)
        allp = [torch.zeros(C * C + C) for _ in range(world)]
        dist.all_gather(allp, torch.from_numpy(part))
        tot = torch.zeros(C * C + C)
        for r in range(world):
            tot += allp[r]
        sums = [None] * world
        dist.all_gather_object(sums, tot.numpy().tobytes())
        if rank == 0:
            U = np.zeros((B, C) + grid)
            for (bx, ul) in parts:
                U[:, :, bx[0][0]:bx[0][1], bx[1][0]:bx[1][1]] = ul
            ref = sp.spectral_conv(v, R, modes)
            err = float(np.linalg.norm(U - ref) / np.linalg.norm(ref))
            owned_all = sorted(k for lo, hi in owned for k in range(lo, hi))
            q.put(dict(err=err, reduce_identical=len(set(sums)) == 1, owned_ok=owned_all == list(range(2 * mz)),
                       boxes_ok=all(list(map(tuple, boxes[r])) == [tuple(x) for x in
                                    dc.local_box((B, C) + grid, (1, 1) + tuple(pg) + (1, 1), r)[2:]]
                                    for r in range(world))))
        for p in plans:
            p.destroy()
        comm.destroy()
    finally:
        dist.destroy_process_group()


def _a2a(send, scounts, rcounts):
    s = torch.from_numpy(np.ascontiguousarray(send).view(np.float64).copy())
    r = torch.empty(2 * sum(rcounts), dtype=torch.float64)
    dist.all_to_all_single(r, s, [2 * c for c in rcounts], [2 * c for c in scounts])
    return r.numpy().view(np.complex128)


@pytest.mark.parametrize("pg,grid,C,modes,B", [((2, 1), (8, 8, 16, 8), 3, (2, 3, 4, 4), 1),
                                                ((1, 2), (8, 8, 16, 8), 2, (3, 2, 4, 4), 2),
                                                ((2, 2), (8, 8, 16, 8), 2, (2, 2, 4, 4), 1),
                                                ((4, 1), (8, 4, 16, 8), 2, (2, 1, 1, 4), 1)])   # 2mz < P
def test_gloo_distributed_spectral_conv_equals_oracle(pg, grid, C, modes, B):
    world = pg[0] * pg[1]
    from paper_2204_01205_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pg, grid, C, modes, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    codes = [p.exitcode for p in procs]
    assert codes == [0] * world, codes
    res = q.get(timeout=10)
    assert res["err"] < 1e-13, res
    assert res["reduce_identical"] and res["owned_ok"] and res["boxes_ok"], res
