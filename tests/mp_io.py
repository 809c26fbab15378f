"""Caller-side 3-D spatial / temporal partitions (SURVEY 8.f N3, App. A
P:292-301) driver, run by tests/test_gpu_multi.py under torchrun: every rank
holds its box of the io partition (px', py', pz', pt'); fno_layer_fwd / _bwd
repartition to the plan's x/y grid and back.  Rank 0 compares the gathered y,
dv and the reduced dW, db with the fp64 oracle.

    torchrun --nproc-per-node 2 tests/mp_io.py --pgrid 2 1 --io 1 1 2 1 --out result.json
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2204_01205_b200 as fno  # noqa: E402
import synth  # noqa: E402
from oracle import spectral as sp  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pgrid", type=int, nargs=2, required=True)
    ap.add_argument("--io", type=int, nargs=4, required=True)
    ap.add_argument("--grid", type=int, nargs=4, default=[16, 16, 16, 8])
    ap.add_argument("--width", type=int, default=4)
    ap.add_argument("--modes", type=int, nargs=4, default=[4, 4, 4, 4])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    grid, C, modes = tuple(a.grid), a.width, tuple(a.modes)
    seed = 913
    v = synth.field((1, C) + grid, modes, seed)
    R = synth.spectral_weights(C, C, modes, seed + 1)
    W, b = synth.channel_weights(C, seed + 2)
    dy = synth.cotangent(v.shape, seed + 3)
    comm = fno.Comm.from_process_group() if world > 1 else None
    plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, pgrid=tuple(a.pgrid)), comm, device=dev,
                    io_pgrid=tuple(a.io))
    box = plan.io_box()
    sl = (slice(None), slice(None)) + tuple(slice(lo, hi) for lo, hi in box)
    k0, k1 = plan.owned_modes()
    t = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).to(dev)   # noqa: E731
    vl, dyl = t(v[sl].astype(np.float32)), t(dy[sl].astype(np.float32))
    Rl = t(R[:, :, :, :, k0:k1].astype(np.complex64))
    Wt, bt = t(W.astype(np.float32)), t(b.astype(np.float32))
    y = torch.empty_like(vl)
    zs = torch.empty_like(vl)
    vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=dev)
    fno.layer_fwd(plan, vl, Rl, Wt, bt, y, zs, vh)
    dv = torch.empty_like(vl)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device=dev)
    dW = torch.empty((C, C), device=dev)
    db = torch.empty((C,), device=dev)
    fno.layer_bwd(plan, vl, zs, vh, dyl, Rl, Wt, dv, dR, dW, db)
    torch.cuda.synchronize()
    mine = dict(box=box, y=y.cpu().numpy(), dv=dv.cpu().numpy(), dR=dR.cpu().numpy())
    gathered = [None] * world
    if world > 1:
        dist.gather_object(mine, gathered if rank == 0 else None, dst=0)
    else:
        gathered = [mine]
    if rank == 0:
        f64 = lambda q: np.asarray(q, np.float32).astype(np.float64)   # noqa: E731
        Y = np.zeros(v.shape)
        DV = np.zeros(v.shape)
        for g in gathered:
            s = (slice(None), slice(None)) + tuple(slice(lo, hi) for lo, hi in g["box"])
            Y[s] = g["y"]
            DV[s] = g["dv"]
        Rd = R.astype(np.complex64).astype(np.complex128)
        y_ref, _ = sp.layer_fwd(f64(v), Rd, f64(W), f64(b), modes)
        dv_r, dR_r, dW_r, db_r = sp.layer_bwd(f64(v), f64(dy), Rd, f64(W), f64(b), modes)
        dRg = np.concatenate([g["dR"] for g in gathered], axis=4)
        res = dict(pgrid=a.pgrid, io=a.io, y_vs_oracle=rel(Y, y_ref), dv_vs_oracle=rel(DV, dv_r),
                   dR_vs_oracle=rel(dRg, dR_r), dW_vs_oracle=rel(dW.cpu().numpy(), dW_r),
                   db_vs_oracle=rel(db.cpu().numpy(), db_r))
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
    if world > 1:
        dist.barrier()
    plan.destroy()
    if comm:
        comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
