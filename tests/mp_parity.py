"""Multi-GPU parity driver (run by tests/test_gpu_multi.py under torchrun).

Every rank holds its x/y box of the global field (pgrid (px, py), rank = ix*py
+ iy), runs the decomposed DFNO block forward + backward through libfno (NCCL
pencil all-to-all), and the gathered results are compared on rank 0 with the
fp64 oracle and with the single-GPU libfno result on the same inputs.

    torchrun --nproc-per-node 2 tests/mp_parity.py --pgrid 2 1 --out result.json
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
from oracle import decomp as dc  # noqa: E402
from oracle import spectral as sp  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pgrid", type=int, nargs=2, required=True)
    ap.add_argument("--grid", type=int, nargs=4, default=[16, 16, 16, 8])
    ap.add_argument("--width", type=int, default=4)
    ap.add_argument("--modes", type=int, nargs=4, default=[4, 4, 4, 4])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    px, py = a.pgrid
    assert px * py == world
    grid, C, modes, B = tuple(a.grid), a.width, tuple(a.modes), a.batch
    seed = 777
    v = synth.field((B, C) + grid, modes, seed)
    R = synth.spectral_weights(C, C, modes, seed + 1)
    W, bias = synth.channel_weights(C, seed + 2)
    dy = synth.cotangent(v.shape, seed + 3)

    comm = fno.Comm.from_process_group()
    plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, batch=B, pgrid=(px, py)), comm, device=dev)
    (x0, x1), (y0, y1), _, _ = plan.local_box()
    k0, k1 = plan.owned_modes()
    t = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    vl = t(v[:, :, x0:x1, y0:y1])
    dyl = t(dy[:, :, x0:x1, y0:y1])
    Rl = t(R[:, :, :, :, k0:k1, :])
    Wt, bt = t(W), t(bias)
    y = torch.empty_like(vl)
    z = torch.empty_like(vl)
    vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=dev)
    fno.layer_fwd(plan, vl, Rl, Wt, bt, y, z, vh)
    dv = torch.empty_like(vl)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device=dev)
    dW = torch.empty((C, C), device=dev)
    db = torch.empty((C,), device=dev)
    fno.layer_bwd(plan, vl, z, vh, dyl, Rl, Wt, dv, dR, dW, db)
    u = torch.empty_like(vl)
    fno.spectral_conv_fwd(plan, vl, Rl, u)
    # repartition round trip x/y blocks -> z blocks -> x/y blocks
    shape6 = (B, C) + grid
    dst_pg = (1, 1, 1, 1, world, 1)
    src_pg = (1, 1, px, py, 1, 1)
    dbox = dc.local_box(shape6, dst_pg, rank)
    zb = torch.empty([hi - lo for lo, hi in dbox], device=dev)
    fno.repartition(comm, shape6, src_pg, dst_pg, vl, zb)
    back = torch.empty_like(vl)
    fno.repartition(comm, shape6, dst_pg, src_pg, zb, back)
    torch.cuda.synchronize()
    zb_ref = v[tuple(slice(lo, hi) for lo, hi in dbox)]
    res_local = dict(repart_fwd_exact=bool(np.array_equal(zb.cpu().numpy(), zb_ref)),
                     repart_roundtrip_exact=bool(torch.equal(back, vl)))

    # gather to rank 0 (boxes are equal-sized)
    def gather(tl):
        bufs = [torch.empty_like(tl) for _ in range(world)] if rank == 0 else None
        dist.gather(tl.contiguous(), bufs, dst=0)
        return bufs

    gy, gz, gdv, gu = gather(y), gather(z), gather(dv), gather(u)
    gdR = [None] * world
    dist.gather_object(dR.cpu().numpy(), gdR if rank == 0 else None, dst=0)
    flags = [None] * world
    dist.gather_object(res_local, flags if rank == 0 else None, dst=0)
    dWc, dbc = dW.cpu().numpy(), db.cpu().numpy()
    if rank == 0:
        def assemble(parts):
            out = np.zeros((B, C) + grid, dtype=np.float64)
            for r, pt in enumerate(parts):
                box = dc.local_box(shape6, src_pg, r)
                (a0, a1), (b0, b1) = box[2], box[3]
                out[:, :, a0:a1, b0:b1] = pt.cpu().numpy()
            return out
        Y, Zs, DV, U = assemble(gy), assemble(gz), assemble(gdv), assemble(gu)
        # single-GPU libfno on the same global inputs
        plan1 = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, batch=B), None, device=dev)
        vg, Rg = t(v), t(R)
        y1 = torch.empty_like(vg); z1 = torch.empty_like(vg)
        vh1 = torch.empty(plan1.vhat_shape(), dtype=torch.complex64, device=dev)
        fno.layer_fwd(plan1, vg, Rg, Wt, bt, y1, z1, vh1)
        dv1 = torch.empty_like(vg)
        dR1 = torch.empty(plan1.weight_shape(), dtype=torch.complex64, device=dev)
        dW1 = torch.empty((C, C), device=dev); db1 = torch.empty((C,), device=dev)
        fno.layer_bwd(plan1, vg, z1, vh1, t(dy), Rg, Wt, dv1, dR1, dW1, db1)
        torch.cuda.synchronize()
        # dR: concatenate the owners' kz blocks
        dRg = np.concatenate([gdR[r] for r in range(world)], axis=4)
        f64 = lambda q: np.asarray(q, dtype=np.float64)
        Rd = R.astype(np.complex128)
        y_ref, z_ref = sp.layer_fwd(f64(v), Rd, f64(W), f64(bias), modes)
        dv_r, dR_r, dW_r, db_r = sp.layer_bwd(f64(v), f64(dy), Rd, f64(W), f64(bias), modes)
        u_ref = sp.spectral_conv(f64(v), Rd, modes)
        out = dict(
            pgrid=[px, py], world=world,
            y_vs_oracle=rel(Y, y_ref), z_vs_oracle=rel(Zs, z_ref), u_vs_oracle=rel(U, u_ref),
            dv_vs_oracle=rel(DV, dv_r), dR_vs_oracle=rel(dRg, dR_r),
            dW_vs_oracle=rel(dWc, dW_r), db_vs_oracle=rel(dbc, db_r),
            y_vs_single=rel(Y, y1.cpu().numpy()), dv_vs_single=rel(DV, dv1.cpu().numpy()),
            dW_vs_single=rel(dWc, dW1.cpu().numpy()),
            repartition=flags,
        )
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))
    dist.barrier()
    plan.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
