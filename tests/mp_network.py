"""Multi-GPU parity driver of the whole DFNO network, run by
tests/test_gpu_multi.py under torchrun.  Every rank holds its x/y box of the
input a and target y, runs fno_net_fwd / fno_net_loss / fno_net_bwd (NCCL or
NVLink-peer pencil exchanges inside the blocks, rank-ordered sums of the
replicated-parameter gradients), and rank 0 compares the gathered u, the loss
and every gradient with the fp64 network oracle on the global inputs.

    torchrun --nproc-per-node 2 tests/mp_network.py --pgrid 2 1 --out result.json
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
from oracle import network as onw  # noqa: E402
from paper_2204_01205_b200.network import Network  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pgrid", type=int, nargs=2, required=True)
    ap.add_argument("--grid", type=int, nargs=4, default=[16, 16, 16, 8])
    ap.add_argument("--width", type=int, default=4)
    ap.add_argument("--modes", type=int, nargs=4, default=[4, 4, 4, 4])
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    px, py = a.pgrid
    grid, C, modes, K, Cin = tuple(a.grid), a.width, tuple(a.modes), a.layers, 2
    X, Y, Z, T = grid
    ain = synth.field((1, Cin, X, Y, Z, 1), modes[:3] + (1,), 31, "co2")
    ytg = synth.field((1, 1, X, Y, Z, T), modes, 32, "co2")
    comm = fno.Comm.from_process_group()
    plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, pgrid=(px, py)), comm, device=dev)
    (x0, x1), (y0, y1), _, _ = plan.local_box()
    k0, k1 = plan.owned_modes()
    net = Network(plan, layers=K, in_channels=Cin, seed=4)
    t = lambda arr: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(dev)   # noqa: E731
    a_loc, y_loc = t(ain[:, :, x0:x1, y0:y1, :, 0]), t(ytg[:, :, x0:x1, y0:y1])
    u = net.forward(a_loc)
    loss3 = net.loss(y_loc)
    net.backward(a_loc, y_loc)
    torch.cuda.synchronize()
    gathered = [None] * world
    mine = dict(box=(x0, x1, y0, y1), kz=(k0, k1), u=u.cpu().numpy(),
                dR=[g.cpu().numpy() for g in net.grads["R"]])
    dist.gather_object(mine, gathered if rank == 0 else None, dst=0)
    if rank == 0:
        f32 = lambda q: np.asarray(q, np.float32).astype(np.float64)   # noqa: E731
        U = np.zeros((1, 1) + grid)
        for g in gathered:
            b = g["box"]
            U[:, :, b[0]:b[1], b[2]:b[3]] = g["u"]
        # the same parameters on the global problem: replicated ones as drawn,
        # R assembled from the owners' kz blocks
        P = {k: (None if v is None else (v.detach().cpu().numpy().astype(np.float64) if not isinstance(v, list) else None))
             for k, v in net.params.items()}
        full = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes), None, device=dev, allocate=False)
        from paper_2204_01205_b200.network import init_params
        Pfull = init_params(full, K, Cin, seed=4, device=dev)
        full.destroy()
        Po = {"Wt": P["Wt"][:, None], "bt": P["bt"], "Wc": P["Wc"], "bc": P["bc"], "Wp": P["Wp"][None, :],
              "bp": P["bp"],
              "R": [x.cpu().numpy().astype(np.complex128) for x in Pfull["R"]],
              "W": [x.cpu().numpy().astype(np.float64) for x in net.params["W"]],
              "b": [x.cpu().numpy().astype(np.float64) for x in net.params["b"]]}
        u_ref, _ = onw.network_fwd(f32(ain), Po, modes)
        loss_ref, gr = onw.network_bwd(f32(ain), f32(ytg), Po, modes)
        g = net.grads
        res = dict(pgrid=[px, py], world=world,
                   u_vs_oracle=rel(U, u_ref), loss_vs_oracle=abs(float(loss3[0]) - loss_ref) / loss_ref,
                   dWt_vs_oracle=rel(g["Wt"].cpu().numpy(), gr["Wt"][:, 0]),
                   dbt_vs_oracle=rel(g["bt"].cpu().numpy(), gr["bt"]),
                   dWc_vs_oracle=rel(g["Wc"].cpu().numpy(), gr["Wc"]),
                   dbc_vs_oracle=rel(g["bc"].cpu().numpy(), gr["bc"]),
                   dWp_vs_oracle=rel(g["Wp"].cpu().numpy(), gr["Wp"][0]),
                   dbp_vs_oracle=rel(g["bp"].cpu().numpy(), gr["bp"]))
        for k in range(K):
            dRg = np.concatenate([gg["dR"][k] for gg in gathered], axis=4)
            res[f"dR{k}_vs_oracle"] = rel(dRg, gr["R"][k])
            res[f"dW{k}_vs_oracle"] = rel(g["W"][k].cpu().numpy(), gr["W"][k])
            res[f"db{k}_vs_oracle"] = rel(g["b"][k].cpu().numpy(), gr["b"][k])
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
    dist.barrier()
    del net
    plan.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
