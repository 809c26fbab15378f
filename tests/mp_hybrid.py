"""Data x domain hybrid driver, run by tests/test_gpu_multi.py
under torchrun: world = dp replicas x (px * py) domain ranks, rank = replica *
(px*py) + domain rank.  Each replica holds a different sample (a_r, y_r) on its
own x/y-decomposed plan; after fno_net_bwd the gradients are averaged over the
replicas (fno_comm_allreduce).  Rank 0 compares them with the mean of the fp64
network oracle's gradients over the samples.

    torchrun --nproc-per-node 2 tests/mp_hybrid.py --dp 2 --pgrid 1 1 --out result.json
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
from paper_2204_01205_b200.network import Network, init_params  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dp", type=int, required=True)
    ap.add_argument("--pgrid", type=int, nargs=2, default=[1, 1])
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
    px, py = a.pgrid
    nd = px * py
    assert world == a.dp * nd
    rep, drank = rank // nd, rank % nd
    # process groups: the domain group of this replica, the data group of this domain rank
    dom_groups = [dist.new_group([r * nd + d for d in range(nd)]) for r in range(a.dp)]
    dp_groups = [dist.new_group([r * nd + d for r in range(a.dp)]) for d in range(nd)]
    grid, C, modes, K, Cin = tuple(a.grid), a.width, tuple(a.modes), 2, 2
    X, Y, Z, T = grid
    dcomm = fno.Comm.from_process_group(dom_groups[rep]) if nd > 1 else None
    pcomm = fno.Comm.from_process_group(dp_groups[drank])
    plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, pgrid=(px, py)), dcomm, device=dev)
    (x0, x1), (y0, y1), _, _ = plan.local_box()
    net = Network(plan, layers=K, in_channels=Cin, seed=9, dp_comm=pcomm)
    samples = [(synth.field((1, Cin, X, Y, Z, 1), modes[:3] + (1,), 41 + 2 * r, "co2"),
                synth.field((1, 1, X, Y, Z, T), modes, 42 + 2 * r, "co2")) for r in range(a.dp)]
    ain, ytg = samples[rep]
    t = lambda arr: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(dev)   # noqa: E731
    a_loc, y_loc = t(ain[:, :, x0:x1, y0:y1, :, 0]), t(ytg[:, :, x0:x1, y0:y1])
    net.forward(a_loc)
    net.loss(y_loc)
    net.backward(a_loc, y_loc)          # gradients averaged over the replicas inside
    torch.cuda.synchronize()
    mine = dict(rep=rep, kz=plan.owned_modes(), dR=[g.cpu().numpy() for g in net.grads["R"]],
                Wc=net.grads["Wc"].cpu().numpy(), W=[g.cpu().numpy() for g in net.grads["W"]],
                Wt=net.grads["Wt"].cpu().numpy(), Wp=net.grads["Wp"].cpu().numpy())
    gathered = [None] * world
    dist.gather_object(mine, gathered if rank == 0 else None, dst=0)
    if rank == 0:
        f32 = lambda q: np.asarray(q, np.float32).astype(np.float64)   # noqa: E731
        full = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes), None, device=dev, allocate=False)
        Pf = init_params(full, K, Cin, seed=9, device=dev)
        full.destroy()
        Po = {"Wt": Pf["Wt"].cpu().numpy().astype(np.float64)[:, None], "bt": Pf["bt"].cpu().numpy().astype(np.float64),
              "Wc": Pf["Wc"].cpu().numpy().astype(np.float64), "bc": Pf["bc"].cpu().numpy().astype(np.float64),
              "Wp": Pf["Wp"].cpu().numpy().astype(np.float64)[None, :], "bp": Pf["bp"].cpu().numpy().astype(np.float64),
              "R": [x.cpu().numpy().astype(np.complex128) for x in Pf["R"]],
              "W": [x.cpu().numpy().astype(np.float64) for x in Pf["W"]],
              "b": [x.cpu().numpy().astype(np.float64) for x in Pf["b"]]}
        gs = [onw.network_bwd(f32(s[0]), f32(s[1]), Po, modes)[1] for s in samples]
        mean = lambda key, k=None: sum((g[key][k] if k is not None else g[key]) for g in gs) / len(gs)   # noqa: E731
        res = dict(dp=a.dp, pgrid=[px, py],
                   dWc_vs_oracle=rel(gathered[0]["Wc"], mean("Wc")),
                   dWt_vs_oracle=rel(gathered[0]["Wt"], mean("Wt")[:, 0]),
                   dWp_vs_oracle=rel(gathered[0]["Wp"], mean("Wp")[0]))
        for k in range(K):
            res[f"dW{k}_vs_oracle"] = rel(gathered[0]["W"][k], mean("W", k))
            dR = np.concatenate([g["dR"][k] for g in gathered[:nd]], axis=4)   # replica 0's domain ranks
            res[f"dR{k}_vs_oracle"] = rel(dR, mean("R", k))
        # every replica holds the same averaged gradients
        res["replicas_identical"] = all(np.array_equal(gathered[r * nd]["Wc"], gathered[0]["Wc"]) for r in range(a.dp))
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
    dist.barrier()
    del net
    plan.destroy()
    if dcomm:
        dcomm.destroy()
    pcomm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
