"""GPU parity of the whole DFNO network (fno_net_*) against the
fp64 oracle (oracle/network.py) on the same seeded fp32 inputs: output u,
relative-L2 loss, the gradient of every parameter, and one Adam step.
Bar: relative L2 <= 1e-5 (the north star's fp32 bar)."""

import numpy as np
import pytest

import synth
from oracle import network as onw
from tests._instances import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_01205_b200 import build
    build.build()


# (grid, C, modes, layers, Cin, proj_bias): a small case, and the c2 shape class
# shrunk in x/y (the forward runs the tensor-core pass C there)
CASES = [
    ((16, 8, 16, 8), 4, (4, 2, 4, 4), 2, 2, True),
    ((16, 8, 16, 8), 3, (2, 2, 3, 3), 3, 1, False),
    ((16, 16, 64, 32), 20, (8, 8, 8, 8), 4, 2, True),
    ((8, 8, 32, 30), 6, (4, 4, 6, 6), 2, 3, True),      # T = 30 (c3 class): scalar t path of the lift adjoint
    ((16, 8, 16, 8), 4, (4, 2, 4, 4), 2, 2, True, 3),    # batch 3: the loss and every sum run over the batch too
]


def _ids(c):
    return "x".join(map(str, c[0])) + f"_C{c[1]}_K{c[3]}_Cin{c[4]}_bp{int(c[5])}" + (f"_B{c[6]}" if len(c) > 6 else "")


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_network_forward_loss_gradients_and_adam_match_oracle(case):
    import torch
    from paper_2204_01205_b200 import Plan, Problem
    from paper_2204_01205_b200.network import Network
    from tests import _gpu as G
    grid, C, modes, K, Cin, bp = case[:6]
    B = case[6] if len(case) > 6 else 1
    X, Y, Z, T = grid
    a = synth.field((B, Cin, X, Y, Z, 1), modes[:3] + (1,), 11, "co2")
    y = synth.field((B, 1, X, Y, Z, T), modes, 12, "co2")
    plan = Plan(Problem(grid=grid, width=C, modes=modes, batch=B))
    net = Network(plan, layers=K, in_channels=Cin, seed=3, proj_bias=bp)
    at, yt = G.t32(a[..., 0]), G.t32(y)
    u = net.forward(at)
    loss3 = net.loss(yt)
    net.backward(at, yt)
    torch.cuda.synchronize()
    P = {k: ([G.np64(x) for x in v] if isinstance(v, list) else (None if v is None else G.np64(v)))
         for k, v in net.params.items()}
    Po = dict(P)
    Po["Wt"] = P["Wt"][:, None]
    Po["Wc"] = P["Wc"]
    Po["Wp"] = P["Wp"][None, :]
    a64, y64 = G.f32(a), G.f32(y)
    u_ref, _ = onw.network_fwd(a64, Po, modes)
    assert rel_l2(G.np64(u), u_ref) < TOL
    loss_ref, g = onw.network_bwd(a64, y64, Po, modes)
    assert abs(float(loss3[0]) - loss_ref) <= TOL * loss_ref
    gg = net.grads
    assert rel_l2(G.np64(gg["Wt"]), g["Wt"][:, 0]) < TOL
    assert rel_l2(G.np64(gg["bt"]), g["bt"]) < TOL
    assert rel_l2(G.np64(gg["Wc"]), g["Wc"]) < TOL
    assert rel_l2(G.np64(gg["bc"]), g["bc"]) < TOL
    assert rel_l2(G.np64(gg["Wp"]), g["Wp"][0]) < TOL
    if bp:
        assert rel_l2(G.np64(gg["bp"]), g["bp"]) < TOL
    for k in range(K):
        assert rel_l2(G.np64(gg["R"][k]), g["R"][k]) < TOL, k
        assert rel_l2(G.np64(gg["W"][k]), g["W"][k]) < TOL, k
        assert rel_l2(G.np64(gg["b"][k]), g["b"][k]) < TOL, k
    # one Adam step on every parameter vs the oracle's Adam on the same gradients
    net.adam_step(lr=1e-3)
    torch.cuda.synchronize()
    for key in ("Wc", "W", "R"):
        new = net.params[key]
        for k in range(K if key in ("W", "R") else 1):
            got = G.np64(new[k] if isinstance(new, list) else new)
            p0 = P[key][k] if isinstance(new, list) else P[key]
            g0 = G.np64(gg[key][k] if isinstance(new, list) else gg[key])
            ref, _, _ = onw.adam_step(p0, g0, np.zeros_like(p0), np.zeros_like(p0), 1, lr=1e-3)
            assert np.max(np.abs(got - ref)) <= 1e-6 + 1e-6 * np.max(np.abs(ref)), key


def test_network_training_reduces_loss():
    """A few Adam steps on a fixed sample lower the relative-L2 misfit."""
    from paper_2204_01205_b200 import Plan, Problem
    from paper_2204_01205_b200.network import Network
    from tests import _gpu as G
    grid, C, modes = (16, 8, 16, 8), 4, (4, 2, 4, 4)
    X, Y, Z, T = grid
    a = synth.field((1, 2, X, Y, Z, 1), modes[:3] + (1,), 21, "co2")
    y = synth.field((1, 1, X, Y, Z, T), modes, 22, "co2")
    net = Network(Plan(Problem(grid=grid, width=C, modes=modes)), layers=2, in_channels=2, seed=5)
    at, yt = G.t32(a[..., 0]), G.t32(y)
    losses = [float(net.train_step(at, yt, lr=1e-2)[0]) for _ in range(8)]
    assert losses[-1] < 0.9 * losses[0], losses
