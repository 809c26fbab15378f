"""The whole DFNO network (PAPER.md "Full Network")
on top of libfno's fno_net_* calls: buffer ownership (torch tensors for the
parameters, gradients, Adam moments, activations and workspaces) and the call
sequence of one training step.  Every arithmetic step -- lift, the K blocks,
projection, relative-L2 loss, all adjoints and Adam -- runs in libfno's
kernels; this module only allocates and marshals.

    net = Network(plan, layers=4, in_channels=2, seed=0)
    loss = net.train_step(a, y, lr=1e-3)          # fwd, loss, bwd, Adam
"""

from __future__ import annotations

import math

from . import Plan, adam, comm_allreduce, net_bwd, net_fwd, net_loss, net_workspace_size

__all__ = ["Network", "init_params"]


def init_params(plan: Plan, layers: int, in_channels: int, seed: int = 0, proj_bias: bool = True, device=None):
    """Seeded random initialisation on the plan's device (reading Q17 for the
    blocks: R complex-uniform / (C C), W, b uniform +-sqrt(1/C); lift and
    projection uniform +-sqrt(1/fan_in)).  Replicated parameters are drawn from
    the same seed on every rank; R is this rank's kz block."""
    import torch
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device="cpu").manual_seed(220401205 + 7919 * seed)
    C, T = plan.problem.width, plan.problem.grid[3]
    kz_lo, kz_hi = plan.owned_modes()
    mx, my, mz, mt = plan.problem.modes

    def u(shape, bound):
        return ((torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1) * bound).float().to(dev)

    P = {"Wt": u((T,), 1.0), "bt": u((T,), 1.0),
         "Wc": u((C, in_channels), math.sqrt(1.0 / in_channels)), "bc": u((C,), math.sqrt(1.0 / in_channels)),
         "R": [], "W": [], "b": [],
         "Wp": u((C,), math.sqrt(1.0 / C)), "bp": u((1,), math.sqrt(1.0 / C)) if proj_bias else None}
    for _ in range(layers):
        full = (C, C, 2 * mx, 2 * my, 2 * mz, mt)
        re = torch.rand(full, generator=g, dtype=torch.float64)
        im = torch.rand(full, generator=g, dtype=torch.float64)
        R = torch.complex(re, im)[:, :, :, :, kz_lo:kz_hi, :] / (C * C)
        P["R"].append(R.to(torch.complex64).contiguous().to(dev))
        P["W"].append(u((C, C), math.sqrt(1.0 / C)))
        P["b"].append(u((C,), math.sqrt(1.0 / C)))
    return P


class Network:
    """Parameters, gradients, Adam state and activations of one DFNO on one plan."""

    def __init__(self, plan: Plan, layers: int = 4, in_channels: int = 2, seed: int = 0, proj_bias: bool = True,
                 params: dict | None = None, dp_comm=None):
        """dp_comm: optional libfno Comm over the data-parallel replicas (same x/y box,
        different samples); backward() then averages every gradient over it (N4)."""
        import torch
        self.plan, self.K, self.cin, self.proj_bias = plan, layers, in_channels, proj_bias
        self.dp_comm = dp_comm
        dev = plan.workspace.device
        self.params = params if params is not None else init_params(plan, layers, in_channels, seed, proj_bias, dev)
        z = lambda t: None if t is None else torch.zeros_like(t)          # noqa: E731
        self.grads = {k: ([z(x) for x in v] if isinstance(v, list) else z(v)) for k, v in self.params.items()}
        self.m = {k: ([z(x) for x in v] if isinstance(v, list) else z(v)) for k, v in self.params.items()}
        self.v = {k: ([z(x) for x in v] if isinstance(v, list) else z(v)) for k, v in self.params.items()}
        shape = plan.local_shape()
        self.acts = {"nu": [torch.empty(shape, device=dev) for _ in range(layers + 1)],
                     "z": [torch.empty(shape, device=dev) for _ in range(layers - 1)],
                     "vhat": [torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=dev) for _ in range(layers)]}
        self.u = torch.empty((shape[0], 1) + tuple(shape[2:]), device=dev)
        self.scratch = [torch.empty(shape, device=dev) for _ in range(2)]
        self.net_ws = torch.empty(max(net_workspace_size(plan, layers, in_channels, proj_bias), 256),
                                  dtype=torch.uint8, device=dev)
        self.loss3 = torch.zeros(3, device=dev)
        self.step_count = 0

    def forward(self, a, stream=None):
        net_fwd(self.plan, self.params, a, self.acts, self.u, self.cin, self.proj_bias, stream)
        return self.u

    def loss(self, y, stream=None):
        net_loss(self.plan, self.u, y, self.loss3, self.net_ws, stream)
        return self.loss3

    def backward(self, a, y, stream=None):
        net_bwd(self.plan, self.params, a, self.acts, self.u, y, self.grads, self.scratch[0], self.scratch[1],
                self.net_ws, self.cin, self.proj_bias, stream)
        if self.dp_comm is not None:
            for g in self.grads.values():
                for t in (g if isinstance(g, list) else [g]):
                    if t is not None:
                        comm_allreduce(self.dp_comm, t, True, stream)

    def adam_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
        self.step_count += 1
        for k, p in self.params.items():
            if p is None:
                continue
            ps = p if isinstance(p, list) else [p]
            gs = self.grads[k] if isinstance(p, list) else [self.grads[k]]
            ms = self.m[k] if isinstance(p, list) else [self.m[k]]
            vs = self.v[k] if isinstance(p, list) else [self.v[k]]
            for pi, gi, mi, vi in zip(ps, gs, ms, vs):
                adam(pi, gi, mi, vi, self.step_count, lr, beta1, beta2, eps, stream)

    def train_step(self, a, y, lr=1e-3, stream=None):
        """One training step: forward, relative-L2 loss, backward,
        Adam.  Returns the device tensor {L, ||u-y||^2, ||y||^2} (no host sync)."""
        self.forward(a, stream)
        self.loss(y, stream)
        self.backward(a, y, stream)
        self.adam_step(lr, stream=stream)
        return self.loss3
