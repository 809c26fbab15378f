#!/usr/bin/env python
"""bench.py — throughput of the 4D FNO spectral-layer hot path (arXiv 2204.01205).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c4|c5]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step is one training pass of the whole hot path over
one synthetic batch: the forward of `layers` DFNO blocks in training mode
(storing z and V^), then their backward (dv, dR, dW, db).  Default workload:
BASELINE.json configs[2] (c3), the shape the metric "fwd+bwd at 1/2/4/8 B200"
is quoted on: the CO2-multiphase-shaped training step,
global grid 64x64x64x30, width 20, modes 12, 4 Fourier layers, batch 1,
strong-scaled over the x/y process grids (1,1) (2,1) (2,2) (4,2),
with the pencil repartitions over NVLink.  --config c2 | c4 (weak, per-GPU box
fixed) | c5 select the other BASELINE configs.

metric: grid-points x channels x layers processed (fwd+bwd) per second, whole
job; value = B * X*Y*Z*T (global) * C * layers / step time, the step time the
median over K repetitions (each bracketed by a barrier, device-timed with CUDA
events, max over ranks).  The line also carries the per-phase times (forward
inference, forward training, backward), the whole-step HBM /
NVLink roofline of SURVEY §8(d) and the dominant kernel's roofline.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "4D FNO layer grid-pts·ch/s fwd+bwd at 1/2/4/8 B200; % HBM/NVLink roofline"
PGRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
CONFIG_INDEX = 3            # BASELINE.json configs[2] (c3, the metric's shape); --config selects another
STRONG = {"c3", "c5"}       # strong-scaled configs: the global grid is fixed (BASELINE.json)
WORKLOADS = {
    "c2": "c2: 4D Navier-Stokes-shaped DFNO training step (fwd+bwd), 64x64x64x32 per GPU, width 20, modes 8, "
          "4 Fourier layers, batch 1 (BASELINE.json configs[1])",
    "c3": "c3: CO2-multiphase-shaped DFNO training step (fwd+bwd), global 64x64x64x30, width 20, modes 12, "
          "4 Fourier layers, batch 1, x/y-decomposed over (1,1)/(2,1)/(2,2)/(4,2) (strong scaling; "
          "BASELINE.json configs[2], the configuration the metric is quoted on)",
    "c4": "c4: weak-scaling 4D FNO, 64x128x128x32 per GPU, width 20, modes 12, 4 Fourier layers, fwd+bwd, batch 1 "
          "(BASELINE.json configs[3])",
    "c5": "c5: largest one-box instance, global 256x256x256x32, width 20, modes 16, 4 Fourier layers, fwd+bwd, "
          "batch 1 (BASELINE.json configs[4])",
}
REF_XY_DIV = 4              # oracle sample: x/y sub-box (1/16 of the per-GPU points) at full width


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, indices, period=0.005):
        self.indices, self.period = indices, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.handles = [pynvml.nvmlDeviceGetHandleByUUID(i) if isinstance(i, str)
                            else pynvml.nvmlDeviceGetHandleByIndex(i) for i in indices]
            self.max_mhz = max(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) for h in self.handles)
        except Exception:
            self.nv = None

    def sample_once(self):
        """One SM-clock / throttle-reason reading per GPU (also called from the
        timing loop after every repetition, so short timed regions are covered
        even when the sampling thread is starved)"""
        nv = self.nv
        if nv is None:
            return
        for h in self.handles:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass

    def _run(self):
        while not self._stop.is_set():
            self.sample_once()
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def nvml_index(cuda_index):
    """NVML handle key of a CUDA device (UUID; falls back to the index)."""
    try:
        import torch
        u = str(torch.cuda.get_device_properties(cuda_index).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        return cuda_index


# ---------------------------------------------------------------------------
# roofline bookkeeping (algorithmic bytes per launch)
# ---------------------------------------------------------------------------
def stage_bytes(prob, plan_info):
    """Algorithmic HBM bytes per launch of each kernel stage (fp32 / complex64)."""
    B, C = prob["B"], prob["C"]
    Xl, Yl, Z, T = prob["local"]
    X, Y = prob["grid"][0], prob["grid"][1]
    mx, my, mz, mt = prob["modes"]
    nkz = plan_info["nkz"]
    P = prob["P"]
    n = B * C * Xl * Yl * Z * T                       # local field elements
    slab = 8 * B * C * Xl * Yl * 2 * mz * mt          # bytes of this rank's slab (send side)
    slab_kz = 8 * P * B * C * Xl * Yl * nkz * mt      # bytes of the kz-block slab (after exchange)
    M = 4 * mx * my * nkz * mt
    H = 8 * B * nkz * C * X * 2 * my * mt
    mode = 8 * B * C * M
    Rb = 8 * C * C * M
    return {
        "fwd.pass_a": 4 * n + slab,
        "fwd.b_y_fwd": slab_kz + H,
        "fwd.b_x_fwd": H + mode,
        "fwd.mix": Rb + 2 * mode,
        "fwd.b_x_inv": mode + H,
        "fwd.b_y_inv": H + slab_kz,
        "fwd.pass_c": slab + 4 * n + 4 * n + 4 * n,         # slab, v, y, z_save
        "bwd.pass_a": 12 * n + slab,                         # dy, z -> slab, dz
        "bwd.b_y_fwd": slab_kz + H,
        "bwd.b_x_fwd": H + mode,
        "bwd.mix": 2 * Rb + 3 * mode,                        # R, dR, V^, G^, W'^
        "bwd.b_x_inv": mode + H,
        "bwd.b_y_inv": H + slab_kz,
        # slab, dz, v -> dv; the split backward (pass C family 5): slab, dz -> dv,
        # then dw_partial reads dz, v (its rows are "bwd.dw")
        "bwd.pass_c": slab + 8 * n + (0 if plan_info.get("split_bwd") else 4 * n),
        "bwd.dw": 8 * n,
        "fwd.exchange_1": slab * (P - 1) / P, "fwd.exchange_2": slab * (P - 1) / P,
        "bwd.exchange_1": slab * (P - 1) / P, "bwd.exchange_2": slab * (P - 1) / P,
    }


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(config):
    """per-launch DRAM bytes of each stage from the committed `ncu --set full`
    capture of this workload (profiles/ncu_traffic.json, keyed by config)"""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(config, {})
    return {}


def step_roofline(grid, local, modes, C, B, L, P, hbm_gbs, a2a):
    """SURVEY §8(d) roofline of one training step per GPU: algorithmic bytes
    per point-channel (fp32 field, complex64 spectra; r = 2mz mt / (Z T) the
    slab fraction, rho = M / N the retained-mode fraction)
        fwd (inference) 12 + 32 r + 8 C rho      fwd (training) + 4 + 8 rho
        bwd             24 + 32 r + 16 C rho + 8 rho
    on HBM, plus 2 x 8 r (P-1)/P per layer pass on NVLink; t_roof = HBM bytes /
    BW_HBM + NVLink bytes / BW_NVL (sum: the stages are a dependency chain)
    and the max() form.  BW_NVL: the NCCL all-to-all measured here at the
    exchange message size (N > 1), 900 GB/s nominal for context."""
    X, Y, Z, T = grid
    mx, my, mz, mt = modes
    r = 2.0 * mz * mt / (Z * T)
    rho = 8.0 * mx * my * mz * mt / float(X * Y * Z * T)
    n_loc = B * C * local[2] * local[3] * local[4] * local[5]
    per = {"fwd_inference": 12 + 32 * r + 8 * C * rho,
           "fwd_train": 12 + 32 * r + 8 * C * rho + 4 + 8 * rho,
           "bwd": 24 + 32 * r + 16 * C * rho + 8 * rho}
    nvl_pass = 2 * 8 * r * (P - 1) / P
    if P > 1 and a2a:
        nvl_gbs, nvl_kind = a2a["GBps_per_gpu"], "measured NCCL all-to-all at the exchange message size"
    else:
        nvl_gbs, nvl_kind = 900.0, "nominal (no exchange at P = 1)" if P == 1 else "nominal"

    def t(hbm_b, nvl_b):
        th = hbm_b / (hbm_gbs * 1e9) * 1e3
        tn = nvl_b / (nvl_gbs * 1e9) * 1e3 if nvl_b else 0.0
        return th, tn

    out = {"bytes_per_pt_ch_per_layer": {k: round(v, 3) for k, v in per.items()},
           "nvl_bytes_per_pt_ch_per_layer_pass": round(nvl_pass, 4),
           "bw_hbm_gbs": hbm_gbs, "bw_hbm_nominal_gbs": 8000.0, "bw_nvl_gbs": round(nvl_gbs, 1),
           "bw_nvl_kind": nvl_kind, "bw_nvl_nominal_gbs": 900.0, "phases": {}}
    for name, b in per.items():
        th, tn = t(b * n_loc * L, nvl_pass * n_loc * L)
        out["phases"][name] = {"t_roof_sum_ms": round(th + tn, 4), "t_roof_max_ms": round(max(th, tn), 4)}
    hbm_step = (per["fwd_train"] + per["bwd"]) * n_loc * L
    nvl_step = 2 * nvl_pass * n_loc * L
    th, tn = t(hbm_step, nvl_step)
    out.update({"hbm_bytes": int(hbm_step), "nvl_bytes": int(nvl_step), "t_hbm_ms": round(th, 4),
                "t_nvl_ms": round(tn, 4), "t_roof_sum_ms": round(th + tn, 4), "t_roof_max_ms": round(max(th, tn), 4)})
    return out


def measure_all_to_all(per_peer_bytes, world, dev, timed):
    """NCCL all-to-all (torch.distributed, the same NVLink fabric the plan's
    communicator uses) with `per_peer_bytes` to every peer: GB/s each GPU sends."""
    import torch
    import torch.distributed as dist
    n = max(1, per_peer_bytes // 4)
    src = torch.ones(n * world, dtype=torch.float32, device=dev)
    dst = torch.empty_like(src)
    for _ in range(3):
        dist.all_to_all_single(dst, src)
    ms = statistics.median(timed(lambda: dist.all_to_all_single(dst, src), 10))
    sent = 4 * n * (world - 1)
    return {"per_peer_bytes": int(4 * n), "ms": round(ms, 4), "GBps_per_gpu": round(sent / (ms / 1e3) / 1e9, 1)}


def plan_kernels(plan):
    """Which pass C kernel family the plan selected per epilogue."""
    try:
        import paper_2204_01205_b200 as fno
        return fno.plan_pass_c_kernels(plan)
    except Exception:
        return None


def torch_cpu_context(local, modes, C, reps=1):
    """Context only: the same DFNO block, fwd + bwd by
    autograd, written with torch CPU fp32 rFFTs on all host cores -- the
    like-for-like of the paper's CPU inference (PyTorch on EPYC).
    Not the oracle, not the product path."""
    import torch
    X, Y, Z, T = local[2:]
    mx, my, mz, mt = modes
    g = torch.Generator().manual_seed(5)
    v = torch.randn((1, C, X, Y, Z, T), generator=g, requires_grad=True)
    R = torch.randn((C, C, 2 * mx, 2 * my, 2 * mz, mt), dtype=torch.complex64, generator=g, requires_grad=True)
    W = torch.randn((C, C), generator=g, requires_grad=True)
    kx = torch.cat([torch.arange(mx), torch.arange(X - mx, X)])
    ky = torch.cat([torch.arange(my), torch.arange(Y - my, Y)])
    kz = torch.cat([torch.arange(mz), torch.arange(Z - mz, Z)])

    def layer(v):
        f = torch.fft.rfftn(v, dim=(2, 3, 4, 5))[:, :, kx][:, :, :, ky][:, :, :, :, kz][..., :mt]
        w = torch.einsum("bixyzt,ioxyzt->boxyzt", f, R)
        full = torch.zeros((1, C, X, Y, Z, T // 2 + 1), dtype=torch.complex64)
        full[:, :, kx[:, None, None], ky[None, :, None], kz[None, None, :], :mt] = w
        u = torch.fft.irfftn(full, s=(X, Y, Z, T), dim=(2, 3, 4, 5))
        return torch.nn.functional.gelu(torch.einsum("oi,bixyzt->boxyzt", W, v) + u)

    layer(v).sum().backward()
    t0 = time.perf_counter()
    for _ in range(reps):
        layer(v).sum().backward()
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(v.numel() / dt, 1), "unit": "grid-pts·ch/s", "threads": torch.get_num_threads(),
            "kind": "torch CPU fp32 rFFT layer fwd+bwd (autograd), context only",
            "sample": f"one block on the per-GPU grid {list(local[2:])}, width {C}; {dt:.2f} s"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2204_01205_b200 as fno
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS[CONFIG_INDEX]
    lx, ly, Z, T = cfg["grid"]
    C, modes, L = cfg["width"], cfg["modes"], args.layers or cfg["layers"]
    B = args.batch
    px, py = PGRIDS[world]
    strong = cfg["name"] in STRONG
    grid = (lx, ly, Z, T) if strong else (lx * px, ly * py, Z, T)
    comm = fno.Comm.from_process_group() if world > 1 else None
    plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes, batch=B, pgrid=(px, py)), comm, device=dev)
    kz_lo, kz_hi = plan.owned_modes()
    local = plan.local_shape()
    # inputs (synthetic, seeded; field on device, weights from the numpy recipe)
    seed = synth.seed_for(CONFIG_INDEX, 0, salt=rank)
    v0 = synth.field_torch(local, modes, seed, cfg["shape"], device=dev)
    dy = torch.randn(local, generator=torch.Generator(device=dev).manual_seed(seed + 3), device=dev)
    Rs, Ws, bs = [], [], []
    for layer in range(L):
        s = synth.seed_for(CONFIG_INDEX, layer)
        R = synth.spectral_weights(C, C, modes, s + 1, kz_range=(kz_lo, kz_hi))
        W, b = synth.channel_weights(C, s + 2)
        Rs.append(torch.from_numpy(R).to(dev))
        Ws.append(torch.from_numpy(W).to(dev))
        bs.append(torch.from_numpy(b).to(dev))
    net = None
    if args.network:
        # whole network: input a [B][2][X][Y][Z] (permeability-, topography-like
        # channels), target y [B][1][X][Y][Z][T]; seeded, CO2-shaped
        from paper_2204_01205_b200.network import Network
        net = Network(plan, layers=L, in_channels=2, seed=CONFIG_INDEX)
        a_in = synth.field_torch((B, 2) + tuple(local[2:5]) + (1,), tuple(modes[:3]) + (1,), seed + 11, "co2",
                                 device=dev)[..., 0].contiguous()
        y_t = synth.field_torch((B, 1) + tuple(local[2:]), modes, seed + 12, "co2", device=dev)
    acts = [v0] + [torch.empty_like(v0) for _ in range(L)]
    zs = [torch.empty_like(v0) for _ in range(L)]
    vhs = [torch.empty(plan.vhat_shape(), dtype=torch.complex64, device=dev) for _ in range(L)]
    dR = [torch.empty(plan.weight_shape(), dtype=torch.complex64, device=dev) for _ in range(L)]
    dW = torch.empty((L, C, C), device=dev)
    db = torch.empty((L, C), device=dev)
    g = [dy, torch.empty_like(v0), torch.empty_like(v0)]

    def step():
        if net is not None:
            net.train_step(a_in, y_t, lr=1e-3)
            return
        for l in range(L):
            fno.layer_fwd(plan, acts[l], Rs[l], Ws[l], bs[l], acts[l + 1], zs[l], vhs[l])
        cur = 0                      # g[0] = upstream dy; dv ping-pongs between g[1], g[2]
        for l in reversed(range(L)):
            nxt = 1 if cur != 1 else 2
            fno.layer_bwd(plan, acts[l], zs[l], vhs[l], g[cur], Rs[l], Ws[l], g[nxt], dR[l], dW[l], db[l])
            cur = nxt

    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- each timed callable as one CUDA graph (layer stack; the network's
    # Adam step count lives on the host, so that mode stays eager) ------------
    use_graph = not args.no_graph and net is None
    graphs = []

    def as_graph(fn):
        if not use_graph:
            return fn, None
        g_ = torch.cuda.CUDAGraph()
        n_c = fno.kernel_launches()
        with torch.cuda.graph(g_):
            fn()
        per = fno.kernel_launches() - n_c
        g_.replay()
        barrier()
        graphs.append(g_)
        return g_.replay, per

    run, per_step = as_graph(step)

    def timed(fn, reps, sampler=None):
        """Per-repetition device times (ms): a barrier before each repetition,
        CUDA events on the launching stream, then the max over ranks."""
        ts = []
        for _ in range(reps):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            if sampler is not None:   # the GPU is still running this repetition
                sampler.sample_once()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = torch.tensor(ts, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.tolist()]

    # ---- timed region: K repetitions of the step ------------------------------
    n0 = fno.kernel_launches()
    sampler = ClockSampler([nvml_index(local_rank)])
    with sampler:
        step_ms = timed(run, args.steps, sampler)
        barrier()
    launches = per_step * args.steps if use_graph else fno.kernel_launches() - n0
    ms_step = float(statistics.median(step_ms))
    ms_mean = float(statistics.fmean(step_ms))
    units = B * grid[0] * grid[1] * grid[2] * grid[3] * C * L
    value = units / (ms_step / 1e3)

    # ---- phases (inference forward, training forward, backward) --
    phases = None
    if net is None and not args.no_phases:
        ys = [torch.empty_like(v0) for _ in range(L)]

        def fwd_infer():
            x = acts[0]
            for l in range(L):
                fno.layer_fwd(plan, x, Rs[l], Ws[l], bs[l], ys[l])
                x = ys[l]

        def fwd_train():
            for l in range(L):
                fno.layer_fwd(plan, acts[l], Rs[l], Ws[l], bs[l], acts[l + 1], zs[l], vhs[l])

        def bwd_only():
            cur = 0
            for l in reversed(range(L)):
                nxt = 1 if cur != 1 else 2
                fno.layer_bwd(plan, acts[l], zs[l], vhs[l], g[cur], Rs[l], Ws[l], g[nxt], dR[l], dW[l], db[l])
                cur = nxt

        phases = {}
        nrep = max(5, min(args.steps, 20))
        for name, fn in (("fwd_inference", fwd_infer), ("fwd_train", fwd_train), ("bwd", bwd_only)):
            fn()
            barrier()
            r_, _ = as_graph(fn)
            ms_ = float(statistics.median(timed(r_, nrep)))
            phases[name] = {"ms": round(ms_, 4), "value": round(units / (ms_ / 1e3), 1),
                            "ms_per_layer": round(ms_ / L, 4)}
        del ys

    # per-stage CUDA events (library profiling hooks) on separate eager steps
    nprof = max(2, min(args.steps, 5))
    plan.profile_enable(True)
    plan.profile_read()
    for _ in range(nprof):
        step()
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile_enable(False)

    # NCCL all-to-all bandwidth at this config's exchange message size (BW_NVL of
    # the SURVEY §8(d) roofline): bytes each GPU sends / device time, median
    a2a = None
    if world > 1:
        per_peer = 8 * B * C * local[2] * local[3] * max(kz_hi - kz_lo, 1) * modes[3]
        a2a = measure_all_to_all(per_peer, world, dev, timed)
    # ---- end to end: pinned host inputs -> device, step, result -> host -------
    res = torch.empty((L, C * C + C), device=dev)
    if net is None:         # layer stack: the field v and the cotangent dy in, dW / db out
        h_v = torch.empty(local, dtype=torch.float32, pin_memory=True)
        h_dy = torch.empty(local, dtype=torch.float32, pin_memory=True)
        h_v.copy_(v0.cpu())
        h_dy.copy_(dy.cpu())
        h_out = torch.empty((L, C * C + C), dtype=torch.float32, pin_memory=True)
    else:                   # network: input a and target y in, the loss out
        h_v = torch.empty(a_in.shape, dtype=torch.float32, pin_memory=True)
        h_dy = torch.empty(y_t.shape, dtype=torch.float32, pin_memory=True)
        h_v.copy_(a_in.cpu())
        h_dy.copy_(y_t.cpu())
        h_out = torch.empty(3, dtype=torch.float32, pin_memory=True)

    def e2e_step():
        if net is not None:
            a_in.copy_(h_v, non_blocking=True)
            y_t.copy_(h_dy, non_blocking=True)
            h_out.copy_(net.train_step(a_in, y_t, lr=1e-3), non_blocking=True)
            return
        acts[0].copy_(h_v, non_blocking=True)
        g[0].copy_(h_dy, non_blocking=True)
        step()
        res[:, :C * C].copy_(dW.view(L, C * C))
        res[:, C * C:].copy_(db)
        h_out.copy_(res, non_blocking=True)

    # layer stack: the next step's inputs are copied on a second stream while the
    # current step computes (two device input slots); each step still moves its
    # own inputs host -> device and its result device -> host
    cstream = torch.cuda.Stream(device=dev)
    vslot = [acts[0], torch.empty_like(acts[0])]
    dyslot = [g[0], torch.empty_like(g[0])]
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    used = [False, False]

    def prefetch(slot):
        with torch.cuda.stream(cstream):
            if used[slot]:
                cstream.wait_event(consumed[slot])
            vslot[slot].copy_(h_v, non_blocking=True)
            dyslot[slot].copy_(h_dy, non_blocking=True)
            copied[slot].record(cstream)

    def run_e2e(n, start_event=None):
        if net is not None:
            for _ in range(n):
                e2e_step()
            return
        if start_event is not None:
            cstream.wait_event(start_event)
        prefetch(0)
        for i in range(n):
            s = i % 2
            if i + 1 < n:
                prefetch(1 - s)
            stream.wait_event(copied[s])
            acts[0], g[0] = vslot[s], dyslot[s]
            step()
            consumed[s].record(stream)
            used[s] = True
            res[:, :C * C].copy_(dW.view(L, C * C))
            res[:, C * C:].copy_(db)
            h_out.copy_(res, non_blocking=True)

    run_e2e(max(2, args.warmup))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run_e2e(args.steps, e0)
    e1.record(stream)
    e1.synchronize()
    cstream.synchronize()
    t2 = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_ms = float(t2.item()) / args.steps
    e2e_value = units / (e2e_ms / 1e3)

    # ---- roofline of the dominant kernel -----------------------------------
    info = dict(nkz=kz_hi - kz_lo, split_bwd=plan_kernels(plan).get("bwd", {}).get("family", "").startswith("split"))
    prob = dict(B=B, C=C, local=local[2:], grid=grid, modes=modes, P=world)
    sb = stage_bytes(prob, info)
    kern = {k: v for k, v in prof.items() if "exchange" not in k and k in sb}
    dom = max(kern, key=lambda k: kern[k][0]) if kern else None
    peak, peak_kind = load_peaks()
    roof = None
    if dom:
        tot_ms, cnt = kern[dom]
        avg_s = tot_ms / cnt / 1e3
        ach = sb[dom] / avg_s / 1e9
        traffic = load_traffic(cfg["name"]).get(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic, "algorithmic_bytes": int(sb[dom]), "avg_launch_us": round(avg_s * 1e6, 2),
                "share_of_step": round(tot_ms / max(sum(v[0] for v in prof.values()), 1e-9), 4)}
    stages = {k: {"ms_per_step": round(v[0] / nprof, 4), "launches_per_step": v[1] / nprof,
                  "GBps": (round(sb[k] / (v[0] / v[1] / 1e3) / 1e9, 1) if k in sb else None)}
              for k, v in sorted(prof.items())}

    # ---- whole-step roofline (algorithmic HBM + NVLink bytes) ---
    step_roof = step_roofline(grid, local, modes, C, B, L, world, peak, a2a)
    step_roof["t_measured_ms"] = round(ms_step, 4)
    step_roof["frac_sum"] = round(step_roof["t_roof_sum_ms"] / ms_step, 4)
    step_roof["frac_max"] = round(step_roof["t_roof_max_ms"] / ms_step, 4)
    if phases:
        for name, ph in phases.items():
            ph["t_roof_ms"] = step_roof["phases"][name]["t_roof_sum_ms"]
            ph["frac"] = round(ph["t_roof_ms"] / ph["ms"], 4)

    # ---- CPU baselines: the oracle on a bounded sample (rank 0, N=1 only) -----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and net is None:
        cpu = oracle_sample(args, v0.detach().cpu().numpy(), dy.detach().cpu().numpy(), modes, repeats=1)
        cpu["context_torch_cpu"] = torch_cpu_context(local, modes, C)

    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "grid-pts·ch/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "ms_per_step_mean": round(ms_mean, 4), "timing": "median of K repetitions, a barrier before each, "
                                                          "CUDA events, max over ranks",
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded {'CO2' if cfg['shape'] == 'co2' else 'NS'}-shaped fields, random-init weights)",
        "config": {"workload": (WORKLOADS[cfg["name"]] if net is None else
                                f"{cfg['name']}-net: whole DFNO training step (lift 2->{C} channels and 1->{T} "
                                f"time steps, {L} blocks, projection {C}->1, relative-L2 loss, backward, Adam; "
                                f"SURVEY 8.f N1) on the {cfg['name']} grid"),
                   "global_grid": list(grid), "pgrid": [px, py], "batch": B, "width": C, "modes": list(modes),
                   "layers": L, "parallelism": f"x/y domain decomposition {px}x{py}",
                   "launch": "one CUDA graph per step (replayed)" if use_graph else "eager",
                   "l2": f"inputs larger than L2 ({B * C * int(np.prod(local[2:])) * 4 / 1e6:.0f} MB field per "
                         f"layer per GPU; L2 126 MB)",
                   "env": {k: v for k, v in sorted(os.environ.items()) if k.startswith("FNO_")},
                   "pass_c": plan_kernels(plan)},
        "e2e": {"value": round(e2e_value, 1), "unit": "grid-pts·ch/s", "ms_per_step": round(e2e_ms, 4),
                "overlap": ("the next step's pinned-host inputs are copied on a second stream while the current step "
                            "computes (two device input slots)" if net is None else "none"),
                "h2d_bytes_per_step": int(h_v.numel() * 4 + h_dy.numel() * 4),
                "d2h_bytes_per_step": int(h_out.numel() * 4)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "step_roofline": step_roof,
        "phases": phases,
        "nccl_all_to_all": a2a,
        "stages": stages,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if graphs:
        torch.cuda.synchronize()
        for g_ in graphs:      # release the captured NCCL / peer-exchange work before the communicator
            g_.reset()
        graphs.clear()
    if world > 1:
        dist.barrier()
    plan.destroy()
    if comm:
        comm.destroy()


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        return {"blas": [(d.get("internal_api"), d.get("num_threads")) for d in info]}
    except Exception as e:       # noqa: BLE001
        return {"blas": f"unknown ({e})"}


def oracle_sample(args, v, dy, modes, repeats=1):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    one DFNO block forward + backward (oracle.spectral.layer_fwd + layer_bwd) at
    the full width of the config, on an x/y sub-box of the per-GPU grid (full
    z, t and modes; REF_XY_DIV along x and y, so the run stays ~10-30 s of
    host time).  Returns the cpu_baseline object (grid-pts·ch/s)."""
    import numpy as np

    import synth
    from oracle import spectral as sp
    B, C, X, Y, Z, T = v.shape
    xs, ys = max(2 * modes[0], X // REF_XY_DIV), max(2 * modes[1], Y // REF_XY_DIV)
    vs = np.asarray(v[:, :, :xs, :ys], dtype=np.float64)
    dys = np.asarray(dy[:, :, :xs, :ys], dtype=np.float64)
    s = synth.seed_for(CONFIG_INDEX, 0)
    R = synth.spectral_weights(C, C, modes, s + 1).astype(np.complex128)
    W, b = synth.channel_weights(C, s + 2)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        sp.layer_fwd(vs, R, W.astype(np.float64), b.astype(np.float64), modes)
        sp.layer_bwd(vs, dys, R, W.astype(np.float64), b.astype(np.float64), modes)
        times.append(time.perf_counter() - t0)
    t = min(times)
    units = vs.size          # grid points x channels of one layer, fwd+bwd
    cores = len(os.sched_getaffinity(0))
    return {"value": round(units / t, 1), "unit": "grid-pts·ch/s", "cores": cores, "kind": "oracle",
            "threads": _blas_threads(),
            "sample": f"one DFNO block fwd+bwd (oracle.spectral.layer_fwd + layer_bwd, fp64 numpy, naive DFT "
                      f"matrices) at full width {C} and modes {list(modes)} on the x/y sub-box "
                      f"{[xs, ys, Z, T]} of the per-GPU grid {[X, Y, Z, T]}, batch {B}; {t:.2f} s wall",
            "seconds": round(t, 3)}


# ---------------------------------------------------------------------------
# reference arm: the oracle on the host cores (rank 0 only)
# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """The reference arm of this tier: the fp64 oracle (as it stands) on the
    box's host cores, each step one bounded sample of our arm's workload (one
    DFNO block fwd+bwd at full width on an x/y sub-box, oracle_sample); rank 0
    only, the other ranks exit without work."""
    if rank != 0:
        return
    import numpy as np

    import synth
    cfg = synth.CONFIGS[CONFIG_INDEX]
    lx, ly, Z, T = cfg["grid"]
    if cfg["name"] in STRONG and world in PGRIDS:     # our arm's per-GPU box at this N
        lx, ly = lx // PGRIDS[world][0], ly // PGRIDS[world][1]
    modes, C = cfg["modes"], cfg["width"]
    xs, ys = max(2 * modes[0], lx // REF_XY_DIV), max(2 * modes[1], ly // REF_XY_DIV)
    shape = (1, C, xs, ys, Z, T)
    s = synth.seed_for(CONFIG_INDEX, 0)
    v = synth.field(shape, modes, s, cfg["shape"], n_waves=4).astype(np.float32)
    dy = synth.cotangent(shape, s + 3).astype(np.float32)
    for _ in range(args.warmup):
        oracle_sample(args, v, dy, modes)
    t0 = time.perf_counter()
    res = [oracle_sample(args, v, dy, modes) for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    units = float(np.prod(shape))
    value = units * args.steps / wall
    cpu = dict(res[0])
    cpu["value"] = round(value, 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "grid-pts·ch/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * wall / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if cfg["name"] in STRONG else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (seeded {'CO2' if cfg['shape'] == 'co2' else 'NS'}-shaped fields, random-init weights)",
        "config": {"workload": WORKLOADS[cfg["name"]] + f"; oracle sample per step: one DFNO block fwd+bwd at width "
                               f"{C} on an x/y box {[xs, ys, Z, T]} (per-GPU grid {[lx, ly, Z, T]}; the box is at "
                               f"least 2m wide, the oracle's retained-mode limit)",
                   "global_grid": list(cfg["grid"]), "sample_grid": [xs, ys, Z, T], "width": C,
                   "modes": list(modes), "batch": 1},
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 1), "unit": "grid-pts·ch/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps eagerly instead of as a CUDA graph")
    ap.add_argument("--network", action="store_true",
                    help="time the whole network's training step (lift, blocks, projection, loss, backward, Adam)")
    ap.add_argument("--config", choices=["c2", "c3", "c4", "c5"], default="c3",
                    help="BASELINE.json workload (default c3 = configs[2], strong; c2 configs[1]; c4 weak; c5 strong)")
    ap.add_argument("--allow-dev", action="store_true", help="allow FNO_LIB / FNO_ABLATE development builds (A/B only)")
    ap.add_argument("--no-phases", action="store_true", help="skip the per-phase (fwd inference / fwd train / bwd) timing")
    args = ap.parse_args()
    global CONFIG_INDEX
    CONFIG_INDEX = int(args.config[1])
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torch.distributed.run",
              file=sys.stderr)
        if world == 1:
            args.gpus = 1
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if (os.environ.get("FNO_ABLATE") or os.environ.get("FNO_LIB")) and not args.allow_dev:
        raise SystemExit("bench.py: FNO_ABLATE / FNO_LIB select development builds; unset them for a bench line "
                         "(--allow-dev for A/B runs; the FNO_* environment is recorded in config.env)")
    if world not in PGRIDS:
        raise SystemExit(f"unsupported world size {world} (1, 2, 4, 8)")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
