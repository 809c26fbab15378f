"""A/B of pass C kernel families on the layer forward / backward at a config (CUDA events, median of 10)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2204_01205_b200 as fno  # noqa: E402
import synth  # noqa: E402

ci = int(sys.argv[1])
cfg = synth.CONFIGS[ci]
grid, C, modes = cfg["grid"], cfg["width"], cfg["modes"]
plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes))
v = synth.field_torch(plan.local_shape(), modes, 1, cfg["shape"])
R = torch.from_numpy(synth.spectral_weights(C, C, modes, 2)).cuda()
W, b = [torch.from_numpy(a).cuda() for a in synth.channel_weights(C, 3)]
y, z = torch.empty_like(v), torch.empty_like(v)
vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device="cuda")
dy = torch.randn_like(v)
dv = torch.empty_like(v)
dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
dW = torch.empty((C, C), device="cuda")
db = torch.empty((C,), device="cuda")


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for mode in ("fwd", "bwd"):
    for fam in ((2, 3, 4) if mode == "fwd" else (2, 4, 5)):
        try:
            fno.plan_set_pass_c(plan, mode, fam)
        except fno.FnoError:
            continue
        plan.profile_enable(True)
        plan.profile_read()
        if mode == "fwd":
            t = timeit(lambda: fno.layer_fwd(plan, v, R, W, b, y, z, vh))
        else:
            t = timeit(lambda: fno.layer_bwd(plan, v, z, vh, dy, R, W, dv, dR, dW, db))
        pr = plan.profile_read()
        plan.profile_enable(False)
        k = f"{mode}.pass_c"
        extra = ""
        if mode == "bwd" and fam == 5 and "bwd.dw" in pr:
            extra = f", dw_partial {pr['bwd.dw'][0] / pr['bwd.dw'][1]:.3f} ms/launch"
        print(f"c{ci} {mode} family {fam}: layer {t:.3f} ms, pass C {pr[k][0] / pr[k][1]:.3f} ms/launch{extra}")
