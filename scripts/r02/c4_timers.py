"""pass_c4 role timers (FNO_C4_PROFILE variant library via FNO_LIB): one layer
forward at a config; prints mean cycles per tile per role."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2204_01205_b200 as fno  # noqa: E402
import synth  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.CONFIGS[ci]
grid, C, modes = cfg["grid"], cfg["width"], cfg["modes"]
plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=modes))
print(fno.plan_pass_c_kernels(plan))
v = synth.field_torch(plan.local_shape(), modes, 1, cfg["shape"])
R = torch.from_numpy(synth.spectral_weights(C, C, modes, 2)).cuda()
W, b = [torch.from_numpy(a).cuda() for a in synth.channel_weights(C, 3)]
y, z = torch.empty_like(v), torch.empty_like(v)
vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device="cuda")
mode = sys.argv[2] if len(sys.argv) > 2 else "fwd"
if mode == "dv":   # the split backward's dv leg: the forward pass_c4 with W^T
    fno.plan_set_pass_c(plan, "fwd", 4)
    fno.plan_set_pass_c(plan, "bwd", 5)
else:
    fno.plan_set_pass_c(plan, mode, 4)
for _ in range(3):
    fno.layer_fwd(plan, v, R, W, b, y, z, vh)
if mode in ("bwd", "dv"):
    dv = torch.empty_like(v)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    for _ in range(3):
        fno.layer_bwd(plan, v, z, vh, torch.randn_like(v), R, W, dv, dR, dW, db)
torch.cuda.synchronize()
L = fno.lib()
L.fno_debug_c4_timers.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
n = 148 * 16
buf = (ctypes.c_ulonglong * n)()
assert L.fno_debug_c4_timers(plan.handle, buf, n) == 0
a = np.array(buf, dtype=np.float64).reshape(148, 16)
X, Y, Z, T = grid
tiles = X * Y * (Z // 16) * ((T + 7) // 8) / 148 if ci != 5 else 1
names = ["prod.wait_xempty", "mma.wait_opfull", "mma.wait_dempty", "epi.split_wait", "epi.split_work",
         "epi.wait_ufull", "epi.wait_dfull", "epi.epilogue_total", "tr.phase1", "tr.wait_uempty", "tr.phase2_total",
         "epi.total"]
print(f"tiles per CTA ~{tiles:.0f}")
for i, nm in enumerate(names):
    print(f"{nm:22s} {a[:, i].mean() / tiles:10.0f} cycles/tile   total {a[:, i].mean() / 1965:10.1f} us")
