"""Small layer fwd + bwd through libfno (for compute-sanitizer / debugging)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2204_01205_b200 as fno
import synth
grid = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,16,64,32").split(","))
C = int(sys.argv[2]) if len(sys.argv) > 2 else 20
m = tuple(int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "8,8,8,8").split(","))
plan = fno.Plan(fno.Problem(grid=grid, width=C, modes=m))
print(fno.plan_pass_c_kernels(plan), flush=True)
v = synth.field_torch(plan.local_shape(), m, 1)
R = torch.from_numpy(synth.spectral_weights(C, C, m, 2)).cuda()
W, b = [torch.from_numpy(a).cuda() for a in synth.channel_weights(C, 3)]
y, z = torch.empty_like(v), torch.empty_like(v)
vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device="cuda")
fno.layer_fwd(plan, v, R, W, b, y, z, vh)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dv = torch.empty_like(v)
dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
dW = torch.empty((C, C), device="cuda"); db = torch.empty((C,), device="cuda")
fno.layer_bwd(plan, v, z, vh, torch.randn_like(v), R, W, dv, dR, dW, db)
torch.cuda.synchronize()
print("bwd ok", float(dW.abs().sum()), flush=True)
