"""GPU parity: libfno's sm_100a path vs the fp64 oracle on the same seeded fp32
inputs.  Bar (north star, BASELINE.json): relative L2 <= 1e-5 for the fp32 path
on u, y, z, V^, dv, dR, dW, db."""

import numpy as np
import pytest

import synth
from oracle import spectral as sp
from tests._instances import rel_l2, worked_example

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_01205_b200 import build
    build.build()


def _problem(grid, C, modes, B=1, seed=0, shape="ns"):
    v = synth.field((B, C) + tuple(grid), modes, seed, shape)
    R = synth.spectral_weights(C, C, modes, seed + 1)
    W, b = synth.channel_weights(C, seed + 2)
    dy = synth.cotangent(v.shape, seed + 3)
    return v, R, W, b, dy


# (grid, C, modes, B): c1 itself plus every instantiated (LZ, LT) pair, shrunk in x/y
CASES = [
    ((16, 16, 16, 8), 4, (4, 4, 4, 4), 1),        # c1 (BASELINE configs[0])
    ((32, 16, 64, 32), 20, (8, 8, 8, 8), 1),      # c2 shape class, x/y shrunk
    ((32, 32, 64, 30), 6, (12, 12, 12, 12), 1),   # c3 shape class (T=30, 2mz does not divide Z)
    ((32, 32, 128, 32), 4, (12, 12, 12, 12), 1),  # c4 shape class
    ((32, 32, 256, 32), 2, (16, 16, 16, 16), 1),  # c5 shape class
    ((12, 10, 12, 10), 3, (3, 2, 3, 3), 2),       # odd sizes, C % 4 != 0, batch 2
    ((8, 8, 8, 8), 5, (4, 4, 4, 5), 1),           # full pass incl. Nyquist kt = T/2
    ((16, 8, 16, 8), 2, (2, 2, 4, 4), 3),         # (LZ, LT) = (8, 8), ragged batch of 3
]


def _ids(c):
    return "x".join(map(str, c[0])) + f"_C{c[1]}_m{'-'.join(map(str, c[2]))}_B{c[3]}"


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_layer_forward_matches_oracle(case):
    from tests import _gpu as G
    grid, C, modes, B = case
    v, R, W, b, _ = _problem(grid, C, modes, B, seed=101)
    plan = G.make_plan(grid, C, modes, B)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    y_ref, z_ref = sp.layer_fwd(G.f32(v), G.f32(R), G.f32(W), G.f32(b), modes)
    vh_ref = sp.forward_modes(G.f32(v), modes)
    assert rel_l2(G.np64(vh), vh_ref) < TOL
    assert rel_l2(G.np64(z), z_ref) < TOL
    assert rel_l2(G.np64(y), y_ref) < TOL


@pytest.mark.parametrize("case", CASES[:3] + CASES[5:], ids=_ids)
def test_spectral_conv_forward_and_adjoint(case):
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, C, modes, B = case
    v, R, W, b, g = _problem(grid, C, modes, B, seed=202)
    plan = G.make_plan(grid, C, modes, B)
    u, vh = G.spectral_fwd(plan, v, R)
    u_ref = sp.spectral_conv(G.f32(v), G.f32(R), modes)
    assert rel_l2(G.np64(u), u_ref) < TOL
    gt = G.t32(g)
    dv = torch.empty_like(gt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    fno.spectral_conv_bwd(plan, gt, G.tc64(R), vh, dv, dR)
    torch.cuda.synchronize()
    dv_ref = sp.spectral_conv_adjoint(G.f32(g), G.f32(R), modes)
    assert rel_l2(G.np64(dv), dv_ref) < TOL
    _, dR_ref, _, _ = sp.layer_bwd(G.f32(v), G.f32(g), G.f32(R), 0 * G.f32(W), None, modes, act="none")
    assert rel_l2(G.np64(dR), dR_ref) < TOL
    # adjoint identity on the GPU results (pin P9, fp32)
    lhs = float(np.sum(G.np64(u) * G.f32(g)))
    rhs = float(np.sum(G.f32(v) * G.np64(dv)))
    assert abs(lhs - rhs) / (np.linalg.norm(G.np64(u)) * np.linalg.norm(g)) < 1e-6


@pytest.mark.parametrize("case", CASES, ids=_ids)
@pytest.mark.parametrize("act", ["gelu", "none"])
def test_layer_backward_matches_oracle(case, act):
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, C, modes, B = case
    if act == "none" and case not in (CASES[0], CASES[5]):
        pytest.skip("act=none covered on two shapes")
    v, R, W, b, dy = _problem(grid, C, modes, B, seed=303)
    plan = G.make_plan(grid, C, modes, B, act=act)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), dtype=torch.float32, device="cuda")
    db = torch.empty((C,), dtype=torch.float32, device="cuda")
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    torch.cuda.synchronize()
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(G.f32(v), G.f32(dy), G.f32(R), G.f32(W), G.f32(b), modes, act=act)
    assert rel_l2(G.np64(dv), dv_r) < TOL
    assert rel_l2(G.np64(dR), dR_r) < TOL
    assert rel_l2(G.np64(dW), dW_r) < TOL
    assert rel_l2(G.np64(db), db_r) < TOL
    # accumulate = 1 adds into dR, dW, db
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db, accumulate=True)
    torch.cuda.synchronize()
    assert rel_l2(G.np64(dR), 2 * dR_r) < TOL
    assert rel_l2(G.np64(dW), 2 * dW_r) < TOL
    assert rel_l2(G.np64(db), 2 * db_r) < TOL


def test_golden_worked_example_on_gpu():
    from tests import _gpu as G
    ex = worked_example()
    plan = G.make_plan(ex["grid"], 2, ex["modes"])
    u, _ = G.spectral_fwd(plan, ex["v"], ex["R"])
    y, _, _ = G.layer_fwd(plan, ex["v"], ex["R"], ex["W"], ex["b"])
    u = G.np64(u)[0]
    y = G.np64(y)[0]
    e = ex["expected"]
    assert abs(u.sum() - e["sum_u"]) < 1e-4
    assert abs((u ** 2).sum() - e["sum_u2"]) / e["sum_u2"] < 1e-5
    assert abs(u[0, 0, 0, 0, 0] - e["u[0,0,0,0,0]"]) < 1e-5
    assert abs(u[1, 1, 2, 3, 1] - e["u[1,1,2,3,1]"]) < 1e-5
    assert abs(y.sum() - e["sum_y"]) / abs(e["sum_y"]) < 1e-5
    assert abs(y[1, 3, 0, 2, 2] - e["y[1,3,0,2,2]"]) < 1e-5


def test_identity_weights_full_pass_is_identity_on_gpu():
    """Pin P6 on the GPU: m = n/2, mt = T/2 + 1, R = I per mode -> S v = v."""
    from tests import _gpu as G
    grid, C, modes = (8, 8, 8, 8), 3, (4, 4, 4, 5)
    v, _, _, _, _ = _problem(grid, C, modes, 1, seed=404)
    R = np.zeros((C, C, 8, 8, 8, 5), dtype=np.complex64)
    for i in range(C):
        R[i, i] = 1.0
    plan = G.make_plan(grid, C, modes)
    u, _ = G.spectral_fwd(plan, v, R)
    assert rel_l2(G.np64(u), G.f32(v)) < TOL


def test_zero_weights_give_gelu_of_zero():
    from tests import _gpu as G
    grid, C, modes = (16, 16, 16, 8), 4, (4, 4, 4, 4)
    v, R, W, b, _ = _problem(grid, C, modes, 1, seed=505)
    plan = G.make_plan(grid, C, modes)
    y, _, _ = G.layer_fwd(plan, v, 0 * R, 0 * W, 0 * b)
    assert float(np.max(np.abs(G.np64(y)))) == 0.0


@pytest.mark.slow
def test_full_size_c2_sampled_outputs():
    """BASELINE configs[1] at full size (64^3 x 32, C=20, m=8), the launch
    configuration bench.py times; the oracle evaluates 512 sampled points."""
    import torch
    from tests import _gpu as G
    cfg = synth.CONFIGS[2]
    grid, C, modes = cfg["grid"], cfg["width"], cfg["modes"]
    pr = synth.problem(2, with_dy=False)
    plan = G.make_plan(grid, C, modes)
    y, z, vh = G.layer_fwd(plan, pr["v"], pr["R"], pr["W"], pr["b"])
    v64 = G.f32(pr["v"])
    vh_ref = sp.forward_modes(v64, modes)
    assert rel_l2(G.np64(vh), vh_ref) < TOL
    what = sp.mix(vh_ref, G.f32(pr["R"]))
    rng = np.random.default_rng(7)
    pts = np.stack([rng.integers(0, n, size=512) for n in grid], -1)
    u_s = sp.inverse_modes_at(what, grid, pts)[0]                      # [C, P]
    vs = v64[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]          # [C, P]
    z_ref = G.f32(pr["W"]) @ vs + G.f32(pr["b"])[:, None] + u_s
    zg = G.np64(z)[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    yg = G.np64(y)[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    assert rel_l2(zg, z_ref) < TOL
    assert rel_l2(yg, sp.gelu(z_ref)) < TOL
    del y, z, vh
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("ci", [3, 4], ids=["c3", "c4"])
def test_full_size_c3_c4_forward_sampled_outputs(ci):
    """BASELINE configs[2] (64^3 x 30, m=12: the cp.async / T=30 path) and
    configs[3] per-GPU box (64x128x128x32, m=12) at full size; the oracle's V^ in
    full and y, z at 512 sampled points."""
    import torch
    from tests import _gpu as G
    cfg = synth.CONFIGS[ci]
    grid, C, modes = cfg["grid"], cfg["width"], cfg["modes"]
    pr = synth.problem(ci, with_dy=False)
    plan = G.make_plan(grid, C, modes)
    y, z, vh = G.layer_fwd(plan, pr["v"], pr["R"], pr["W"], pr["b"])
    v64 = G.f32(pr["v"])
    vh_ref = sp.forward_modes(v64, modes)
    assert rel_l2(G.np64(vh), vh_ref) < TOL
    what = sp.mix(vh_ref, G.f32(pr["R"]))
    rng = np.random.default_rng(ci)
    pts = np.stack([rng.integers(0, n, size=512) for n in grid], -1)
    u_s = sp.inverse_modes_at(what, grid, pts)[0]
    vs = v64[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    z_ref = G.f32(pr["W"]) @ vs + G.f32(pr["b"])[:, None] + u_s
    zg = G.np64(z)[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    yg = G.np64(y)[0][:, pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]]
    assert rel_l2(zg, z_ref) < TOL
    assert rel_l2(yg, sp.gelu(z_ref)) < TOL
    del y, z, vh
    torch.cuda.empty_cache()


def _backward_vs_oracle(grid, C, modes, pr, seed_pts, n_pts=512):
    """Layer fwd + bwd through libfno on pr's inputs; the oracle forms z, dz on
    the whole grid, then dR, dW, db in full and dv at n_pts sampled points
    (dv = W^T dz + S^T dz with S^T by R^H, reading of P:74)."""
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    plan = G.make_plan(grid, C, modes)
    vt, Rt, Wt, bt = G.t32(pr["v"]), G.tc64(pr["R"]), G.t32(pr["W"]), G.t32(pr["b"])
    y = torch.empty_like(vt)
    z = torch.empty_like(vt)
    vh = torch.empty(plan.vhat_shape(), dtype=torch.complex64, device="cuda")
    fno.layer_fwd(plan, vt, Rt, Wt, bt, y, z, vh)
    dv = torch.empty_like(vt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.layer_bwd(plan, vt, z, vh, G.t32(pr["dy"]), Rt, Wt, dv, dR, dW, db)
    torch.cuda.synchronize()
    del y, z, vh
    v64, R64, W64, b64, dy64 = G.f32(pr["v"]), G.f32(pr["R"]), G.f32(pr["W"]), G.f32(pr["b"]), G.f32(pr["dy"])
    _, z_ref = sp.layer_fwd(v64, R64, W64, b64, modes)
    dz = dy64 * sp.gelu_prime(z_ref)
    del z_ref
    vh_ref = sp.forward_modes(v64, modes)
    gh = sp.forward_modes(dz, modes)
    X, Y, Z, T = grid
    cw = sp.c_weight(T, modes[3])
    dR_ref = np.einsum("bixyzt,boxyzt->ioxyzt", np.conj(vh_ref), gh) * (cw / float(X * Y * Z * T))
    errs = {"dR": rel_l2(G.np64(dR), dR_ref)}
    errs["dW"] = rel_l2(G.np64(dW), np.einsum("boxyzt,bixyzt->oi", dz, v64))
    errs["db"] = rel_l2(G.np64(db), dz.sum(axis=(0, 2, 3, 4, 5)))
    RH = np.conj(np.swapaxes(R64, 0, 1))
    wh = sp.mix(gh, RH)
    rng = np.random.default_rng(seed_pts)
    pts = np.stack([rng.integers(0, n, size=n_pts) for n in grid], -1)
    sel = (slice(None), pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3])          # [C, P] of batch 0
    dv_ref = W64.T @ dz[0][sel] + sp.inverse_modes_at(wh, grid, pts)[0]
    errs["dv"] = rel_l2(G.np64(dv)[0][sel], dv_ref)
    del dv, dR
    torch.cuda.empty_cache()
    bad = {k: e for k, e in errs.items() if not e < TOL}
    assert not bad, errs


@pytest.mark.slow
@pytest.mark.parametrize("ci", [2, 3], ids=["c2", "c3"])
def test_full_size_backward(ci):
    """BASELINE configs[1] (c2) and configs[2] (c3, the metric's training-step
    shape: 64^3 x 30, width 20, modes 12) backward at full size, in the launch
    configuration bench.py times."""
    cfg = synth.CONFIGS[ci]
    _backward_vs_oracle(cfg["grid"], cfg["width"], cfg["modes"], synth.problem(ci, with_dy=True), seed_pts=11 + ci)


# Width-20 backward instantiations of the other configs.  The pass-C kernels
# are specialised on (LZ, LT, CP) -- fixed by Z, T, modes and C -- and launched
# on min(columns, 2 x 148) persistent CTAs; with >= 1024 x/y columns the launch
# (grid, shared memory, tile buffers) equals the full-size one, so these x/y-
# reduced boxes run exactly the c4 / c5 kernels and launch configurations at a
# size the fp64 oracle affords in full.  Plus the odd-T ragged-tile path
# (T = 15: the 4-row TMA group view, tma_g = 4).
INSTANCES = [
    ("c4_box", (32, 32, 128, 32), 20, (12, 12, 12, 12), "ns"),     # c4: LZ 16, LT 32, CP 20
    ("c5_box", (32, 32, 256, 32), 20, (16, 16, 16, 16), "ns"),     # c5: LZ 32, LT 32, CP 20
    ("oddT", (32, 32, 32, 15), 20, (8, 8, 8, 6), "co2"),           # T odd: tma_g = 4, ragged chunks
    ("oddT_c8", (16, 32, 64, 15), 8, (6, 6, 12, 8), "ns"),         # T odd, LT = 15, CP 8
]


@pytest.mark.slow
@pytest.mark.parametrize("inst", INSTANCES, ids=lambda c: c[0])
def test_width20_instantiations_fwd_bwd(inst):
    from tests import _gpu as G
    name, grid, C, modes, shape = inst
    v = synth.field((1, C) + grid, modes, 1234, shape)
    R = synth.spectral_weights(C, C, modes, 1235)
    W, b = synth.channel_weights(C, 1236)
    dy = synth.cotangent(v.shape, 1237)
    plan = G.make_plan(grid, C, modes)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    y_ref, z_ref = sp.layer_fwd(G.f32(v), G.f32(R), G.f32(W), G.f32(b), modes)
    assert rel_l2(G.np64(z), z_ref) < TOL
    assert rel_l2(G.np64(y), y_ref) < TOL
    _backward_vs_oracle(grid, C, modes, dict(v=v, R=R, W=W, b=b, dy=dy), seed_pts=5)


@pytest.mark.parametrize("C", [24, 32], ids=["C24", "C32"])
def test_wide_channels_fwd_bwd(C):
    """Widths above 20 (the network accepts C <= 32): layer forward and backward
    vs the oracle."""
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, modes = (16, 16, 32, 16), (4, 4, 6, 6)
    v, R, W, b, dy = _problem(grid, C, modes, 1, seed=606)
    plan = G.make_plan(grid, C, modes)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    y_ref, z_ref = sp.layer_fwd(G.f32(v), G.f32(R), G.f32(W), G.f32(b), modes)
    assert rel_l2(G.np64(y), y_ref) < TOL
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    torch.cuda.synchronize()
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(G.f32(v), G.f32(dy), G.f32(R), G.f32(W), G.f32(b), modes)
    for name, got, ref in (("dv", dv, dv_r), ("dR", dR, dR_r), ("dW", dW, dW_r), ("db", db, db_r)):
        assert rel_l2(G.np64(got), ref) < TOL, name


# Every pass C kernel family the plan can select (fno_plan_set_pass_c), forced on
# the shapes that exercise their tile geometries: forward and backward vs the
# oracle.  Families: 2 pass_c2 (FFMA), 3 pass_c3 (tcgen05 1x1), 4 pass_c4
# (warp-specialised, TMA ring, tcgen05 1x1 / W^T dz / dW).
FAMILY_CASES = [
    ((32, 16, 64, 32), 20, (8, 8, 8, 8)),       # c2 class: T % 4 == 0, HALF (2mz = LZ)
    ((32, 32, 64, 30), 20, (12, 12, 12, 12)),   # c3 class: T = 30, row-group TMA view, ragged chunks
    ((16, 32, 32, 15), 8, (6, 6, 8, 6)),        # odd T: 4-row groups
]


@pytest.mark.parametrize("family", [2, 3, 4, 5])
@pytest.mark.parametrize("case", FAMILY_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_C{c[1]}")
def test_pass_c_families_fwd_bwd(case, family):
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, C, modes = case
    v, R, W, b, dy = _problem(grid, C, modes, 1, seed=707)
    plan = G.make_plan(grid, C, modes)
    ran = []
    for mode in ("fwd", "bwd"):
        try:
            fno.plan_set_pass_c(plan, mode, family)
            ran.append(mode)
        except fno.FnoError:
            pass
    if not ran:
        pytest.skip(f"family {family} does not cover this shape")
    assert {m: fno.plan_pass_c_kernels(plan)[m]["family"][:7] for m in ran}
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    y_ref, z_ref = sp.layer_fwd(G.f32(v), G.f32(R), G.f32(W), G.f32(b), modes)
    assert rel_l2(G.np64(z), z_ref) < TOL
    assert rel_l2(G.np64(y), y_ref) < TOL
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    torch.cuda.synchronize()
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(G.f32(v), G.f32(dy), G.f32(R), G.f32(W), G.f32(b), modes)
    for name, got, ref in (("dv", dv, dv_r), ("dR", dR, dR_r), ("dW", dW, dW_r), ("db", db, db_r)):
        assert rel_l2(G.np64(got), ref) < TOL, (name, rel_l2(G.np64(got), ref))


# The split backward (family 5) with each forward kernel as its dv leg (the
# contraction with W^T: w_t), on the FAMILY_CASES shapes plus a batch of 2, an
# odd width, and a v that is not 16-byte aligned (dw_partial's plain-load path;
# Xl Yl Z T is a multiple of 4 for every instantiated transform size, so only a
# misaligned base pointer takes it).
SPLIT_CASES = [c + (1, False) for c in FAMILY_CASES] + [
    ((16, 16, 16, 8), 6, (4, 4, 4, 4), 2, False),
    ((12, 10, 12, 10), 3, (3, 2, 3, 3), 2, True),
    ((32, 32, 64, 30), 20, (12, 12, 12, 12), 1, True),
]


@pytest.mark.parametrize("fwd_family", [2, 3, 4])
@pytest.mark.parametrize("case", SPLIT_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_C{c[1]}_B{c[3]}"
                         + ("_misaligned" if c[4] else ""))
def test_split_backward_dv_kernels(case, fwd_family):
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, C, modes, B, misalign = case
    v, R, W, b, dy = _problem(grid, C, modes, B, seed=717)
    plan = G.make_plan(grid, C, modes, B)
    try:
        fno.plan_set_pass_c(plan, "fwd", fwd_family)
        fno.plan_set_pass_c(plan, "bwd", 5)
    except fno.FnoError:
        pytest.skip(f"forward family {fwd_family} does not cover this shape")
    info = fno.plan_pass_c_kernels(plan)
    assert info["bwd"]["family"].startswith("split") and info["bwd"]["dv_kernel"] == info["fwd"]["family"]
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.full((C, C), 7.0, device="cuda")
    db = torch.full((C,), 7.0, device="cuda")
    vt = G.t32(v)
    if misalign:   # the same values one float past a 16-byte boundary
        buf = torch.empty(vt.numel() + 1, device="cuda")
        vt = buf[1:].view(vt.shape)
        vt.copy_(G.t32(v))
        assert vt.data_ptr() % 16 != 0
    fno.layer_bwd(plan, vt, z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    torch.cuda.synchronize()
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(G.f32(v), G.f32(dy), G.f32(R), G.f32(W), G.f32(b), modes)
    for name, got, ref in (("dv", dv, dv_r), ("dR", dR, dR_r), ("dW", dW, dW_r), ("db", db, db_r)):
        assert rel_l2(G.np64(got), ref) < TOL, (name, rel_l2(G.np64(got), ref))
    # accumulate = 1 adds into dW / db
    dW2, db2 = dW.clone(), db.clone()
    fno.layer_bwd(plan, vt, z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW2, db2, accumulate=True)
    torch.cuda.synchronize()
    assert rel_l2(G.np64(dW2), 2 * dW_r) < TOL and rel_l2(G.np64(db2), 2 * db_r) < TOL
    plan.destroy()


# Batched mixing: B > 1 reads R once per mode for all batch
# rows (chunks of 16 beyond that); forward and backward vs the oracle.
@pytest.mark.parametrize("B", [4, 8, 20])
def test_batched_mixing_fwd_bwd(B):
    import torch
    from tests import _gpu as G
    import paper_2204_01205_b200 as fno
    grid, C, modes = (16, 16, 16, 8), 6, (4, 4, 4, 4)
    v, R, W, b, dy = _problem(grid, C, modes, B, seed=808 + B)
    plan = G.make_plan(grid, C, modes, B)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    y_ref, z_ref = sp.layer_fwd(G.f32(v), G.f32(R), G.f32(W), G.f32(b), modes)
    assert rel_l2(G.np64(vh), sp.forward_modes(G.f32(v), modes)) < TOL
    assert rel_l2(G.np64(y), y_ref) < TOL
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    torch.cuda.synchronize()
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(G.f32(v), G.f32(dy), G.f32(R), G.f32(W), G.f32(b), modes)
    for name, got, ref in (("dv", dv, dv_r), ("dR", dR, dR_r), ("dW", dW, dW_r), ("db", db, db_r)):
        assert rel_l2(G.np64(got), ref) < TOL, (name, rel_l2(G.np64(got), ref))
    # accumulate adds a second dR
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db, accumulate=True)
    torch.cuda.synchronize()
    assert rel_l2(G.np64(dR), 2 * dR_r) < TOL
