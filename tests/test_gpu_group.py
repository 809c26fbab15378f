"""Decomposed-path parity on ONE GPU: the P ranks of an x/y decomposition as a
plan group (fno_group_*, include/fno.h).  Every rank's box, the send-ready slab
chunks stored straight into the kz owners' buffers (exchange 1), pass B on
the owned kz block with the kz-sharded R, the y-inverse stores into the
x/y owners' buffers (exchange 2, the adjoint) and the rank-ordered dW / db
sum run exactly as on P GPUs; only the transport differs (same-device
stores in stream order instead of NVLink peer stores + barrier).  This is the
driver-visible check of rows a2 / a6 / e on a 1-GPU box, including P = 8 (4,2);
the NVLink / NCCL transports themselves are tests/test_gpu_multi.py.

Bars (north star): decomposed vs fp64 oracle rel-L2 <= 1e-5; decomposed vs the
single-GPU plan on the same inputs <= 1e-5 (S_dist = S)."""

import numpy as np
import pytest

import synth
from oracle import spectral as sp
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


def _run_group(pgrid, grid, C, modes, B, v, R, W, b, dy, act="gelu"):
    """Layer fwd + bwd and the spectral conv through a plan group; results
    gathered to global arrays (x/y boxes, kz blocks of dR / V^)."""
    import torch
    import paper_2204_01205_b200 as fno
    from tests import _gpu as G
    g = fno.PlanGroup(fno.Problem(grid=grid, width=C, modes=modes, batch=B, pgrid=pgrid, act=act))
    boxes = [p.local_box() for p in g.plans]
    kzs = [p.owned_modes() for p in g.plans]
    loc = lambda a, r: np.ascontiguousarray(a[:, :, boxes[r][0][0]:boxes[r][0][1], boxes[r][1][0]:boxes[r][1][1]])
    vs = [G.t32(loc(v, r)) for r in range(g.n)]
    dys = [G.t32(loc(dy, r)) for r in range(g.n)]
    Rs = [G.tc64(R[:, :, :, :, kzs[r][0]:kzs[r][1]]) for r in range(g.n)]
    Wt, bt = G.t32(W), G.t32(b)
    ys = [torch.empty_like(t) for t in vs]
    zs = [torch.empty_like(t) for t in vs]
    vhs = [torch.empty(p.vhat_shape(), dtype=torch.complex64, device="cuda") for p in g.plans]
    fno.group_layer_fwd(g, vs, Rs, Wt, bt, ys, zs, vhs)
    dvs = [torch.empty_like(t) for t in vs]
    dRs = [torch.empty(p.weight_shape(), dtype=torch.complex64, device="cuda") for p in g.plans]
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.group_layer_bwd(g, vs, zs, vhs, dys, Rs, Wt, dvs, dRs, dW, db)
    us = [torch.empty_like(t) for t in vs]
    fno.group_spectral_conv_fwd(g, vs, Rs, us)
    torch.cuda.synchronize()

    def gather(ts):
        out = np.zeros(v.shape, dtype=np.float64)
        for r, t in enumerate(ts):
            (x0, x1), (y0, y1) = boxes[r][0], boxes[r][1]
            out[:, :, x0:x1, y0:y1] = G.np64(t)
        return out

    res = {"y": gather(ys), "z": gather(zs), "dv": gather(dvs), "u": gather(us),
           "dR": np.concatenate([G.np64(t) for t in dRs], axis=4),
           "vh": np.concatenate([G.np64(t) for t in vhs], axis=4),
           "dW": G.np64(dW), "db": G.np64(db)}
    g.destroy()
    return res


def _run_single(grid, C, modes, B, v, R, W, b, dy, act="gelu"):
    import torch
    import paper_2204_01205_b200 as fno
    from tests import _gpu as G
    plan = G.make_plan(grid, C, modes, B, act=act)
    y, z, vh = G.layer_fwd(plan, v, R, W, b)
    dyt = G.t32(dy)
    dv = torch.empty_like(dyt)
    dR = torch.empty(plan.weight_shape(), dtype=torch.complex64, device="cuda")
    dW = torch.empty((C, C), device="cuda")
    db = torch.empty((C,), device="cuda")
    fno.layer_bwd(plan, G.t32(v), z, vh, dyt, G.tc64(R), G.t32(W), dv, dR, dW, db)
    u, _ = G.spectral_fwd(plan, v, R)
    torch.cuda.synchronize()
    res = {k: G.np64(t) for k, t in dict(y=y, z=z, dv=dv, u=u, dR=dR, vh=vh, dW=dW, db=db).items()}
    plan.destroy()
    return res


def _inputs(grid, C, modes, B, seed, shape="ns"):
    v = synth.field((B, C) + tuple(grid), modes, seed, shape)
    R = synth.spectral_weights(C, C, modes, seed + 1)
    W, b = synth.channel_weights(C, seed + 2)
    dy = synth.cotangent(v.shape, seed + 3)
    return v, R, W, b, dy


# (pgrid, grid, C, modes, B): every pgrid the bench runs ((2,1) (2,2) (4,2)) and
# the SPEC-style corner cases (1,py), 2mz < P (ranks owning no modes), odd sizes
CASES = [
    ((2, 1), (16, 16, 16, 8), 4, (4, 4, 4, 4), 1),        # c1 at P = 2
    ((1, 2), (16, 16, 16, 8), 3, (4, 4, 4, 4), 2),        # y-split, batch 2
    ((2, 2), (16, 16, 16, 8), 4, (4, 4, 4, 4), 1),        # c1 at P = 4
    ((4, 2), (16, 16, 16, 8), 4, (4, 4, 4, 4), 1),        # c1 at P = 8 (the bench's 8-GPU pgrid)
    ((4, 1), (16, 8, 16, 8), 2, (2, 2, 1, 4), 1),         # 2mz = 2 < P = 4: two ranks own no modes
    ((2, 2), (32, 32, 64, 30), 20, (12, 12, 12, 12), 1),  # c3 class at width 20 (T = 30, CP = 20 kernels)
    ((4, 2), (32, 32, 64, 30), 20, (12, 12, 12, 12), 1),  # c3 class at P = 8: 2mz = 24 -> 3 kz planes per rank
    ((2, 1), (12, 10, 12, 10), 3, (3, 2, 3, 3), 2),       # odd sizes, C % 4 != 0
]


def _ids(c):
    return f"pg{c[0][0]}x{c[0][1]}_" + "x".join(map(str, c[1])) + f"_C{c[2]}_B{c[4]}"


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_group_decomposed_matches_oracle_and_single(case):
    from tests import _gpu as G
    pgrid, grid, C, modes, B = case
    v, R, W, b, dy = _inputs(grid, C, modes, B, seed=900 + C, shape="co2" if grid[3] == 30 else "ns")
    res = _run_group(pgrid, grid, C, modes, B, v, R, W, b, dy)
    one = _run_single(grid, C, modes, B, v, R, W, b, dy)
    for k in one:
        assert rel_l2(res[k], one[k]) < TOL, (k, rel_l2(res[k], one[k]))
    v64, R64, W64, b64, dy64 = G.f32(v), G.f32(R), G.f32(W), G.f32(b), G.f32(dy)
    y_r, z_r = sp.layer_fwd(v64, R64, W64, b64, modes)
    assert rel_l2(res["y"], y_r) < TOL
    assert rel_l2(res["z"], z_r) < TOL
    assert rel_l2(res["u"], sp.spectral_conv(v64, R64, modes)) < TOL
    dv_r, dR_r, dW_r, db_r = sp.layer_bwd(v64, dy64, R64, W64, b64, modes)
    assert rel_l2(res["dv"], dv_r) < TOL
    assert rel_l2(res["dR"], dR_r) < TOL
    assert rel_l2(res["dW"], dW_r) < TOL
    assert rel_l2(res["db"], db_r) < TOL


@pytest.mark.slow
@pytest.mark.parametrize("pgrid", [(2, 1), (2, 2), (4, 2)], ids=lambda p: f"pg{p[0]}x{p[1]}")
def test_group_full_size_c3_matches_single(pgrid):
    """BASELINE configs[2] (c3: 64^3 x 30, width 20, modes 12, fwd+bwd) at full
    size on the bench's strong-scaling pgrids: decomposed == single-GPU on every
    output (the single-GPU c3 path is itself checked against the oracle in
    tests/test_gpu_parity.py)."""
    import torch
    cfg = synth.CONFIGS[3]
    grid, C, modes = cfg["grid"], cfg["width"], cfg["modes"]
    pr = synth.problem(3, with_dy=True)
    res = _run_group(pgrid, grid, C, modes, 1, pr["v"], pr["R"], pr["W"], pr["b"], pr["dy"])
    one = _run_single(grid, C, modes, 1, pr["v"], pr["R"], pr["W"], pr["b"], pr["dy"])
    bad = {k: rel_l2(res[k], one[k]) for k in one if not rel_l2(res[k], one[k]) < TOL}
    assert not bad, bad
    torch.cuda.empty_cache()


def test_group_rejects_per_plan_calls_and_bad_groups():
    import torch
    import paper_2204_01205_b200 as fno
    g = fno.PlanGroup(fno.Problem(grid=(16, 16, 16, 8), width=4, modes=(4, 4, 4, 4), pgrid=(2, 1)))
    p = g.plans[0]
    v = torch.zeros(p.local_shape(), device="cuda")
    R = torch.zeros(p.weight_shape(), dtype=torch.complex64, device="cuda")
    with pytest.raises(fno.FnoError) as e:
        fno.spectral_conv_fwd(p, v, R, torch.empty_like(v))
    assert e.value.status == 3
    # plans out of rank order are not a group
    h = (fno.ctypes.c_void_p * 2)(g.plans[1].handle.value, g.plans[0].handle.value)
    ptrs = (fno.ctypes.c_void_p * 2)(v.data_ptr(), v.data_ptr())
    rs = (fno.ctypes.c_void_p * 2)(R.data_ptr(), R.data_ptr())
    assert fno.lib().fno_group_spectral_conv_fwd(2, h, ptrs, rs, ptrs, None, None) == 3
    g.destroy()
