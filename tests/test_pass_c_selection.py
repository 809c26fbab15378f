"""CPU tests of the host-side pass C kernel selection (api.cu fno_plan_create,
pass_c4.cu pass_c4_config; no compute calls): the split backward (family 5:
dv = W^T dz + S^T dz by the forward kernel, dW / db by dw_partial, the
broadcast adjoint of P:64 / Eq. dist_block) is the default wherever
C <= 20 (with pass_c4 as the forward), can be forced for the backward only, and bench.py's
algorithmic bytes follow the family (the dv leg moves slab + dz +
dv, dw_partial dz + v)."""

import importlib.util
import os

import pytest

import paper_2204_01205_b200 as fno

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2204_01205_b200 import build
    build.build()
    return fno.lib()


def _plan(grid, C, modes):
    return fno.Plan(fno.Problem(grid=grid, width=C, modes=modes), allocate=False)


def test_split_backward_and_pass_c4_are_the_defaults_up_to_width_20(L):
    for grid, modes in (((64, 64, 64, 30), (12, 12, 12, 12)),    # BASELINE configs[2] (c3)
                        ((64, 64, 64, 32), (8, 8, 8, 8))):       # configs[1] (c2)
        k = fno.plan_pass_c_kernels(_plan(grid, 20, modes))
        assert k["bwd"]["family"].startswith("split")
        assert k["bwd"]["dv_kernel"] == k["fwd"]["family"]
        assert k["fwd"]["family"].startswith("pass_c4")


def test_split_backward_can_be_forced_and_is_backward_only(L):
    p = _plan((64, 64, 64, 32), 20, (8, 8, 8, 8))
    fno.plan_set_pass_c(p, "bwd", 5)
    assert fno.plan_pass_c_kernels(p)["bwd"]["family"].startswith("split")
    fno.plan_set_pass_c(p, "bwd", 2)
    assert fno.plan_pass_c_kernels(p)["bwd"]["family"].startswith("pass_c2")
    for mode in ("u", "fwd"):
        with pytest.raises(fno.FnoError):
            fno.plan_set_pass_c(p, mode, 5)
    with pytest.raises(fno.FnoError):
        fno.plan_set_pass_c(p, "bwd", 6)


def test_split_backward_needs_width_at_most_20(L):
    wide = _plan((16, 16, 16, 8), 24, (4, 4, 4, 4))
    assert not fno.plan_pass_c_kernels(wide)["bwd"]["family"].startswith("split")
    with pytest.raises(fno.FnoError):
        fno.plan_set_pass_c(wide, "bwd", 5)


def test_bench_algorithmic_bytes_follow_the_backward_family():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    prob = dict(B=1, C=20, local=(64, 64, 64, 30), grid=(64, 64, 64, 30), modes=(12, 12, 12, 12), P=1)
    n = 20 * 64 * 64 * 64 * 30
    slab = 8 * 20 * 64 * 64 * 24 * 12
    fused = bench.stage_bytes(prob, dict(nkz=24, split_bwd=False))
    split = bench.stage_bytes(prob, dict(nkz=24, split_bwd=True))
    assert fused["bwd.pass_c"] == slab + 12 * n          # slab, dz, v -> dv
    assert split["bwd.pass_c"] == slab + 8 * n           # slab, dz -> dv
    assert split["bwd.dw"] == 8 * n                      # dz, v
