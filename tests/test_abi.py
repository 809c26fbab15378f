"""CPU tests of the C-ABI library: it loads, exports every symbol include/fno.h
declares, validates problems, and its host-side plan logic (local boxes, kz
ownership, workspace sizing) agrees with the partition algebra of the paper
 as pinned in tests/test_oracle_decomp.py.  No compute calls."""

import ctypes

import numpy as np
import os
import re

import pytest

import paper_2204_01205_b200 as fno
from oracle import decomp as dc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2204_01205_b200 import build
    build.build()
    return fno.lib()


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "fno.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fno_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(L):
    syms = _declared_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(L, s), f"libfno.so does not export {s}"
    assert L.fno_abi_version() == 1
    assert L.fno_status_string(0) == b"FNO_OK"
    assert L.fno_status_string(6) == b"FNO_ERR_WORKSPACE"


@pytest.mark.parametrize("bad,expect", [
    (dict(grid=(0, 8, 8, 8)), 1),
    (dict(modes=(5, 2, 2, 2)), 1),          # 2m > n on x
    (dict(modes=(2, 2, 2, 6)), 1),          # mt > T/2 + 1
    (dict(width=0), 1),
    (dict(pgrid=(2, 1)), 1),                # px*py != comm size (NULL comm)
])
def test_plan_validation(L, bad, expect):
    args = dict(grid=(8, 8, 8, 8), width=2, modes=(2, 2, 2, 2))
    args.update(bad)
    with pytest.raises(fno.FnoError) as e:
        fno.Plan(fno.Problem(**args), allocate=False)
    assert e.value.status == expect


def test_unsupported_transform_size_is_a_plan_error(L):
    with pytest.raises(fno.FnoError) as e:
        fno.Plan(fno.Problem(grid=(8, 8, 7, 8), width=2, modes=(2, 2, 2, 2)), allocate=False)
    assert e.value.status == 2


@pytest.mark.parametrize("grid,pg,mz", [((64, 64, 64, 32), (4, 2), 8), ((16, 16, 16, 8), (2, 2), 4),
                                        ((64, 64, 64, 30), (2, 1), 12), ((256, 256, 64, 32), (4, 2), 2)])
def test_boxes_and_kz_ownership_match_partition_algebra(L, grid, pg, mz):
    P = pg[0] * pg[1]
    owned = []
    for r in range(P):
        comm = fno.Comm.local(P, r)
        plan = fno.Plan(fno.Problem(grid=grid, width=4, modes=(4, 4, mz, 4), pgrid=pg), comm, allocate=False)
        box = plan.local_box()
        ref = dc.local_box((1, 4) + tuple(grid), (1, 1, pg[0], pg[1], 1, 1), r)[2:]
        assert [tuple(b) for b in box] == [tuple(b) for b in ref]
        lo, hi = plan.owned_modes()
        assert (lo, hi) == dc.owned_kz(mz, P, r)
        owned.extend(range(lo, hi))
        assert plan.workspace_size() > 0
        plan.destroy()
        comm.destroy()
    assert owned == list(range(2 * mz))


def test_workspace_errors(L):
    plan = fno.Plan(fno.Problem(grid=(16, 16, 16, 8), width=4, modes=(4, 4, 4, 4)), allocate=False)
    with pytest.raises(fno.FnoError) as e:
        fno._check(L.fno_plan_set_workspace(plan.handle, ctypes.c_void_p(256), 16), "set_workspace")
    assert e.value.status == 6
    # compute call before the workspace is set -> invalid state
    st = L.fno_spectral_conv_fwd(plan.handle, ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.c_void_p(256), None, None)
    assert st == 3


def test_repartition_workspace_query_and_validation(L):
    n = ctypes.c_size_t(0)
    shp = (ctypes.c_int64 * 2)(8, 6)
    one = (ctypes.c_int32 * 2)(1, 1)
    assert L.fno_repartition(None, 2, shp, one, one, 4, None, None, None, ctypes.byref(n), None) == 0
    assert n.value >= 2 * 8 * 6 * 4
    two = (ctypes.c_int32 * 2)(2, 1)
    assert L.fno_repartition(None, 2, shp, one, two, 4, None, None, None, ctypes.byref(n), None) == 1


@pytest.mark.parametrize("grid,pg,io", [((16, 16, 16, 8), (2, 1), (1, 1, 2, 1)), ((16, 16, 16, 8), (2, 1), (1, 1, 1, 2)),
                                        ((32, 16, 64, 30), (2, 2), (1, 2, 2, 1)), ((64, 64, 64, 32), (4, 2), (2, 1, 2, 2)),
                                        ((16, 16, 16, 8), (2, 2), (2, 2, 1, 1))])
def test_io_partition_boxes_tile_the_domain(L, grid, pg, io):
    """fno_plan_set_io_partition: every rank's io box is the
    balanced block of the row-major (px', py', pz', pt') grid (partition algebra
    of the oracle), the boxes tile the domain, and the workspace grows by the
    staging buffers unless io is the plan's own x/y grid."""
    P = pg[0] * pg[1]
    cover = np.zeros(grid, dtype=np.int32)
    for r in range(P):
        comm = fno.Comm.local(P, r)
        base = fno.Plan(fno.Problem(grid=grid, width=4, modes=(4, 4, 4, 4), pgrid=pg), comm, allocate=False)
        plan = fno.Plan(fno.Problem(grid=grid, width=4, modes=(4, 4, 4, 4), pgrid=pg), comm, allocate=False, io_pgrid=io)
        box = plan.io_box()
        ref = dc.local_box((1, 4) + tuple(grid), (1, 1) + tuple(io), r)[2:]
        assert [tuple(b) for b in box] == [tuple(b) for b in ref]
        cover[tuple(slice(lo, hi) for lo, hi in box)] += 1
        same = tuple(io) == (pg[0], pg[1], 1, 1)
        assert (plan.workspace_size() == base.workspace_size()) if same else (plan.workspace_size() > base.workspace_size())
        plan.destroy()
        base.destroy()
        comm.destroy()
    assert (cover == 1).all()


def test_io_partition_validation(L):
    comm = fno.Comm.local(2, 0)
    plan = fno.Plan(fno.Problem(grid=(16, 16, 16, 8), width=4, modes=(4, 4, 4, 4), pgrid=(2, 1)), comm, allocate=False)
    for bad, status in [((1, 1, 1, 1), 1),      # 1 rank != 2
                        ((1, 1, 3, 1), 1),      # 16 % 3 != 0, and 3 ranks
                        ((1, 1, 1, 16), 1)]:    # 16 ranks
        arr = (ctypes.c_int32 * 4)(*bad)
        assert L.fno_plan_set_io_partition(plan.handle, arr) == status
    ok = (ctypes.c_int32 * 4)(1, 1, 2, 1)
    assert L.fno_plan_set_io_partition(plan.handle, ok) == 0
    assert L.fno_plan_set_io_partition(plan.handle, ok) == 3     # already set
    plan.destroy()
    # after the workspace is set: invalid state
    plan2 = fno.Plan(fno.Problem(grid=(16, 16, 16, 8), width=4, modes=(4, 4, 4, 4)), allocate=False)
    fno._check(L.fno_plan_set_workspace(plan2.handle, ctypes.c_void_p(1 << 20), plan2.workspace_size()), "set_workspace")
    one = (ctypes.c_int32 * 4)(1, 1, 1, 1)
    assert L.fno_plan_set_io_partition(plan2.handle, one) == 3
    plan2.destroy()
    comm.destroy()
