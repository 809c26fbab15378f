"""Pins of the partition algebra, repartition and the decomposition simulator (P13)."""

import numpy as np
import pytest

from oracle import decomp as dc
from oracle import spectral as sp
from tests._instances import rel_l2


def test_block_range_spec_examples():
    # SPEC block_range examples: (60,4,0) -> [0,15) [PAPER §3.1 60x15 per worker]
    assert dc.block_range(60, 4, 0) == (0, 15)
    assert [dc.block_range(7, 3, i) for i in range(3)] == [(0, 3), (3, 5), (5, 7)]
    assert dc.block_range(2, 4, 3) == (2, 2)
    with pytest.raises(ValueError):
        dc.block_range(5, 2, 2)


def test_local_box_paper_partition():
    # partition 1x1x1x4x1x1 -> per-worker 60x15 in y; coord (0,0,0,1,0,0) -> [15, 30)
    pg = (1, 1, 1, 4, 1, 1)
    r = dc.coords_to_rank(pg, (0, 0, 0, 1, 0, 0))
    box = dc.local_box((1, 2, 60, 60, 64, 30), pg, r)
    assert box[3] == (15, 30) and box[2] == (0, 60)
    assert dc.local_box((9, 9), (3, 3), dc.coords_to_rank((3, 3), (2, 2))) == [(6, 9), (6, 9)]


@pytest.mark.parametrize("shape,pg", [((7, 5), (3, 2)), ((4, 9, 2), (2, 4, 3)), ((1, 1, 8, 6, 3, 2), (1, 1, 4, 2, 1, 1)),
                                      ((2, 3), (4, 1))])
def test_boxes_tile_exactly_once(shape, pg):
    assert dc.all_boxes_tile(shape, pg)


def test_row_major_ranks():
    pg = (1, 1, 2, 2, 2, 1)
    coords = [dc.rank_to_coords(pg, r) for r in range(8)]
    assert coords[1] == (0, 0, 0, 0, 1, 0) and coords[2] == (0, 0, 0, 1, 0, 0) and coords[4] == (0, 0, 1, 0, 0, 0)


def test_transfer_plan_spec_example():
    # (2,) -> (4,) over shape (8,): sender 0 splits [0,4) into [0,2)->0, [2,4)->1; rank 2 receives {4,5}
    plan = dc.transfer_plan((8,), (2,), (4,))
    assert [(s, d, b) for s, d, b in plan if s == 0] == [(0, 0, [(0, 2)]), (0, 1, [(2, 4)])]
    g = np.arange(8.0)
    src = [g[0:4], g[4:8]]
    dst = dc.repartition(src, (8,), (2,), (4,))
    assert list(dst[2]) == [4.0, 5.0]


@pytest.mark.parametrize("shape,P,Q", [((6, 7, 5), (3, 1, 2), (1, 2, 3)),          # Fig. repartition shapes
                                       ((1, 2, 8, 6, 4, 3), (1, 1, 2, 2, 1, 1), (1, 1, 1, 1, 4, 1)),
                                       ((5, 4), (2, 2), (4, 1))])
def test_repartition_definition_roundtrip_adjoint(shape, P, Q):
    rng = np.random.default_rng(0)
    g = rng.standard_normal(shape)
    nP = int(np.prod(P))
    src = [g[tuple(slice(lo, hi) for lo, hi in dc.local_box(shape, P, r))] for r in range(nP)]
    dst = dc.repartition(src, shape, P, Q)
    # definition: destination worker holds the global tensor restricted to its box
    for r, blk in enumerate(dst):
        ref = g[tuple(slice(lo, hi) for lo, hi in dc.local_box(shape, Q, r))]
        assert np.array_equal(blk, ref)
    # round trip R_{Q->P} R_{P->Q} = I, bitwise
    back = dc.repartition(dst, shape, Q, P)
    assert all(np.array_equal(a, b) for a, b in zip(back, src))
    # adjoint: <R x, y> = <x, R_{Q->P} y>
    h = rng.standard_normal(shape)
    ys = [h[tuple(slice(lo, hi) for lo, hi in dc.local_box(shape, Q, r))] for r in range(int(np.prod(Q)))]
    lhs = sum(np.sum(a * b) for a, b in zip(dst, ys))
    rhs = sum(np.sum(a * b) for a, b in zip(src, dc.repartition(ys, shape, Q, P)))
    assert abs(lhs - rhs) < 1e-12 * max(1, abs(lhs))


@pytest.mark.parametrize("mz,P", [(8, 8), (12, 8), (4, 3), (1, 4), (16, 8)])
def test_kz_ownership_partitions_retained_set(mz, P):
    """SPEC mode-ownership invariant: union of owned modes == sequential set, no duplicates."""
    owned = []
    for r in range(P):
        lo, hi = dc.owned_kz(mz, P, r)
        owned.extend(range(lo, hi))
    assert owned == list(range(2 * mz))


@pytest.mark.parametrize("pg", [(1, 1), (2, 1), (2, 2), (4, 2), (3, 3), (1, 4)])
def test_p13_decomposition_simulator_matches_undecomposed(pg):
    grid, modes = (8, 8, 8, 6), (2, 3, 3, 3)
    rng = np.random.default_rng(1)
    v = rng.standard_normal((2, 3) + grid)
    R = rng.standard_normal((3, 3, 4, 6, 6, 3)) + 1j * rng.standard_normal((3, 3, 4, 6, 6, 3))
    ref = sp.spectral_conv(v, R, modes)
    got = dc.simulate_spectral_conv(v, R, modes, pg)
    assert rel_l2(got, ref) < 1e-14
