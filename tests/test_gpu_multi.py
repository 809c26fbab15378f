"""Multi-GPU parity of the x/y-decomposed path (NCCL pencil all-to-all):
decomposed == single-GPU == fp64 oracle within 1e-5 (north star), plus the
repartition round trip.  Needs >= 2 visible GPUs; run as
`gpurun --gpus 2 -- python -m pytest tests -m gpu -k multi`."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


CASES = [((2, 1), [16, 16, 16, 8], 4, [4, 4, 4, 4], 1),
         ((1, 2), [16, 16, 16, 8], 3, [4, 4, 4, 4], 2),
         ((2, 1), [32, 16, 64, 30], 6, [12, 8, 12, 12], 1),
         ((2, 2), [16, 16, 16, 8], 4, [4, 4, 4, 4], 1),
         ((2, 2), [32, 32, 64, 32], 5, [8, 8, 8, 8], 1),
         ((4, 1), [16, 8, 16, 8], 2, [2, 2, 1, 4], 1)]    # 2mz = 2 < P: ranks with no modes


# exchange transport: direct NVLink peer stores (default) or NCCL send/recv
@pytest.mark.parametrize("peer", ["1", "0"], ids=["peer", "nccl"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"pg{c[0][0]}x{c[0][1]}_" + "x".join(map(str, c[1])))
def test_decomposed_matches_single_and_oracle(case, peer, tmp_path):
    pg, grid, C, modes, B = case
    n = pg[0] * pg[1]
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    from paper_2204_01205_b200 import build
    build.build()
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(ROOT, "tests", "mp_parity.py"),
           "--pgrid", str(pg[0]), str(pg[1]), "--grid", *map(str, grid), "--width", str(C),
           "--modes", *map(str, modes), "--batch", str(B), "--out", str(out)]
    env = dict(os.environ, FNO_PEER_EXCHANGE=peer)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    for k, v in res.items():
        if k.endswith("_vs_oracle") or k.endswith("_vs_single"):
            assert v < 1e-5, (k, v, res)
    for f in res["repartition"]:
        assert f["repart_fwd_exact"] and f["repart_roundtrip_exact"], res


# whole network: decomposed fno_net_* == fp64 network oracle
NET_CASES = [((2, 1), [16, 16, 16, 8], 4, [4, 4, 4, 4], "1"),
             ((1, 2), [16, 16, 16, 8], 4, [4, 2, 4, 4], "0"),
             ((2, 2), [16, 16, 32, 16], 6, [4, 4, 8, 8], "1")]


@pytest.mark.parametrize("case", NET_CASES, ids=lambda c: f"net_pg{c[0][0]}x{c[0][1]}_peer{c[4]}")
def test_decomposed_network_matches_oracle(case, tmp_path):
    pg, grid, C, modes, peer = case
    n = pg[0] * pg[1]
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    from paper_2204_01205_b200 import build
    build.build()
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29613", os.path.join(ROOT, "tests", "mp_network.py"),
           "--pgrid", str(pg[0]), str(pg[1]), "--grid", *map(str, grid), "--width", str(C),
           "--modes", *map(str, modes), "--out", str(out)]
    env = dict(os.environ, FNO_PEER_EXCHANGE=peer)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    bad = {k: v for k, v in res.items() if k.endswith("_vs_oracle") and not v < 1e-5}
    assert not bad, bad


# data x domain hybrid: gradients averaged over replicas == mean oracle gradient
HYB_CASES = [(2, (1, 1)), (2, (2, 1))]


@pytest.mark.parametrize("case", HYB_CASES, ids=lambda c: f"dp{c[0]}_pg{c[1][0]}x{c[1][1]}")
def test_data_domain_hybrid_gradients_match_oracle(case, tmp_path):
    dp, pg = case
    n = dp * pg[0] * pg[1]
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    from paper_2204_01205_b200 import build
    build.build()
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29615", os.path.join(ROOT, "tests", "mp_hybrid.py"),
           "--dp", str(dp), "--pgrid", str(pg[0]), str(pg[1]), "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["replicas_identical"]
    bad = {k: v for k, v in res.items() if k.endswith("_vs_oracle") and not v < 1e-5}
    assert not bad, bad


# caller-side 3-D spatial / temporal partitions: io partition
# != the plan's x/y grid, repartitioned around the layer
IO_CASES = [((2, 1), (1, 1, 2, 1)), ((2, 1), (1, 1, 1, 2)), ((1, 2), (2, 1, 1, 1)),
            ((2, 2), (1, 2, 2, 1)), ((2, 2), (1, 1, 2, 2))]


@pytest.mark.parametrize("case", IO_CASES, ids=lambda c: f"pg{c[0][0]}x{c[0][1]}_io" + "x".join(map(str, c[1])))
def test_io_partition_layer_matches_oracle(case, tmp_path):
    pg, io = case
    n = pg[0] * pg[1]
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    from paper_2204_01205_b200 import build
    build.build()
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29617", os.path.join(ROOT, "tests", "mp_io.py"),
           "--pgrid", str(pg[0]), str(pg[1]), "--io", *map(str, io), "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    bad = {k: v for k, v in res.items() if k.endswith("_vs_oracle") and not v < 1e-5}
    assert not bad, bad
