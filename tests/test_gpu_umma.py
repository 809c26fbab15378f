"""tcgen05 kind::tf32 operand-layout probe (tests/csrc/umma_probe.cu): one MMA
with K-major interleaved A and B, as pass C uses them, must reproduce an exact
integer GEMM."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_umma_tf32_kmajor_layout_is_exact(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "umma_probe"
    r = subprocess.run([nvcc, "-std=c++17", "-O2", "--expt-relaxed-constexpr", "-diag-suppress", "20013",
                        "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                        os.path.join(HERE, "csrc", "umma_probe.cu")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout
