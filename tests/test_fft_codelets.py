"""Host (CPU) unit test of the register FFT codelets used by every kernel
(paper_2204_01205_b200/csrc/fft.cuh): nvcc builds tests/csrc/test_fft_host.cu
as a host program, which compares fft<N, DIR> for N in {2..64} (radix 2, 3,
4, 5 and a prime) with a brute-force double DFT and checks the constexpr
twiddle generator against libm."""

import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"), reason="no nvcc")
def test_fft_codelets_match_brute_force_dft(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "test_fft_host"
    src = os.path.join(HERE, "csrc", "test_fft_host.cu")
    r = subprocess.run([nvcc, "-std=c++17", "-O2", "--expt-relaxed-constexpr", "-diag-suppress", "20013",
                        "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout
