"""Bounds and injectivity of the tiled fill's fp32 shadow layout (block-major
rows with interleaved quad minima, rotor_common.cuh), checked on the host by
tests/native/layout_check.cu: every cell / quad-minimum row inside its table
and used once, every ring stage the middle copies contiguous and in bounds."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shadow_layout_bounds(tmp_path):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "layout_check"
    src = os.path.join(ROOT, "tests", "native", "layout_check.cu")
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_1911_13214_b200", "csrc")]
    subprocess.run([nvcc, "-std=c++17", "-O1", *inc, src, "-o", str(exe)], check=True, capture_output=True)
    r = subprocess.run([str(exe), "1000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "layout ok" in r.stdout
