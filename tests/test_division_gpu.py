"""The STRICT locate's division (div_axis in csrc/b2m_mover.cuh: q = x*rd,
r = fma(-q, d, x), fma(r, rd, q) with rd = RN(1/d)) against the IEEE
division __ddiv_rn on the GPU: random positions over 40 binades below l for
the C1-C5 / test spacings and 4000 random spacings, and every position within
32 ulps of each cell face.  grid_cell_of (grid.hpp:69-71) needs RN(x/d)
exactly, so any difference would break STRICT's bitwise contract."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_division_matches_ieee(gpu, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "div_check"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                    "-I" + os.path.join(ROOT, "include"),
                    "-I" + os.path.join(ROOT, "paper_1904_03684_b200", "csrc"),
                    os.path.join(ROOT, "tools", "micro", "div_check.cu"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "faces:" in r.stdout and " 0 mismatches" in r.stdout, r.stdout
